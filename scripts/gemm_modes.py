"""GEMM schedule A/B on the model shapes: single-CTA vs CTA-pair tiles (CUDA
events, warm; the stream-K arm was removed with the schedule). python scripts/gemm_modes.py [c3]"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_03182_b200 import kernels as K

h, s, f = 2048, 2048, 8192
if len(sys.argv) > 1 and sys.argv[1] == "c3":
    h, s, f = 4096, 4096, 16384
M = s
E = K
shapes = [("qkv_fprop", M, 3 * h, h, 1, 1, E.EPI_BIAS), ("o_fprop", M, h, h, 1, 1, E.EPI_BIAS_RES),
          ("fc1_fprop", M, f, h, 1, 1, E.EPI_BIAS_GELU), ("fc2_fprop", M, h, f, 1, 1, E.EPI_BIAS_RES),
          ("fc2_dgrad", M, f, h, 1, 0, E.EPI_DGELU), ("fc2_wgrad", h, f, M, 0, 0, E.EPI_ACC_F32),
          ("fc1_wgrad", f, h, M, 0, 0, E.EPI_ACC_F32), ("fc1_dgrad", M, h, f, 1, 0, E.EPI_STORE),
          ("o_wgrad", h, h, M, 0, 0, E.EPI_ACC_F32), ("o_dgrad", M, h, h, 1, 0, E.EPI_STORE),
          ("qkv_wgrad", 3 * h, h, M, 0, 0, E.EPI_ACC_F32), ("qkv_dgrad", M, h, 3 * h, 1, 0, E.EPI_STORE)]


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


tot = {}
for name, m, n, k, ak, bk, epi in shapes:
    A = torch.randn((m, k) if ak else (k, m), device="cuda").to(torch.bfloat16)
    B = torch.randn((n, k) if bk else (k, n), device="cuda").to(torch.bfloat16)
    f32 = epi in (E.EPI_ACC_F32, E.EPI_STORE_F32)
    C = torch.zeros((m, n), device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    C2 = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
    Rr = torch.zeros((m, n), device="cuda", dtype=torch.bfloat16)
    bias = torch.zeros(n, device="cuda", dtype=torch.bfloat16)
    row = {"kernel": name, "M": m, "N": n, "K": k}
    for pair in (0, 1):
        for sk in (0,):
            K.tpipe_k_gemm_set_pair(pair)
            fn = lambda: K.tpipe_k_gemm(1, m, n, k, A, k if ak else m, ak, B, k if bk else n, bk, epi, C, n,
                                        bias=bias, R=Rr, ldr=n, C2=C2, ldc2=n, aux=Rr, ldaux=n)
            ms = timeit(fn)
            key = f"pair{pair}_sk{sk}"
            row[key] = round(2 * m * n * k / ms / 1e9, 1)
            tot[key] = tot.get(key, 0.0) + ms
    print(json.dumps(row), flush=True)
K.tpipe_k_gemm_set_pair(1)
print(json.dumps({"total_ms_per_layer_set": {k: round(v, 4) for k, v in tot.items()}}))
