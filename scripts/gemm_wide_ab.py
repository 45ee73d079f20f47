"""A/B of 256x512 vs 256x256 CTA-pair tiles (tpipe_k_gemm_set_wide) on the
GEMM shapes of one GPT-3 1.3B layer + the LM head, production epilogues.
Each case: 20 launches captured in one CUDA graph, CUDA-event timed replay.
python scripts/gemm_wide_ab.py > gpurun_out/gemm_wide_ab.jsonl"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_03182_b200 import kernels as K

h, s, f, V = 2048, 2048, 8192, 50304
M = s
E = K
shapes = [("qkv_fprop", M, 3 * h, h, 1, 1, E.EPI_BIAS), ("o_fprop", M, h, h, 1, 1, E.EPI_BIAS_RES),
          ("fc1_fprop", M, f, h, 1, 1, E.EPI_BIAS_GELU), ("fc2_fprop", M, h, f, 1, 1, E.EPI_BIAS_RES),
          ("fc2_dgrad", M, f, h, 1, 0, E.EPI_DGELU), ("fc2_wgrad", h, f, M, 0, 0, E.EPI_ACC_F32),
          ("fc1_wgrad", f, h, M, 0, 0, E.EPI_ACC_F32), ("fc1_dgrad", M, h, f, 1, 0, E.EPI_STORE),
          ("o_wgrad", h, h, M, 0, 0, E.EPI_ACC_F32), ("o_dgrad", M, h, h, 1, 0, E.EPI_STORE),
          ("qkv_wgrad", 3 * h, h, M, 0, 0, E.EPI_ACC_F32), ("qkv_dgrad", M, h, 3 * h, 1, 0, E.EPI_STORE),
          ("head_fprop", M, V, h, 1, 1, E.EPI_STORE_F32), ("head_dgrad", M, h, V, 1, 0, E.EPI_STORE),
          ("head_wgrad", V, h, M, 0, 0, E.EPI_ACC_F32)]


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            for _ in range(iters):
                fn()
    torch.cuda.current_stream().wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


tot = {0: 0.0, 1: 0.0}
for name, m, n, k, ak, bk, epi in shapes:
    A = torch.randn((m, k) if ak else (k, m), device="cuda").to(torch.bfloat16)
    B = torch.randn((n, k) if bk else (k, n), device="cuda").to(torch.bfloat16)
    f32 = epi in (E.EPI_ACC_F32, E.EPI_STORE_F32)
    C = torch.zeros((m, n), device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    C2 = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
    Rr = torch.zeros((m, n), device="cuda", dtype=torch.bfloat16)
    bias = torch.zeros(n, device="cuda", dtype=torch.bfloat16)
    fn = lambda: K.tpipe_k_gemm(1, m, n, k, A, k if ak else m, ak, B, k if bk else n, bk, epi, C, n,
                                bias=bias, R=Rr, ldr=n, C2=C2, ldc2=n, aux=Rr, ldaux=n)
    row = {"kernel": name, "M": m, "N": n, "K": k}
    for wide in (0, 1):
        K.tpipe_k_gemm_set_wide(wide)
        ms = timed(fn)
        tot[wide] += ms
        row[f"wide{wide}_us"] = round(ms * 1e3, 2)
        row[f"wide{wide}_tflops"] = round(2 * m * n * k / ms / 1e9, 1)
    K.tpipe_k_gemm_set_wide(0)
    print(json.dumps(row), flush=True)
    del A, B, C, C2, Rr
print(json.dumps({"total_ms": {"wide0": round(tot[0], 4), "wide1": round(tot[1], 4)}}))
