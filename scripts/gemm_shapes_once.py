"""Run each model-shape GEMM of one C2 layer (fwd + bwd, 12 shapes) twice:
a warm-up pass, then a measured pass, in the production configuration (CTA
pairs, data-parallel). For ncu: -k regex:gemm_tc_kernel -s 12 -c 12 captures
the second pass in shape order; prints the shapes and algorithmic bytes.
python scripts/gemm_shapes_once.py"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_03182_b200 import kernels as K

h, s, f = 2048, 2048, 8192
M = s
E = K
shapes = [("qkv_fprop", M, 3 * h, h, 1, 1, E.EPI_BIAS), ("o_fprop", M, h, h, 1, 1, E.EPI_BIAS_RES),
          ("fc1_fprop", M, f, h, 1, 1, E.EPI_BIAS_GELU), ("fc2_fprop", M, h, f, 1, 1, E.EPI_BIAS_RES),
          ("fc2_dgrad", M, f, h, 1, 0, E.EPI_DGELU), ("fc2_wgrad", h, f, M, 0, 0, E.EPI_ACC_F32),
          ("fc1_wgrad", f, h, M, 0, 0, E.EPI_ACC_F32), ("fc1_dgrad", M, h, f, 1, 0, E.EPI_STORE),
          ("o_wgrad", h, h, M, 0, 0, E.EPI_ACC_F32), ("o_dgrad", M, h, h, 1, 0, E.EPI_STORE),
          ("qkv_wgrad", 3 * h, h, M, 0, 0, E.EPI_ACC_F32), ("qkv_dgrad", M, h, 3 * h, 1, 0, E.EPI_STORE)]
calls = []
for name, m, n, k, ak, bk, epi in shapes:
    A = torch.randn((m, k) if ak else (k, m), device="cuda").to(torch.bfloat16)
    B = torch.randn((n, k) if bk else (k, n), device="cuda").to(torch.bfloat16)
    f32 = epi in (E.EPI_ACC_F32, E.EPI_STORE_F32)
    C = torch.zeros((m, n), device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    C2 = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
    Rr = torch.zeros((m, n), device="cuda", dtype=torch.bfloat16)
    bias = torch.zeros(n, device="cuda", dtype=torch.bfloat16)
    # algorithmic bytes: A, B once; C written (fp32 reduce-add: read+write); residual / aux read; 2nd output
    byts = 2 * (m * k + n * k) + (8 if epi == E.EPI_ACC_F32 else 2) * m * n
    if epi in (E.EPI_BIAS_RES, E.EPI_DGELU):
        byts += 2 * m * n
    if epi in (E.EPI_BIAS_GELU, E.EPI_DGELU):
        byts += 2 * m * n
    fn = (lambda m=m, n=n, k=k, A=A, ak=ak, B=B, bk=bk, epi=epi, C=C, bias=bias, Rr=Rr, C2=C2:
          K.tpipe_k_gemm(1, m, n, k, A, k if ak else m, ak, B, k if bk else n, bk, epi, C, n,
                         bias=bias, R=Rr, ldr=n, C2=C2, ldc2=n, aux=Rr, ldaux=n))
    calls.append((name, m, n, k, byts, fn))
K.tpipe_k_gemm_set_pair(1)
for rep in range(2):
    for c in calls:
        c[5]()
    torch.cuda.synchronize()
for name, m, n, k, byts, _ in calls:
    print(json.dumps({"kernel": name, "M": m, "N": n, "K": k, "flops": 2 * m * n * k, "alg_bytes": byts}))
