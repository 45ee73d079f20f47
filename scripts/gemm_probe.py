"""Run one GEMM shape a few times (for ncu A/B): python scripts/gemm_probe.py M N K ak bk epi sk"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_03182_b200 import kernels as K
M, N, Kd, ak, bk, epi, sk = (int(v) for v in sys.argv[1:8])
K.tpipe_k_gemm_set_stream_k(sk)
A = torch.randn((M, Kd) if ak else (Kd, M), device="cuda").to(torch.bfloat16)
B = torch.randn((N, Kd) if bk else (Kd, N), device="cuda").to(torch.bfloat16)
f32 = epi in (K.EPI_ACC_F32, K.EPI_STORE_F32)
C = torch.zeros((M, N), device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
bias = torch.zeros(N, device="cuda", dtype=torch.bfloat16)
for _ in range(6):
    K.tpipe_k_gemm(1, M, N, Kd, A, Kd if ak else M, ak, B, Kd if bk else N, bk, epi, C, N, bias=bias)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    K.tpipe_k_gemm(1, M, N, Kd, A, Kd if ak else M, ak, B, Kd if bk else N, bk, epi, C, N, bias=bias)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"M={M} N={N} K={Kd} sk={sk} ms={ms:.4f} tflops={2*M*N*Kd/ms/1e9:.1f}")
