"""Two model GEMM shapes through cuBLAS (torch.matmul) and through our
tcgen05 kernel, for a side-by-side ncu capture (warm caches):

  ncu --set full --cache-control none --clock-control none \
      -k regex:"nvjet|gemm_tc" -o rep python scripts/gemm_vs_cublas_ncu.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2503_03182_b200 import kernels as K  # noqa: E402

for (m, n, k) in ((2048, 8192, 2048), (2048, 2048, 2048)):
    A = torch.randn(m, k, device="cuda").bfloat16()
    W = torch.randn(n, k, device="cuda").bfloat16()
    C = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        torch.matmul(A, W.t(), out=C)             # cuBLAS, C = A W^T
    for _ in range(3):
        K.tpipe_k_gemm(1, m, n, k, A, k, 1, W, k, 1, K.EPI_STORE, C, n)
    torch.cuda.synchronize()
    print(m, n, k, flush=True)
