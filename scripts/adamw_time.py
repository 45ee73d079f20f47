"""AdamW over 64M parameters (bf16 weights), CUDA-graph-timed: achieved GB/s of
the 30 algorithmic bytes per parameter vs the measured HBM peak."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch  # noqa: E402

from paper_2503_03182_b200 import kernels as K  # noqa: E402
from gemm_vs_cublas import timed  # noqa: E402

n = 1 << 26
dev = "cuda"
master, m, v, g = (torch.randn(n, device=dev), torch.zeros(n, device=dev), torch.zeros(n, device=dev),
                   torch.randn(n, device=dev))
w = torch.empty(n, device=dev, dtype=torch.bfloat16)
t = timed(lambda: K.tpipe_k_adamw(1, master, m, v, g, w, n, 1, 1e-4, 0.9, 0.95, 1e-8, 0.1, 0.1, 0.05))
print(json.dumps({"kernel": "adamw_64M", "us": round(t * 1e3, 1), "GBs": round(30 * n / t / 1e6, 1),
                  "frac": round(30 * n / t / 1e6 / 6547.2, 3)}))
