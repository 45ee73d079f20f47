"""Which part of the tcgen05 GEMM pipeline bounds each model shape?
Runs the probe library (libtpipe_gprobe.so, `make -C paper_2503_03182_b200 gprobe`)
with TPIPE_GEMM_PROBE = 0 (full kernel), 1 (no TMA loads), 2 (no epilogue
math/stores), 3 (neither): CUDA-graph-timed, 20 launches per graph.
  for p in 0 1 2 3; do TPIPE_GEMM_PROBE=$p python scripts/gemm_probe.py; done"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2503_03182_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.join(ROOT, "paper_2503_03182_b200",
                            os.environ.get("TPIPE_PROBE_LIB", "libtpipe_gprobe.so"))
from paper_2503_03182_b200 import kernels as K  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "scripts"))
from gemm_vs_cublas import shapes, timed  # noqa: E402

probe = int(os.environ.get("TPIPE_GEMM_PROBE", "0"))
wide = os.environ.get("GEMM_WIDE")
if wide is not None:
    K.tpipe_k_gemm_set_wide_choice(int(wide))
only = os.environ.get("GEMM_PROBE_SHAPES")
for name, m, n, k, ak, bk, epi in shapes:
    if only and name not in only.split(","):
        continue
    A = torch.randn((m, k) if ak else (k, m), device="cuda").to(torch.bfloat16)
    B = torch.randn((n, k) if bk else (k, n), device="cuda").to(torch.bfloat16)
    f32 = epi in (K.EPI_ACC_F32, K.EPI_STORE_F32)
    C = torch.zeros((m, n), device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    C2 = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
    Rr = torch.zeros((m, n), device="cuda", dtype=torch.bfloat16)
    bias = torch.zeros(n, device="cuda", dtype=torch.bfloat16)
    ours = lambda: K.tpipe_k_gemm(1, m, n, k, A, k if ak else m, ak, B, k if bk else n, bk, epi, C, n,  # noqa: E731
                                  bias=bias, R=Rr, ldr=n, C2=C2, ldc2=n, aux=Rr, ldaux=n)
    t = timed(ours)
    fl = 2 * m * n * k
    print(json.dumps({"lib": os.path.basename(_lib.LIB_PATH) + ("" if wide is None else f":wide{wide}") + f":p{probe}", "probe": probe, "kernel": name, "M": m, "N": n, "K": k, "us": round(t * 1e3, 2),
                      "tflops": round(fl / t / 1e9, 1)}), flush=True)
    del A, B, C, C2, Rr
