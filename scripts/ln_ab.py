"""LayerNorm kernels at the C2 launch shape (M = 2048 rows, h = 2048):
CUDA-graph-timed (20 launches) row-parallel vs staged LN backward (with the
fused residual column sum and the partial reduce) and the LN forward;
achieved GB/s of the algorithmic bytes vs the measured HBM peak.
python scripts/ln_ab.py > gpurun_out/ln_ab.jsonl"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch  # noqa: E402

from paper_2503_03182_b200 import kernels as K  # noqa: E402
from gemm_vs_cublas import timed  # noqa: E402

peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6547.2) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6547.2
M, h = 2048, 2048
dev, bf = "cuda", torch.bfloat16
x = torch.randn((M, h), device=dev).to(bf)
dy = torch.randn((M, h), device=dev).to(bf)
res = torch.randn((M, h), device=dev).to(bf)
y, dx = torch.empty_like(x), torch.empty_like(x)
g, b = torch.ones(h, device=dev, dtype=bf), torch.zeros(h, device=dev, dtype=bf)
mean, rstd = torch.empty(M, device=dev), torch.empty(M, device=dev)
dg, db, drs = torch.zeros(h, device=dev), torch.zeros(h, device=dev), torch.zeros(h, device=dev)
ws = torch.empty(3 * ((M + 15) // 16) * h, device=dev)
K.tpipe_k_ln_fwd(1, x, g, b, y, mean, rstd, M, h)
rows = []
for rows_on in (0, 1, 0, 1):
    K.tpipe_k_ln_set_rows_bwd(rows_on)
    t = timed(lambda: K.tpipe_k_ln_bwd_rsum(1, dy, x, g, mean, rstd, res, dx, dg, db, drs, ws, M, h))
    alg = 4 * 2 * M * h + 8 * M
    rows.append({"kernel": "ln_bwd_rsum(+reduce)", "rows_kernel": rows_on, "us": round(t * 1e3, 2),
                 "GBs": round(alg / t / 1e6, 1), "frac": round(alg / t / 1e6 / peak, 3)})
K.tpipe_k_ln_set_rows_bwd(1)
t = timed(lambda: K.tpipe_k_ln_fwd(1, x, g, b, y, mean, rstd, M, h))
alg = 2 * 2 * M * h + 8 * M
rows.append({"kernel": "ln_fwd", "us": round(t * 1e3, 2), "GBs": round(alg / t / 1e6, 1),
             "frac": round(alg / t / 1e6 / peak, 3)})
for r in rows:
    print(json.dumps(r))
