"""SM-clock timeline of CTA 0 of one tcgen05 GEMM launch (probe library
libtpipe_gprobe.so): MMA k-block issue times, operand-wait completions,
epilogue windows, producer empty-waits. Prints per-k-block issue intervals
(floor = 4 MMAs x N/2 cycles) split by whether an epilogue was running.
  TPIPE_GEMM_PROBE=<bits> python scripts/gemm_trace.py [shape]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_03182_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.join(ROOT, "paper_2503_03182_b200", "libtpipe_gprobe.so")
from paper_2503_03182_b200 import kernels as K  # noqa: E402
from gemm_vs_cublas import shapes  # noqa: E402

N_TR = 1024
if os.environ.get("GEMM_WIDE") is not None:
    K.tpipe_k_gemm_set_wide_choice(int(os.environ["GEMM_WIDE"]))
want = sys.argv[1] if len(sys.argv) > 1 else "fc1_fprop"
for name, m, n, k, ak, bk, epi in shapes:
    if name != want:
        continue
    A = torch.randn((m, k) if ak else (k, m), device="cuda").to(torch.bfloat16)
    B = torch.randn((n, k) if bk else (k, n), device="cuda").to(torch.bfloat16)
    f32 = epi in (K.EPI_ACC_F32, K.EPI_STORE_F32)
    C = torch.zeros((m, n), device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    C2 = torch.empty((m, n), device="cuda", dtype=torch.bfloat16)
    Rr = torch.zeros((m, n), device="cuda", dtype=torch.bfloat16)
    bias = torch.zeros(n, device="cuda", dtype=torch.bfloat16)

    def run():
        K.tpipe_k_gemm(1, m, n, k, A, k if ak else m, ak, B, k if bk else n, bk, epi, C, n, bias=bias,
                       R=Rr, ldr=n, C2=C2, ldc2=n, aux=Rr, ldaux=n)
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    buf = torch.zeros(14 * N_TR, dtype=torch.int64, device="cuda")
    L = _lib.lib()
    L.tpipe_gemm_trace_set.argtypes = [_lib.vp]
    L.tpipe_gemm_trace_set(buf.data_ptr())
    run()
    torch.cuda.synchronize()
    L.tpipe_gemm_trace_set(None)
    tr = buf.view(14, N_TR).cpu().numpy().astype(np.int64)
    t0 = tr[:5][tr[:5] > 0].min()
    issue, fullw, ep0, ep1, empw = [r[r > 0] - t0 for r in tr[:5]]
    nb = int((tr[5] > 0).sum())
    g0 = tr[5][:nb].min()
    entry, exit_, first_mma, last_epi = [(tr[e][:nb] - g0) for e in (5, 6, 9, 10)]
    clk = (tr[8][:nb] - tr[7][:nb]) / np.maximum(tr[6][:nb] - tr[5][:nb], 1)   # cycles per ns = GHz
    ctas = {"n": nb, "kernel_span_ns": int(exit_.max()), "entry_ns_max": int(entry.max()),
            "first_mma_ns": [int(first_mma[first_mma > 0].min()), int(np.median(first_mma[first_mma > 0])),
                             int(first_mma[first_mma > 0].max())],
            "last_epilogue_done_ns_p10_50_90_max": [int(np.percentile(last_epi, q)) for q in (10, 50, 90, 100)],
            "exit_ns_p10_50_90_max": [int(np.percentile(exit_, q)) for q in (10, 50, 90, 100)],
            "sm_ghz_median": float(np.median(clk))}
    kbs = (k + 63) // 64
    bn = 256
    floor_kb = 4 * bn // 2
    iv = np.diff(issue)
    in_epi = np.zeros(len(iv), bool)
    for a, b in zip(ep0, ep1):
        in_epi |= (issue[1:] > a) & (issue[:-1] < b)
    tile_start = (np.arange(1, len(issue)) % kbs) == 0
    out = {"probe": int(os.environ.get("TPIPE_GEMM_PROBE", "0")), "kernel": name, "kblocks_per_tile": kbs,
           "n_kblocks": int(len(issue)), "floor_cycles_per_kblock": floor_kb,
           "total_cycles": int(issue[-1] - issue[0]) if len(issue) else 0,
           "kblock_interval_median": float(np.median(iv)),
           "kblock_interval_mean_in_epilogue": float(iv[in_epi & ~tile_start].mean()) if (in_epi & ~tile_start).any() else None,
           "kblock_interval_mean_no_epilogue": float(iv[~in_epi & ~tile_start].mean()) if (~in_epi & ~tile_start).any() else None,
           "tile_boundary_intervals": [int(x) for x in iv[tile_start]],
           "epilogue_windows": [[int(a), int(b)] for a, b in zip(ep0, ep1)],
           "tile_first_issue": [int(issue[i]) for i in range(0, len(issue), kbs)],
           "full_wait_minus_prev_issue_p50": float(np.median(fullw[1:len(issue)] - issue[:len(fullw[1:len(issue)])])),
           "epi_chunks": [[int(tr[e][i] - t0) if tr[e][i] else 0 for e in (11, 12, 13)] for i in range(32)],
           "interval_pcts": {p: float(np.percentile(iv, p)) for p in (10, 50, 90, 99)}, "ctas": ctas}
    print(json.dumps(out))
