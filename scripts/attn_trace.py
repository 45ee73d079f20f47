"""Timeline of CTA 0's roles in the tcgen05 attention kernels (probe build
libtpipe_trace.so, `make trace`: SM clock64 stamps, events listed in
attn_tc5.cu TR(...)). Bench shape by default: b=1 s=2048 a=16 d=128.

    python scripts/attn_trace.py [b s a d] > gpurun_out/attn_trace.txt
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2503_03182_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.join(ROOT, "paper_2503_03182_b200", "libtpipe_trace.so")
from paper_2503_03182_b200 import kernels as K  # noqa: E402

b, s, a, d = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (1, 2048, 16, 128)
TR_N, NEV = 512, 26
h = a * d
torch.manual_seed(0)
qkv = torch.randn((b * s, 3 * h), device="cuda").to(torch.bfloat16)
o = torch.empty((b * s, h), device="cuda", dtype=torch.bfloat16)
lse = torch.empty((b, a, s), device="cuda")
dout = torch.randn_like(o)
dqkv = torch.empty_like(qkv)
ws = torch.empty((b, a, s), device="cuda")
buf = torch.zeros(NEV * TR_N, dtype=torch.int64, device="cuda")
assert _lib.lib().tpipe_attn_trace_set(_lib.C.c_void_p(buf.data_ptr())) == 0


def run():
    K.tpipe_k_attn_fwd(1, qkv, o, lse, b, s, a, d)
    K.tpipe_k_attn_bwd(1, qkv, o, dout, lse, dqkv, ws, b, s, a, d)


for _ in range(3):
    run()
torch.cuda.synchronize()
buf.zero_()
run()
torch.cuda.synchronize()
T = buf.cpu().numpy().reshape(NEV, TR_N).astype(np.int64)


def series(ev):
    x = T[ev]
    n = int(np.max(np.nonzero(x)[0]) + 1) if np.any(x) else 0
    return x[:n]


def report(name, evs, labels):
    xs = {e: series(e) for e in evs}
    t0 = min(int(v[v > 0].min()) for v in xs.values() if len(v) and np.any(v > 0))
    n = max(len(v) for v in xs.values())
    print(f"== {name}: CTA 0, {n} units; clock64 relative to the first stamp")
    print("  g " + " ".join(f"{labels[e]:>9s}" for e in evs))
    for g in range(n):
        row = []
        for e in evs:
            v = xs[e]
            row.append(f"{int(v[g]) - t0:9d}" if g < len(v) and v[g] else f"{'-':>9s}")
        print(f"{g:3d} " + " ".join(row))
    return xs, t0


res = {}
fw = report("fwd2", [0, 1, 24, 3, 4, 5, 6, 7, 2, 25],
            {0: "Kload", 1: "S_iss", 24: "S_done", 3: "S_seen", 4: "max_st", 5: "P_st", 6: "pfull0", 7: "pfull7",
             2: "PV_iss", 25: "PV_done"})
kv = report("dkdv2", [8, 9, 11, 12, 13, 14, 15, 10],
            {8: "Qload", 9: "S_iss", 11: "ld_seen", 12: "S_seen", 13: "ld_done", 14: "pfull0", 15: "pfull7",
             10: "G_iss"})
dq = report("dq2", [16, 17, 19, 20, 21, 22, 23, 18],
            {16: "KVload", 17: "S_iss", 19: "gd_seen", 20: "S_seen", 21: "ld_done", 22: "pfull0", 23: "pfull7",
             18: "G_iss"})


def med(x):
    x = np.asarray(x, dtype=np.float64)
    return float(np.median(x)) if len(x) else float("nan")


def summary(name, xs, pairs):
    out = {}
    for lab, (e0, e1) in pairs.items():
        a0, a1 = xs[e0], xs[e1]
        n = min(len(a0), len(a1))
        dd = [int(a1[i]) - int(a0[i]) for i in range(2, n) if a0[i] and a1[i]]
        out[lab] = med(dd)
    print(name, json.dumps(out))
    res[name] = out


summary("fwd2 median cycles", fw[0], {"S_issue->seen": (1, 3), "seen->max_stored": (3, 4),
                                       "max->P_stored": (4, 5), "P_stored->pfull": (5, 6),
                                       "pfull->PV_issue": (6, 2)})
summary("dkdv2 median cycles", kv[0], {"S_issue->seen": (9, 12), "seen->ld_done": (12, 13),
                                        "ld_done->pfull": (13, 14), "pfull->G_issue": (14, 10)})
summary("dq2 median cycles", dq[0], {"S_issue->seen": (17, 20), "seen->ld_done": (20, 21),
                                      "ld_done->pfull": (21, 22), "pfull->G_issue": (22, 18)})
for nm, xs, e in (("fwd2", fw[0], 3), ("dkdv2", kv[0], 12), ("dq2", dq[0], 20)):
    v = xs[e]
    per = np.diff(v[v > 0].astype(np.int64))
    print(f"{nm} period between consecutive S_seen: median {med(per):.0f} cycles, n={len(per)}")
