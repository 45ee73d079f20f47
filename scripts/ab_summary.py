"""Summarise gpurun_out/gemm_ab.jsonl (+ gemm_trace_ab.jsonl): best-of time per shape and library."""
import json
import sys
from collections import defaultdict

import numpy as np

rows = [json.loads(l) for l in open("gpurun_out/gemm_ab.jsonl")]
t = defaultdict(lambda: defaultdict(list))
for r in rows:
    t[r["kernel"]][r["lib"]].append(r["us"])
tot = defaultdict(float)
for k, v in t.items():
    best = {lib: min(xs) for lib, xs in v.items()}
    libs = sorted(best)
    print(f"{k:11s}", best, f"ratio {libs[0]}/{libs[-1]} = {best[libs[0]] / best[libs[-1]]:.3f}")
    if k != "sq8192":
        for lib, x in best.items():
            tot[lib] += x
libs = sorted(tot)
print(dict(tot), f"speedup {libs[0]}/{libs[-1]}", round(tot[libs[0]] / tot[libs[-1]], 4))
try:
    for l in open("gpurun_out/gemm_trace_ab.jsonl"):
        d = json.loads(l)
        ch = [c[0] for c in d["epi_chunks"] if c[0]]
        print(d["kernel"], "span_ns", d["ctas"]["kernel_span_ns"], "ghz", round(d["ctas"]["sm_ghz_median"], 3),
              "epi", d["epilogue_windows"][:2], "chunk intervals", [int(x) for x in np.diff(ch[:4])])
except FileNotFoundError:
    pass
