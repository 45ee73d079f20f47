"""Host issue time vs step time on the bench workload (is the step
submission-bound?): python scripts/host_issue.py"""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import synth
from paper_2503_03182_b200 import plan as P, runtime as RT

c = bench.C2
md = P.Model(c["n_layers"], c["hidden"], c["n_heads"], c["ffn_hidden"], c["vocab"], c["seq_len"],
             c["micro_batch"], P.BF16)
plan = P.Plan(md, 1, c["m"], strategy="tpipe")
rt = RT.Runtime(plan, stage=-1, lr=1e-4)
rng = np.random.default_rng(0)
for ch in range(1, plan.v + 1):
    rt.set_params(0, ch, bench.init_chunk(plan, 0, ch, rng))
tok, tgt = synth.tokens(c["vocab"], c["m"], 1, c["seq_len"], vocab_eff=c["vocab_eff"])
dt = torch.tensor(tok, dtype=torch.int32, device="cuda")
dg = torch.tensor(tgt, dtype=torch.int32, device="cuda")
for i in range(5):
    t0 = time.perf_counter()
    rt.step_device(dt.data_ptr(), dg.data_ptr())
    wall = (time.perf_counter() - t0) * 1e3
    st = rt.stats()
    print(json.dumps({"step": i, "wall_ms": round(wall, 1), "host_issue_ms": round(st["host_issue_ms"], 1),
                      "launches": st["kernel_launches"]}), flush=True)
