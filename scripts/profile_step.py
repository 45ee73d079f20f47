"""Runs N training steps of the bench workload (for ncu captures):
python scripts/profile_step.py [steps] [strategy]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import synth
from paper_2503_03182_b200 import plan as P, runtime as RT

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
strategy = sys.argv[2] if len(sys.argv) > 2 else "tpipe"
c = bench.C2
md = P.Model(c["n_layers"], c["hidden"], c["n_heads"], c["ffn_hidden"], c["vocab"], c["seq_len"],
             c["micro_batch"], P.BF16)
plan = P.Plan(md, 1, c["m"], strategy=strategy)
rt = RT.Runtime(plan, stage=-1, lr=1e-4)
rng = np.random.default_rng(0)
for ch in range(1, plan.v + 1):
    rt.set_params(0, ch, bench.init_chunk(plan, 0, ch, rng))
tok, tgt = synth.tokens(c["vocab"], c["m"], 1, c["seq_len"], vocab_eff=c["vocab_eff"])
dt = torch.tensor(tok, dtype=torch.int32, device="cuda")
dg = torch.tensor(tgt, dtype=torch.int32, device="cuda")
for i in range(steps):
    loss = rt.step_device(dt.data_ptr(), dg.data_ptr())
    print("step", i, "loss", loss, "launches", rt.stats()["kernel_launches"], flush=True)
