"""A/B of the CTA-pair crossover in the bench step (C2 1.3B, T-Pipe, p=1,
m=32): python scripts/ab_gemm_pair.py [steps]; interleaved repetitions."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import synth
from paper_2503_03182_b200 import plan as P, runtime as RT
from paper_2503_03182_b200._lib import lib

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
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
ext = torch.cuda.ExternalStream(rt.stream())


def run(k):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    for _ in range(k):
        rt.step_device(dt.data_ptr(), dg.data_ptr())
    e1.record(ext)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


for rep in range(3):
    for n in (96, 64, 48):
        lib().tpipe_k_gemm_set_pair_min_tiles(n)
        run(2)
        ms = run(steps)
        print(json.dumps({"rep": rep, "pair_min_tiles": n, "ms_per_step": round(ms, 2),
                          "tokens_s": round(65536 / ms * 1e3, 1)}), flush=True)
lib().tpipe_k_gemm_set_pair_min_tiles(96)
