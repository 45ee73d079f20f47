"""T-Offload timing on the bench workload at N=1 (bench.measure_offload vs
T-Recomp without offload): python scripts/offload_time.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import synth

class A: steps = 4
c = bench.C2
tok, tgt = synth.tokens(c["vocab"], c["m"], 1, c["seq_len"], step=0, vocab_eff=c["vocab_eff"])
dtok = torch.tensor(tok, dtype=torch.int32, device="cuda")
dtgt = torch.tensor(tgt, dtype=torch.int32, device="cuda")
base = bench.quick_measure("tpipe_trecomp", 1, c["m"], dtok, dtgt, A)
print(json.dumps({"tpipe_trecomp": base}))
print(json.dumps(bench.measure_offload(1, c["m"], dtok, dtgt, A, base["ms_per_step"])))
print(json.dumps(bench.measure_offload(1, c["m"], dtok, dtgt, A, base["ms_per_step"], device_opt=True)))
