#!/usr/bin/env python
"""bench.py — TPipe training-step throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tpipe|reference]

Workload (BASELINE.json configs[1]): GPT-3 1.3B (L=24, h=2048, a=16,
ffn=8192, V=50304), seq 2048, micro-batch 1, m=32 micro-batches per step
(65,536 tokens), bf16, T-Pipe schedule with p = N pipeline stages (one stage
per GPU; at N=1 the two T-Pipe chunks run on one GPU). Synthetic seeded
tokens (uniform < 50257) and random-init weights (N(0, 0.02)).

A "step" is one pass of the whole hot path: every F/B(/R) op of every
micro-batch in the plan's order, the stage transport, and the AdamW update.
`value` = tokens/s over all ranks with tokens already resident in HBM;
`e2e` = the same through tpipe_step with host (pinned) tokens copied in and
the loss copied out inside the timed region. The step's working set
(weights + activations, >> 126 MB L2) exceeds L2, so no explicit flush.
`roofline` = the dominant kernel class (tcgen05 GEMMs), algorithmic 2MNK
FLOPs / summed CUDA-event durations of its launches, from a profiled pass of
the same K steps (events on the runtime's launch stream), vs the measured
sustained bf16 peak in MEASURED_PEAKS.json.
`cpu_baseline` = the fp64 NumPy oracle (oracle/model.py) doing one
micro-batch forward+backward of one layer at the same (h, s), scaled to
model tokens/s (/L), on this host's cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "max trainable params at fixed HBM/GPU; tokens/s vs 1F1B+recomp, 1-8 B200"
C2 = dict(n_layers=24, hidden=2048, n_heads=16, ffn_hidden=8192, vocab=50304, seq_len=2048,
          micro_batch=1, vocab_eff=50257, m=32)
C5 = dict(hidden=4096, n_heads=32, ffn_hidden=16384, vocab=32000, seq_len=8192, micro_batch=1)
BUDGET = 80 * 2 ** 30


def model_flops_per_token(c):
    """Algorithmic FLOPs/token, causal attention at its triangle:
    L(72h^2 + 6sh) + 6hV (uses ffn = 4h)."""
    L, h, s, V = c["n_layers"], c["hidden"], c["seq_len"], c["vocab"]
    return L * (72 * h * h + 6 * s * h) + 6 * h * V


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, idx):
        self.idx, self.samples, self.stop = idx, [], threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons}


def init_chunk(plan, s, c, rng):
    """Random-init packed chunk vector (N(0,0.02) matrices, LN gamma 1, zero
    biases) in the packed order of DESIGN.md §2.3."""
    from paper_2503_03182_b200 import params as PR
    h, f = plan.model.hidden, plan.model.ffn_hidden
    V, sl = plan.model.vocab, plan.model.seq_len
    shapes = {"wte": (V, h), "wpe": (sl, h), "lnf_g": (h,), "lnf_b": (h,), "w_head": (V, h)}
    import synth
    shapes.update(synth.layer_shapes(h, f))
    parts = []
    for k, _l in PR.chunk_entries(plan.p, plan.v, plan.partition, s, c):
        shp = shapes[k]
        n = int(np.prod(shp))
        if len(shp) == 2:
            parts.append(rng.standard_normal(n, dtype=np.float32) * np.float32(0.02))
        elif k.endswith("_g"):
            parts.append(np.ones(n, np.float32))
        else:
            parts.append(np.zeros(n, np.float32))
    return np.concatenate(parts)


def cpu_baseline(c, seconds_cap=30.0):
    """fp64 oracle: one micro-batch forward+backward of ONE layer at (h, s) of
    the workload; model tokens/s = layer tokens/s / L."""
    from oracle import model as R
    import synth
    h, f, s, a = c["hidden"], c["ffn_hidden"], c["seq_len"], c["n_heads"]
    W = synth.weights(1, h, f, 64, s, seed=1)
    L = R.to64(W)["layers"][0]
    rng = np.random.default_rng(0)
    x = rng.standard_normal((1, s, h))
    dy = rng.standard_normal((1, s, h))
    t0 = time.perf_counter()
    n = 0
    while True:
        y, cache = R.layer_fwd(x, L, a)
        R.layer_bwd(dy, cache, L, a)
        n += 1
        if time.perf_counter() - t0 > seconds_cap / 3 or n >= 3:
            break
    dt = time.perf_counter() - t0
    layer_tps = n * s / dt
    try:
        from threadpoolctl import threadpool_info
        blas = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        blas = None
    cores = len(os.sched_getaffinity(0))
    # single-thread figure: the same layer on one core, bounded
    # to a 512-token slice of the sequence (attention cost grows with s)
    one = None
    try:
        from threadpoolctl import threadpool_limits
        s1 = min(s, 512)
        with threadpool_limits(limits=1):
            t3 = time.perf_counter()
            y, cache = R.layer_fwd(x[:, :s1], L, a)
            R.layer_bwd(dy[:, :s1], cache, L, a)
            dt1 = time.perf_counter() - t3
        one = {"value": round(s1 / dt1 / c["n_layers"], 3), "unit": "tokens/s", "threads": 1,
               "sample": f"1 micro-batch fwd+bwd of 1 layer on a {s1}-token slice (h={h}), fp64, "
                         f"{dt1:.1f}s; / L={c['n_layers']}"}
    except Exception as e:   # reported, not fatal
        one = {"error": str(e)[:120]}
    # SURVEY §8(d) "oracle timing beside the GPU": (i) the exact schedule simulator
    # for p = 8, m = 32, all strategies; (ii) one full fp64 training step of C1
    from oracle import schedule as S
    t1 = time.perf_counter()
    for st in ("tpipe", "tpipe_trecomp", "1f1b", "1f1b_full_recomp", "interleave", "interleave_trecomp"):
        orders, v, rec, dur = S.strategy_orders(st, 8, 32)
        S.simulate(orders, 8, v, dur, rec)
    sim_s = time.perf_counter() - t1
    W1 = synth.weights(8, 64, 256, 256, 32, seed=1)
    tok1, tgt1 = synth.tokens(256, 8, 2, 32, step=0)
    t2 = time.perf_counter()
    R.step_grads(R.to64(W1), tok1, tgt1, 4)
    c1_s = time.perf_counter() - t2
    return {"value": layer_tps / c["n_layers"], "unit": "tokens/s", "cores": cores,
            "blas_threads": blas, "kind": "oracle",
            "schedule_sim_p8_m32_all_strategies_s": round(sim_s, 3),
            "c1_fp64_step_s": round(c1_s, 3), "single_thread": one,
            "sample": f"{n} x (1 micro-batch fwd+bwd of 1 layer, h={h}, s={s}, fp64 NumPy) "
                      f"in {dt:.1f}s; model tokens/s = layer tokens/s / L={c['n_layers']}"}


WORKLOADS = {  # BASELINE.json configs[2] / [3] layer shapes
    "c3": dict(name="configs[2]: Llama-style 7B shape (L=32, h=4096, a=32, ffn=16384, V=32000, s=4096)",
               n_layers=32, hidden=4096, n_heads=32, ffn_hidden=16384, vocab=32000, seq_len=4096),
    "c4": dict(name="configs[3]: Llama-style 13B shape (L=40, h=5120, a=40, ffn=20480, V=32000, s=8192)",
               n_layers=40, hidden=5120, n_heads=40, ffn_hidden=20480, vocab=32000, seq_len=8192),
}


def run_workload(args):
    """The C3 / C4 model shapes through the same runtime on ONE B200 (p = 1,
    m = 8): the planner's auto ladder (R28) under the GPU's free HBM picks the
    strategy (C4 needs T-Recomp + T-Offload to fit). Not the 8-stage configs
    themselves (one GPU here); a throughput line at those shapes."""
    import torch
    from paper_2503_03182_b200 import plan as P, runtime as RT
    import synth
    w = WORKLOADS[args.workload]
    m = 8
    md = P.Model(w["n_layers"], w["hidden"], w["n_heads"], w["ffn_hidden"], w["vocab"], w["seq_len"], 1, P.BF16)
    free_b, _ = torch.cuda.mem_get_info()
    budget = int(free_b * 0.93) - (1 << 30)
    plan = P.Plan(md, 1, m, hbm_budget=budget, strategy="auto",
                  offload=P.OFFLOAD_MODEL_STATE | P.OFFLOAD_DEVICE_OPT | P.OFFLOAD_ACTIVATIONS)
    rt = RT.Runtime(plan, stage=-1, lr=1e-5)
    pool = (np.random.default_rng(5).standard_normal(1 << 24, dtype=np.float32) * np.float32(0.02))
    for ch in range(1, plan.v + 1):
        rt.set_params(0, ch, fast_init_chunk(plan, 0, ch, pool))
    tok, tgt = synth.tokens(w["vocab"], m, 1, w["seq_len"], step=0)
    dtok = torch.tensor(tok, dtype=torch.int32, device="cuda")
    dtgt = torch.tensor(tgt, dtype=torch.int32, device="cuda")
    ext = torch.cuda.ExternalStream(rt.stream())
    for _ in range(args.warmup):
        rt.step_device(dtok.data_ptr(), dtgt.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(0) as clk:
        e0.record(ext)
        for _ in range(args.steps):
            rt.step_device(dtok.data_ptr(), dtgt.data_ptr())
        e1.record(ext)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    tokens = m * w["seq_len"]
    fl = model_flops_per_token(w)
    _, _, pk, src = peaks()
    st = rt.stats()
    out = {"metric": METRIC, "value": round(tokens / (ms / 1e3), 1), "unit": "tokens/s", "n_gpus": 1,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 2), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights)",
           "config": {"workload": w["name"] + ", p=1 on one B200, m=8", "params_B": round(plan.params_total / 1e9, 2),
                      "hbm_budget_GiB": round(budget / 2 ** 30, 1),
                      "plan": {"strategy": ["1f1b", "1f1b_full_recomp", "tpipe", "tpipe_trecomp", "interleave",
                                            "interleave_trecomp"][plan.strategy], "offload": plan.offload,
                               "recomp_layers": plan.recomp_layers, "chunks": plan.v},
                      "plan_peak_GiB": round(plan.peak(0)["total_peak"] / 2 ** 30, 2),
                      "pool_high_water_GiB": round(st["pool_high_water"][0] / 2 ** 30, 2)},
           "mfu": round(tokens / (ms / 1e3) * fl / (pk * 1e12), 4), "mfu_peak": f"{pk} ({src})",
           "clocks": clk.summary()}
    rt.close()
    return out


def oracle_layer_timing():
    """fp64 oracle, one layer forward + backward of one micro-batch at the C3
    (Llama-7B shape, s = 4096) and C4 (13B shape, s = 8192) layer shapes,
    all host cores (SURVEY §8(d) item iii). C4's attention at s = 8192 would
    materialise 40 x 8192^2 fp64 scores (21 GB per tensor), so C4 is timed on
    a 2048-token sample and reported as such."""
    from oracle import model as R
    import synth
    out = {}
    for name, (h, a, f, s, s_run) in {"C3": (4096, 32, 16384, 4096, 4096),
                                      "C4": (5120, 40, 20480, 8192, 2048)}.items():
        W = synth.weights(1, h, f, 64, s_run, seed=1)
        L = R.to64(W)["layers"][0]
        rng = np.random.default_rng(0)
        x = rng.standard_normal((1, s_run, h))
        t0 = time.perf_counter()
        y, cache = R.layer_fwd(x, L, a)
        R.layer_bwd(x, cache, L, a)
        dt = time.perf_counter() - t0
        out[name] = {"h": h, "a": a, "ffn": f, "seq_len": s, "tokens_timed": s_run, "s": round(dt, 2),
                     "layer_tokens_per_s": round(s_run / dt, 2), "cores": len(os.sched_getaffinity(0))}
        del cache, y
    return out


def capacity(p, strategies=("1f1b", "tpipe", "tpipe_trecomp", "tpipe_all", "interleave",
                            "interleave_trecomp")):
    """Max trainable layers / params under an 80 GiB per-GPU plan peak for the
    C5 sweep shape (h=4096, s=8192), L in steps of p (planner byte model)."""
    from paper_2503_03182_b200 import plan as P
    from paper_2503_03182_b200._lib import TPipeError
    out = {}
    for st in strategies:
        strat, off = ("tpipe_trecomp", 1) if st == "tpipe_all" else (st, 0)
        best = None
        L = 2 * p
        while L <= 400:
            md = P.Model(L, C5["hidden"], C5["n_heads"], C5["ffn_hidden"], C5["vocab"],
                         C5["seq_len"], C5["micro_batch"], P.BF16)
            try:
                pl = P.Plan(md, p, 32, hbm_budget=BUDGET, strategy=strat, offload=off)
                best = (L, pl.params_total)
            except TPipeError:
                break
            L += 2 * p
        out[st] = {"max_layers": best[0] if best else 0,
                   "max_params_B": round(best[1] / 1e9, 2) if best else 0}
    return out


def fast_init_chunk(plan, s, c, pool):
    """init_chunk's layout (N(0,0.02) matrices, gamma 1, zero biases) with the
    matrix values tiled from one pre-drawn N(0,0.02) pool: multi-billion-param
    models initialise in seconds (throughput does not depend on the values)."""
    from paper_2503_03182_b200 import params as PR
    import synth
    h, f = plan.model.hidden, plan.model.ffn_hidden
    V, sl = plan.model.vocab, plan.model.seq_len
    shapes = {"wte": (V, h), "wpe": (sl, h), "lnf_g": (h,), "lnf_b": (h,), "w_head": (V, h)}
    shapes.update(synth.layer_shapes(h, f))
    ents = PR.chunk_entries(plan.p, plan.v, plan.partition, s, c)
    out = np.empty(sum(int(np.prod(shapes[k])) for k, _ in ents), np.float32)
    off = 0
    for k, _l in ents:
        shp = shapes[k]
        n = int(np.prod(shp))
        if len(shp) == 2:
            for o in range(0, n, pool.size):
                w = min(pool.size, n - o)
                out[off + o: off + o + w] = pool[:w]
        else:
            out[off: off + n] = 1.0 if k.endswith("_g") else 0.0
        off += n
    return out


CAP_P, CAP_BUDGET_GIB, CAP_M = 8, 20, 16


def plan_of(md, p, m, budget, strat, off):
    """P.Plan for a strategy name with an optional '@v<chunks>' suffix ('auto':
    the ladder also tries 3 and 4 chunks) or '@r50' (1F1B + layer-grouped
    recompute of half of each stage's layers, the paper's 1F1B + R50)."""
    from paper_2503_03182_b200 import plan as P
    if strat.endswith("@r50"):
        return P.Plan(md, p, m, hbm_budget=budget, strategy=strat[:-4], offload=off,
                      recomp_layers=max(1, md.n_layers // p // 2))
    name, _, v = strat.partition("@v")
    return P.Plan(md, p, m, hbm_budget=budget, strategy=name, offload=off,
                  chunks=int(v) if v else (0 if name == "auto" else 2))


def capacity_plans(p=CAP_P, budget=CAP_BUDGET_GIB * 2 ** 30, m=CAP_M):
    """Largest L (multiple of p) each strategy fits under `budget` bytes per
    stage for the C5 shape (h=4096, s=8192), from the planner's byte model."""
    from paper_2503_03182_b200 import plan as P
    from paper_2503_03182_b200._lib import TPipeError
    ms = P.OFFLOAD_MODEL_STATE | P.OFFLOAD_DEVICE_OPT
    strategies = {"1f1b": ("1f1b", 0), "1f1b_full_recomp": ("1f1b_full_recomp", 0),
                  "1f1b_r50": ("1f1b_full_recomp@r50", 0),
                  "tpipe": ("tpipe", 0), "tpipe_trecomp": ("tpipe_trecomp", 0),
                  "tpipe_all": ("tpipe_trecomp", ms),
                  # ladder rungs without recompute (R28): model-state T-Offload, activation
                  # offload, both
                  "tpipe_offload": ("tpipe", ms), "tpipe_actoff": ("tpipe", P.OFFLOAD_ACTIVATIONS),
                  "tpipe_actoff_offload": ("tpipe", P.OFFLOAD_ACTIVATIONS | ms),
                  "interleave": ("interleave", 0), "interleave_trecomp": ("interleave_trecomp", 0),
                  # v = 3 chunks (R32): T-Recomp of chunk 1 (a third of the stage's layers)
                  # + T-Offload of chunks 2 and 3
                  "tpipe_all_v3": ("tpipe_trecomp@v3", ms), "tpipe_offload_v3": ("tpipe@v3", ms)}
    best = {}
    for name, (strat, off) in strategies.items():
        for L in range(p, 400, p):
            md = P.Model(L, C5["hidden"], C5["n_heads"], C5["ffn_hidden"], C5["vocab"],
                         C5["seq_len"], C5["micro_batch"], P.BF16)
            try:
                plan_of(md, p, m, budget, strat, off)
                best[name] = (L, strat, off)
            except TPipeError:
                # odd chunk splits are invalid for v=2 at small L; a budget
                # failure at L means every larger L fails too
                if L >= 4 * p:
                    break
    return best


def run_capacity(args):
    """Executed capacity at a fixed per-stage HBM budget on ONE B200: all p=8
    pipeline stages of the C5 shape run in one process (virtual pipeline, the
    in-process D2D transport), each stage's pool ledger capped at the budget
    (a plan/ledger bug would raise E_OOM). For every strategy the largest
    model its plan fits is built, stepped, and timed: the pool high-water of
    every stage is read back from the runtime, and model TFLOP/s (causal
    F_tok) is reported next to tokens/s (Q18: a 2x larger model halves
    tokens/s at equal MFU). Also: T-Pipe-ALL at the 1F1B+full-recompute size
    (north star: beat 1F1B+full recompute at equal model size)."""
    import torch
    from paper_2503_03182_b200 import plan as P, runtime as RT
    import synth
    p, m = args.cap_p or CAP_P, CAP_M
    budget_gib = args.cap_budget_gib or CAP_BUDGET_GIB
    budget = int(budget_gib * 2 ** 30)
    best = capacity_plans(p, budget, m)
    names = ("1f1b", "1f1b_full_recomp", "1f1b_r50", "tpipe", "tpipe_trecomp", "tpipe_all", "tpipe_offload",
             "tpipe_actoff", "tpipe_actoff_offload", "interleave", "interleave_trecomp", "tpipe_all_v3",
             "tpipe_offload_v3")
    only = os.environ.get("TPIPE_CAPACITY_ONLY")
    if only:
        names = tuple(n for n in names if n in only.split(",") or n == "1f1b")
    runs = [(n, *best[n]) for n in names if n in best]
    if "1f1b_full_recomp" in best and "tpipe_all" in best:
        runs.append(("tpipe_all@1f1b_full_recomp_size", best["1f1b_full_recomp"][0], *best["tpipe_all"][1:]))
    if "1f1b" in best:
        # north star: a model >= 2x the 1F1B-max params, planned by the auto ladder
        # (T-Pipe -> partial T-Recomp r=1..n1 -> + T-Offload), least recompute that fits
        def params_at(L):
            md = P.Model(L, C5["hidden"], C5["n_heads"], C5["ffn_hidden"], C5["vocab"],
                         C5["seq_len"], C5["micro_batch"], P.BF16)
            return P.Plan(md, p, m, strategy="1f1b").params_total
        target = 2 * params_at(best["1f1b"][0])
        L2 = next(L for L in range(p, 400, p) if params_at(L) >= target)
        runs.append(("auto@2x_1f1b_params", L2, "auto",
                     P.OFFLOAD_MODEL_STATE | P.OFFLOAD_DEVICE_OPT | P.OFFLOAD_ACTIVATIONS))
    pool = (np.random.default_rng(5).standard_normal(1 << 24, dtype=np.float32)
            * np.float32(0.02))
    tok, tgt = synth.tokens(C5["vocab"], m, C5["micro_batch"], C5["seq_len"], step=0)
    dtok = torch.tensor(tok, dtype=torch.int32, device="cuda")
    dtgt = torch.tensor(tgt, dtype=torch.int32, device="cuda")
    tokens = m * C5["micro_batch"] * C5["seq_len"]
    _, _, pk_sust, src = peaks()
    res = {}
    for name, L, strat, off in runs:
        md = P.Model(L, C5["hidden"], C5["n_heads"], C5["ffn_hidden"], C5["vocab"],
                     C5["seq_len"], C5["micro_batch"], P.BF16)
        try:
            plan = plan_of(md, p, m, budget, strat, off)
        except Exception as e:   # e.g. no rung fits the budget at this size
            res[name] = {"n_layers": L, "strategy": strat, "error": str(e)[:160]}
            continue
        t0 = time.perf_counter()
        rt = RT.Runtime(plan, stage=-1, lr=1e-5, pool_cap=budget)
        for s in range(p):
            for ch in range(1, plan.v + 1):
                rt.set_params(s, ch, fast_init_chunk(plan, s, ch, pool))
        setup_s = time.perf_counter() - t0
        free_b, total_b = torch.cuda.mem_get_info()
        ext = torch.cuda.ExternalStream(rt.stream())
        loss0 = rt.step_device(dtok.data_ptr(), dtgt.data_ptr())
        torch.cuda.synchronize()
        k = 2
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        for _ in range(k):
            loss = rt.step_device(dtok.data_ptr(), dtgt.data_ptr())
        e1.record(ext)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        hw = rt.stats()["pool_high_water"]
        fl = model_flops_per_token(dict(n_layers=L, hidden=C5["hidden"], seq_len=C5["seq_len"],
                                        vocab=C5["vocab"]))
        tf = tokens * fl / (ms / 1e3) / 1e12
        res[name] = {"strategy": strat, "offload": plan.offload, "n_layers": L,
                     "plan_strategy": ["1f1b", "1f1b_full_recomp", "tpipe", "tpipe_trecomp", "interleave",
                                       "interleave_trecomp"][plan.strategy],
                     "recomp_layers": plan.recomp_layers, "layers_chunk": list(plan.partition[0]),
                     "chunks": plan.v,
                     "params_B": round(plan.params_total / 1e9, 3),
                     "plan_peak_GiB": [round(plan.peak(s)["total_peak"] / 2 ** 30, 3) for s in range(p)],
                     "pool_high_water_GiB": [round(x / 2 ** 30, 3) for x in hw],
                     "high_water_eq_plan": all(hw[s] == plan.peak(s)["total_peak"] for s in range(p)),
                     "max_stage_GiB": round(max(hw) / 2 ** 30, 3),
                     "fits_budget": max(hw) <= budget, "stages": p, "budget_GiB": budget_gib,
                     "device_used_GiB": round((total_b - free_b) / 2 ** 30, 1),
                     "loss_first": round(float(loss0), 4), "loss_last": round(float(loss), 4),
                     "ms_per_step": round(ms, 1), "tokens_s": round(tokens / (ms / 1e3), 1),
                     "model_tflops": round(tf, 1), "mfu_1gpu": round(tf / pk_sust, 4),
                     "setup_s": round(setup_s, 1)}
        print(json.dumps({name: res[name]}), file=sys.stderr, flush=True)
        rt.close()
        del rt, plan
        torch.cuda.synchronize()
    out = {"capacity_measured": {
        "how": f"one B200, all p={p} stages in one process (virtual pipeline), pool ledger per stage "
               f"capped at {budget_gib} GiB, shape h=4096 a=32 f=16384 V=32000 s=8192 b=1 m={m}, "
               f"largest L (multiple of p) the planner fits, then built and stepped ({src} peak {pk_sust})",
        "runs": res}}
    b = res.get("1f1b")
    if b:
        for n, r in res.items():
            if "error" in r:
                continue
            r["params_vs_1f1b"] = round(r["params_B"] / b["params_B"], 3)
            r["model_tflops_vs_1f1b"] = round(r["model_tflops"] / b["model_tflops"], 3)
    fr, ta = res.get("1f1b_full_recomp"), res.get("tpipe_all@1f1b_full_recomp_size")
    if fr and ta and "tokens_s" in fr and "tokens_s" in ta:
        out["capacity_measured"]["equal_size_tpipe_all_vs_1f1b_full_recomp_tokens_s"] = \
            round(ta["tokens_s"] / fr["tokens_s"], 3)
    return out


def hbm_kernels(c, hbm_peak):
    """HBM-bound stage-executor kernels at the workload's launch shape (M = b*s
    rows): achieved GB/s = algorithmic bytes (each operand read
    once, each result written once) / CUDA-event time of 20 back-to-back
    launches on torch's current stream (the kernels' launch stream), captured
    in one CUDA graph, vs the measured HBM copy peak. Working sets of 8-100 MB partly hit L2 between
    launches, so back-to-back figures are an upper bound on the in-step rate."""
    import torch
    from paper_2503_03182_b200 import kernels as K
    M, h, f, V = c["seq_len"] * c["micro_batch"], c["hidden"], c["ffn_hidden"], c["vocab"]
    dev = "cuda"
    bf = torch.bfloat16

    def tm(fn, iters=20):
        # the launches are captured in a CUDA graph so that the ctypes call
        # overhead (~10 us) does not starve the GPU between launches
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with torch.cuda.graph(gr, stream=side):
                for _ in range(iters):
                    fn()
        torch.cuda.current_stream().wait_stream(side)
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters

    x = torch.randn((M, h), device=dev).to(bf)
    dy = torch.randn((M, h), device=dev).to(bf)
    res = torch.randn((M, h), device=dev).to(bf)
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    g = torch.ones(h, device=dev, dtype=bf)
    b = torch.zeros(h, device=dev, dtype=bf)
    mean = torch.empty(M, device=dev)
    rstd = torch.empty(M, device=dev)
    dg = torch.zeros(h, device=dev)
    db = torch.zeros(h, device=dev)
    drs = torch.zeros(h, device=dev)
    ws = torch.empty(((M + 15) // 16) * max(f, 3 * h), device=dev)
    du = torch.randn((M, f), device=dev).to(bf)
    dbias = torch.zeros(f, device=dev)
    n_p = 1 << 26
    master = torch.randn(n_p, device=dev)
    mm_, vv = torch.zeros(n_p, device=dev), torch.zeros(n_p, device=dev)
    grad = torch.randn(n_p, device=dev)
    w = torch.empty(n_p, device=dev, dtype=bf)
    cases = [
        ("ln_fwd", lambda: K.tpipe_k_ln_fwd(1, x, g, b, y, mean, rstd, M, h), 2 * 2 * M * h + 8 * M),
        ("ln_bwd_rsum", lambda: K.tpipe_k_ln_bwd_rsum(1, dy, x, g, mean, rstd, res, dx, dg, db, drs, ws, M, h),
         4 * 2 * M * h + 8 * M),
        # the layer backward's form: the same kernel, column partials left for the
        # layer's one shared reduce launch (bytes: the partials written, too)
        ("ln_bwd_partials", lambda: K.tpipe_k_ln_bwd_partials(dy, x, g, mean, rstd, res, dx, ws, M, h, 1),
         4 * 2 * M * h + 8 * M + 3 * 4 * ((M + 15) // 16) * h),
        ("colsum_ffn", lambda: K.tpipe_k_colsum(1, du, dbias, ws, M, f), 2 * M * f),
        ("adamw_64M", lambda: K.tpipe_k_adamw(1, master, mm_, vv, grad, w, n_p, 1, 1e-4, 0.9, 0.95, 1e-8,
                                                0.1, 0.1, 0.05), 30 * n_p),
    ]
    out = {}
    for name, fn, nbytes in cases:
        ms = tm(fn)
        gbs = nbytes / (ms / 1e3) / 1e9
        out[name] = {"us": round(ms * 1e3, 2), "alg_bytes": int(nbytes), "GBs": round(gbs, 1),
                     "frac": round(gbs / hbm_peak, 3)}
    return out


def balanced_partition(L, p, v, head_layers):
    """Cost-balanced per-stage layer vector (DESIGN R27, SURVEY D-12): the last
    stage also runs the LM head, worth `head_layers` layers of work (6hV vs
    72h^2 + 6sh FLOPs per token); choose its layer count n_last >= v to
    minimise the largest stage cost, spread the other L - n_last layers as
    evenly as possible (extra layers on the earliest stages)."""
    best = None
    for n_last in range(v, L // p + 1):
        rest = L - n_last
        if rest < v * (p - 1):
            break
        hi = -(-rest // (p - 1)) if p > 1 else 0
        cost = max(hi, n_last + head_layers)
        if best is None or cost < best[0] - 1e-9:
            best = (cost, n_last)
    if p == 1 or best is None:
        return None
    n_last = best[1]
    rest = L - n_last
    base, extra = divmod(rest, p - 1)
    return [base + (1 if s < extra else 0) for s in range(p - 1)] + [n_last]


def modeled_makespan(plan, head_layers):
    """Unit-model makespan of a plan with per-op durations from its layer
    counts (F = layers of the chunk + the LM head's layer-equivalents on the
    last stage's last chunk, B = 2F, R = the recomputed layers), replayed by
    tpipe_plan_simulate_durations."""
    ms = []
    for s in range(plan.p):
        ops, _ = plan.ops(s)
        d = []
        for o in ops:
            if o["kind"] not in ("F", "B", "R"):
                continue
            ch = o["chunk"]
            f = plan.partition[s][ch - 1] + (head_layers if (s == plan.p - 1 and ch == plan.v) else 0.0)
            if o["kind"] == "R":
                f = min(plan.recomp_layers, plan.partition[s][0])
            d.append(2 * f if o["kind"] == "B" else f)
        ms.append(d)
    return plan.simulate_durations(ms)[0]


def pipeline_replay(ps=(8,), strategies=("1f1b", "tpipe", "tpipe_trecomp", "1f1b_full_recomp",
                                         "1f1b_bal", "tpipe_bal", "tpipe_trecomp_bal"), m=None):
    """Measured-duration replay of the p-stage pipeline (SURVEY §8(d) bubble
    fraction, D-12 stage balance): all p stages of the C2 model run on this
    GPU as a virtual pipeline with TPIPE_STEP_OP_TIMES, so every F / B / R op
    is timed on its own (CUDA events on the stage stream); the planner's
    ASAP replay (tpipe_plan_simulate_durations) then schedules those measured
    durations on p GPUs. Stage transport (one [b*s, h] bf16 message per hop,
    8 MiB here, ~10 us over NVLink 5) is not modelled. Returns, per p and
    strategy: predicted ms/step, tokens/s on p GPUs, MFU, per-stage bubble
    fraction and the ratio to 1F1B."""
    import torch
    from paper_2503_03182_b200 import plan as P, runtime as RT
    import synth
    c = C2
    m = m or c["m"]
    pool = (np.random.default_rng(5).standard_normal(1 << 22, dtype=np.float32) * np.float32(0.02))
    tok, tgt = synth.tokens(c["vocab"], m, c["micro_batch"], c["seq_len"], step=0, vocab_eff=c["vocab_eff"])
    dtok = torch.tensor(tok, dtype=torch.int32, device="cuda")
    dtgt = torch.tensor(tgt, dtype=torch.int32, device="cuda")
    tokens = m * c["micro_batch"] * c["seq_len"]
    _, _, pk_sust, _src = peaks()
    out = {}
    for p in ps:
        res = {}
        for st in strategies:
            md = P.Model(c["n_layers"], c["hidden"], c["n_heads"], c["ffn_hidden"], c["vocab"],
                         c["seq_len"], c["micro_batch"], P.BF16)
            # "_bal": the planner's duration-aware partition (R27 / R29, balance);
            # "_v3": three chunks per stage (R32)
            bal, v3 = st.endswith("_bal"), st.endswith("_v3")
            base_st = st[:-4] if bal else (st[:-3] if v3 else st)
            part = None
            try:
                plan = P.Plan(md, p, m, strategy=base_st, balance=bal and p > 1, chunks=3 if v3 else 2)
            except Exception as e:   # e.g. an invalid chunk split
                res[st] = {"error": str(e)[:120]}
                continue
            rt = RT.Runtime(plan, stage=-1, lr=1e-5)
            for s in range(p):
                for ch in range(1, plan.v + 1):
                    rt.set_params(s, ch, fast_init_chunk(plan, s, ch, pool))
            rt.step_device(dtok.data_ptr(), dtgt.data_ptr())
            rt.step_device(dtok.data_ptr(), dtgt.data_ptr(), RT.STEP_OP_TIMES)
            op_ms = [rt.op_times(s) for s in range(p)]
            rt.close()
            mk, busy = plan.simulate_durations(op_ms)
            tps = tokens / (mk / 1e3)
            res[st] = {"partition": [list(x) for x in plan.partition],
                       "ms_per_step": round(mk, 2),
                       "tokens_s": round(tps, 1),
                       "mfu": round(tps * model_flops_per_token(c) / (p * pk_sust * 1e12), 4),
                       "bubble_fraction": [round(1.0 - b / mk, 4) for b in busy[:p]],
                       "compute_ms_per_stage": [round(b, 2) for b in busy[:p]]}
        base = res.get("1f1b", {}).get("tokens_s")
        if base:
            for st, r in res.items():
                if "tokens_s" in r:
                    r["vs_1f1b"] = round(r["tokens_s"] / base, 3)
        out[f"p{p}"] = res
    return out


def gemm_traffic():
    """Per-launch DRAM traffic of the tcgen05 GEMM class from the committed
    `ncu --set full` capture of the 12 layer GEMM shapes (scripts/
    gemm_shapes_once.py): mean dram__bytes_read.sum + dram__bytes_write.sum."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_gemm_ncu_full_v*.jsonl")))
    path = files[-1] if files else ""
    try:
        with open(path) as f:
            for line in f:
                d = json.loads(line)
                if "summary" in d:
                    return int(d["mean_dram_bytes"]), int(d["mean_alg_bytes"])
    except Exception:
        pass
    return None, None


def host_link_peak():
    """Pinned host <-> HBM copy bandwidth (GB/s) for 1 GiB, best of 3 each way."""
    import torch
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        best = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[name + "_GBs"] = round(n / (best / 1e3) / 1e9, 1)
    del h, d
    return out


def measure_offload(N, m, dtok, dtgt, args, base_ms, device_opt=False):
    """T-Offload of the deep chunk's model states on top of T-Recomp at
    N=1: step time, the copy engines' busy time and achieved host-link GB/s,
    the host AdamW time, and the overlap fraction
    1 - (t_offload - t_trecomp) / (D2H + host AdamW + H2D)."""
    import torch
    from paper_2503_03182_b200 import plan as P, runtime as RT
    c = C2
    md = P.Model(c["n_layers"], c["hidden"], c["n_heads"], c["ffn_hidden"], c["vocab"],
                 c["seq_len"], c["micro_batch"], P.BF16)
    off = P.OFFLOAD_MODEL_STATE | (P.OFFLOAD_DEVICE_OPT if device_opt else 0)
    plan = P.Plan(md, N, m, strategy="tpipe_trecomp", offload=off)
    rt = RT.Runtime(plan, stage=-1, lr=1e-4)
    rng = np.random.default_rng(99)
    for s in range(N):
        for ch in range(1, plan.v + 1):
            rt.set_params(s, ch, init_chunk(plan, s, ch, rng))
    ext = torch.cuda.ExternalStream(rt.stream())
    for _ in range(2):
        rt.step_device(dtok.data_ptr(), dtgt.data_ptr())
    torch.cuda.synchronize()
    k = max(2, args.steps // 2)
    tot = 0.0
    st = None
    for _ in range(k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        rt.step_device(dtok.data_ptr(), dtgt.data_ptr())
        e1.record(ext)
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
        st = rt.stats()
    ms = tot / k
    d2h_b, h2d_b = st["offload_d2h_bytes"], st["offload_h2d_bytes"]
    d2h_ms, h2d_ms, host_ms = st["offload_d2h_ms"], st["offload_h2d_ms"], st["host_opt_ms"]
    # host AdamW: grads D2H -> host update -> weights H2D run in series;
    # streamed device AdamW: H2D and D2H slices overlap (full duplex), the longer bounds it
    serial = max(d2h_ms, h2d_ms) if device_opt else d2h_ms + h2d_ms + host_ms
    exposed = max(0.0, ms - base_ms)
    res = {"strategy": "tpipe_trecomp + T-Offload(model states of chunk 2), " +
                       ("streamed device AdamW (R24)" if device_opt else "host AdamW (P:402)"),
           "tokens_s": round(m * c["seq_len"] / (ms / 1e3), 1), "ms_per_step": round(ms, 2),
           "plan_peak_GiB": round(plan.peak(0)["total_peak"] / 2 ** 30, 2),
           "d2h_bytes": int(d2h_b), "h2d_bytes": int(h2d_b),
           "d2h_ms": round(d2h_ms, 2), "h2d_ms": round(h2d_ms, 2),
           "host_adamw_ms": None if device_opt else round(host_ms, 2),
           "d2h_GBs": round(d2h_b / (d2h_ms / 1e3) / 1e9, 1) if d2h_ms else None,
           "h2d_GBs": round(h2d_b / (h2d_ms / 1e3) / 1e9, 1) if h2d_ms else None,
           "exposed_ms": round(exposed, 2),
           "overlap_fraction": round(1.0 - min(1.0, exposed / serial), 3) if serial else None,
           "note": "p=1: the Eq. 5/7 windows 2(p-b-1), (p-a-1) T_unit are empty at one stage, "
                   "so only the copy-engine / host-thread concurrency with the remaining "
                   "backward and next forward hides the offload"}
    rt.close()
    return res


def quick_measure(strategy, N, m, dtok, dtgt, args, recomp_layers=0, offload=0, act_distance=0):
    """tokens/s of another schedule on the same kernels/workload (N=1)."""
    import torch
    from paper_2503_03182_b200 import plan as P, runtime as RT
    c = C2
    md = P.Model(c["n_layers"], c["hidden"], c["n_heads"], c["ffn_hidden"], c["vocab"],
                 c["seq_len"], c["micro_batch"], P.BF16)
    plan = P.Plan(md, N, m, strategy=strategy, recomp_layers=recomp_layers, offload=offload,
                  act_distance=act_distance)
    rt = RT.Runtime(plan, stage=-1, lr=1e-4)
    rng = np.random.default_rng(99)
    for s in range(N):
        for ch in range(1, plan.v + 1):
            rt.set_params(s, ch, init_chunk(plan, s, ch, rng))
    ext = torch.cuda.ExternalStream(rt.stream())
    for _ in range(2):
        rt.step_device(dtok.data_ptr(), dtgt.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = max(2, args.steps // 2)
    e0.record(ext)
    for _ in range(k):
        rt.step_device(dtok.data_ptr(), dtgt.data_ptr())
    e1.record(ext)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    tokens = m * c["micro_batch"] * c["seq_len"]
    st = rt.stats()
    res = {"tokens_s": round(tokens / (ms / 1e3), 1), "ms_per_step": round(ms, 2),
           "steps": k, "plan_peak_GiB": round(plan.peak(0)["total_peak"] / 2 ** 30, 2),
           "pool_high_water_GiB": round(st["pool_high_water"][0] / 2 ** 30, 2)}
    if offload & P.OFFLOAD_ACTIVATIONS:
        d2h_b, h2d_b = st["offload_d2h_bytes"], st["offload_h2d_bytes"]
        res.update({"act_d2h_bytes": int(d2h_b), "act_h2d_bytes": int(h2d_b),
                    "d2h_GBs": round(d2h_b / (st["offload_d2h_ms"] / 1e3) / 1e9, 1) if st["offload_d2h_ms"] else None,
                    "h2d_GBs": round(h2d_b / (st["offload_h2d_ms"] / 1e3) / 1e9, 1) if st["offload_h2d_ms"] else None,
                    "act_distance": plan.act_distance})
    rt.close()
    return res


def latest_capacity_claim():
    """The executed-capacity headline, read from the newest round's committed
    profiles/r<N>_capacity_measured*.json files (so the printed claim cannot go
    stale): the largest executed model and the fastest one >= 2x 1F1B's size,
    each ratio against the 1F1B run of its own file."""
    import glob
    import re
    files = glob.glob(os.path.join(ROOT, "profiles", "r*_capacity_measured*.json"))
    if not files:
        return None
    rnd = max(int(re.findall(r"r(\d+)_", os.path.basename(f))[0]) for f in files)
    runs = []
    for f in sorted(files):
        if int(re.findall(r"r(\d+)_", os.path.basename(f))[0]) != rnd:
            continue
        for r in json.load(open(f))["capacity_measured"]["runs"].values():
            if r.get("fits_budget") and "params_vs_1f1b" in r:
                runs.append((os.path.relpath(f, ROOT), r))
    if not runs:
        return None
    fb, best = max(runs, key=lambda x: x[1]["params_vs_1f1b"])
    s = (f"{fb}: largest executed model {best['params_B']}B params = {best['params_vs_1f1b']}x 1F1B's at "
         f"{best['model_tflops_vs_1f1b']}x its model TFLOP/s ({best['plan_strategy']}, "
         f"chunks={best.get('chunks', 2)}, offload={best.get('offload', 0)})")
    # against the paper's 1F1B + R50 baseline, within one capacity file
    for f in sorted({x[0] for x in runs}):
        r50 = next((r for ff, r in runs if ff == f and r.get("plan_strategy") == "1f1b_full_recomp"
                    and 0 < r.get("recomp_layers", 0) < r.get("n_layers", 0) // r.get("stages", CAP_P)),
                   None)
        if r50:
            big = max((r for ff, r in runs if ff == f), key=lambda r: r["params_B"])
            s += (f"; {f}: vs 1F1B+R50 {round(big['params_B'] / r50['params_B'], 2)}x params at "
                  f"{round(big['model_tflops'] / r50['model_tflops'], 3)}x its model TFLOP/s")
    two = [x for x in runs if x[1]["params_vs_1f1b"] >= 2]
    if two:
        ft, t = max(two, key=lambda x: x[1]["model_tflops_vs_1f1b"])
        s += (f"; {ft}: fastest >= 2x model {t['params_vs_1f1b']}x params at {t['model_tflops_vs_1f1b']}x "
              f"({t['plan_strategy']}, chunks={t.get('chunks', 2)}, offload={t.get('offload', 0)}, "
              f"r={t.get('recomp_layers', 0)})")
    return s


def launch_ranks(args):
    """`bench.py --gpus N` outside torchrun: start N ranks (one process per GPU)
    with torch.distributed.run and relay rank 0's line; refuse when the box has
    fewer than N GPUs (a one-GPU virtual pipeline is --virtual-stages, and is
    labelled n_gpus = 1)."""
    import subprocess
    import torch
    n_dev = torch.cuda.device_count()
    if n_dev < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this box has {n_dev} "
              f"(use --virtual-stages {args.gpus} for a one-GPU virtual pipeline)", file=sys.stderr)
        sys.exit(2)
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def run_tpipe(args):
    import torch
    from paper_2503_03182_b200 import plan as P, runtime as RT
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1 and args.virtual_stages:
        raise SystemExit("bench.py: --virtual-stages is a one-process option")
    # p pipeline stages: one per rank (N > 1; with --pp P < N the other ranks are
    # dp = N / P data-parallel replicas, ZeRO-1, R31), or a one-GPU virtual pipeline
    pp = args.pp or world
    if world > 1 and (world % pp or (world // pp > 1 and args.transport != "ipc")):
        raise SystemExit(f"bench.py: --pp {pp} must divide {world} ranks; dp > 1 needs --transport ipc")
    dp = world // pp if world > 1 else 1
    N = pp if world > 1 else (args.virtual_stages or 1)
    stage = rank % N if world > 1 else -1
    dp_rank = rank // N if world > 1 else 0
    n_gpus = world
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    # test hook: every rank on GPU 0 (exercises the N-rank path on a one-GPU
    # box; the number is NOT an N-GPU measurement and the line says so)
    same_gpu = os.environ.get("TPIPE_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    c = C2
    md = P.Model(c["n_layers"], c["hidden"], c["n_heads"], c["ffn_hidden"], c["vocab"],
                 c["seq_len"], c["micro_batch"], P.BF16)
    m = c["m"]
    # p > 1: the planner picks the cost-balanced stage partition when its cost
    # model says it pays (R27/R28)
    plan = P.Plan(md, N, m, strategy=args.strategy, balance=N > 1, dp=dp)
    transport = RT.TRANSPORT_IPC if args.transport == "ipc" else RT.TRANSPORT_NCCL

    def make_runtime(tr):
        ids, ipc_name = None, None
        if world > 1:
            if tr == RT.TRANSPORT_NCCL:
                ids = [b"".join(RT.nccl_unique_id() for _ in plan.channels)] if rank == 0 else [None]
            else:
                ids = [f"/tpipe_bench_{os.getpid()}_{np.random.default_rng().integers(1 << 40)}"] \
                    if rank == 0 else [None]
            dist.broadcast_object_list(ids, src=0)
            ids, ipc_name = (ids[0], None) if tr == RT.TRANSPORT_NCCL else (None, ids[0])
        return RT.Runtime(plan, stage=stage, device=local, nccl_ids=ids, lr=1e-4, transport=tr,
                          ipc_name=ipc_name, dp_rank=dp_rank, timeout_ms=120000)

    if world > 1 and transport == RT.TRANSPORT_IPC and dp == 1:
        # CUDA IPC first; if any rank cannot set it up (no peer access, shm
        # unavailable), every rank falls back to NCCL together
        rt, err = None, ""
        try:
            rt = make_runtime(RT.TRANSPORT_IPC)
        except Exception as e:   # reported in the line, not fatal
            err = str(e)[:200]
        ok = torch.tensor([1 if rt is not None else 0])
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok[0]) == 0:
            if rt is not None:
                rt.close()
            rt = make_runtime(RT.TRANSPORT_NCCL)
            args.transport = f"nccl (ipc setup failed: {err or 'on another rank'})"
    else:
        rt = make_runtime(transport)
    rng = np.random.default_rng(1234 + max(stage, 0))   # replicas of a stage start equal
    stages = [stage] if world > 1 else list(range(N))
    for s in stages:
        for ch in range(1, plan.v + 1):
            rt.set_params(s, ch, init_chunk(plan, s, ch, rng))
    import synth
    tok, tgt = synth.tokens(c["vocab"], m, c["micro_batch"], c["seq_len"], step=dp_rank,
                            vocab_eff=c["vocab_eff"])   # each replica its own micro-batches
    dtok = torch.tensor(tok, dtype=torch.int32, device="cuda")
    dtgt = torch.tensor(tgt, dtype=torch.int32, device="cuda")
    ext = torch.cuda.ExternalStream(rt.stream())

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def timed(fn, k):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        for _ in range(k):
            fn()
        e1.record(ext)
        barrier()
        ms = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms])
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t[0])
        return ms

    # CUDA-graph steps (TPIPE_STEP_GRAPH: captured in the first warm-up step,
    # replayed after) where the plan allows it: one process, no T-Offload, no DP
    gf = RT.STEP_GRAPH if (args.graph and world == 1 and dp == 1 and not plan.offload) else 0
    for _ in range(args.warmup):
        rt.step_device(dtok.data_ptr(), dtgt.data_ptr(), gf)
    with Clocks(local) as clk:
        ms = timed(lambda: rt.step_device(dtok.data_ptr(), dtgt.data_ptr(), gf), args.steps)
    launches = rt.stats()["kernel_launches"]
    # e2e: host tokens (pinned) -> tpipe_step (H2D inside) -> loss D2H
    htok = torch.from_numpy(tok).pin_memory().numpy()
    htgt = torch.from_numpy(tgt).pin_memory().numpy()
    ms_e2e = timed(lambda: rt.step(htok, htgt, gf), args.steps)
    # profiled pass of the same K steps: per-kernel-class CUDA-event timing
    kms = np.zeros(4)
    kfl = np.zeros(4)
    kcnt = np.zeros(4)
    for _ in range(args.steps):
        rt.step_device(dtok.data_ptr(), dtgt.data_ptr(), RT.STEP_PROFILE)
        st = rt.stats()
        kms += st["kernel_ms"]
        kfl += st["kernel_flops"]
        kcnt += st["kernel_count"]
    hw = rt.stats()["pool_high_water"]
    tokens = dp * m * c["micro_batch"] * c["seq_len"]   # all replicas
    value = tokens * args.steps / (ms / 1e3)
    e2e = tokens * args.steps / (ms_e2e / 1e3)
    hbm, pk_burst, pk_sust, src = peaks()
    gemm_tf = kfl[0] / (kms[0] / 1e3) / 1e12 if kms[0] else None
    # executed FLOPs per step: every GEMM launch (incl. recompute), attention
    # forward, and attention backward at 7 of its 5 algorithmic GEMMs (S and dP
    # are recomputed in both the dK/dV and the dQ kernel)
    hw_flops = (kfl[0] + kfl[1] + kfl[2] * 7.0 / 5.0) / args.steps
    mk, busy = plan.simulate()   # unit-model replay of this plan (F=1, B=2, R=1 T_unit)
    bubble = [round(1.0 - b / mk, 4) for b in busy[:N]] if mk else None
    traffic, alg_bytes = gemm_traffic()
    step_ms = ms / args.steps
    prof_step_ms = None
    out = None
    if rank == 0:
        mfu = value * model_flops_per_token(c) / (n_gpus * pk_sust * 1e12)
        out = {
            "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": n_gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 3),
            "higher_is_better": True, "scaling": "strong" if dp == 1 else "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic (seeded uniform tokens < 50257; random-init weights)",
            "config": {"workload": "configs[1]: GPT-3 1.3B, seq 2048, T-Pipe, m=32 micro-batches",
                       "model": "gpt3-1.3b", "n_layers": 24, "hidden": 2048, "seq_len": 2048,
                       "micro_batch": 1, "n_microbatches": m, "global_batch_tokens": tokens,
                       "pp": N, "dp": dp,
                       "strategy": args.strategy,
                       "parallelism": (f"pp{N}" if dp == 1 else f"dp{dp}xpp{N} (ZeRO-1)") if world > 1 else
                       (f"virtual pp{N} on 1 GPU" if N > 1 else "pp1"),
                       "transport": (args.transport if world > 1 else "in-process"),
                       "step_issue": ("CUDA graph replay (TPIPE_STEP_GRAPH; captured in warm-up)" if gf
                                      else "instruction stream issued per step"),
                       **({"same_gpu_test": "all ranks on GPU 0 (TPIPE_BENCH_SAME_GPU): "
                                            "not an N-GPU measurement"} if same_gpu else {}),
                       "layers_per_chunk": list(plan.layers_chunk),
                       "stage_layers": [sum(x) for x in plan.partition],
                       "l2": "working set >> 126 MB L2 (no flush needed)"},
            "mfu": round(mfu, 4),
            "hfu": round(hw_flops / (step_ms / 1e3) / (n_gpus * pk_sust * 1e12), 4),
            "mfu_peak": f"{pk_sust} TFLOP/s bf16 sustained ({src})",
            "bubble_fraction_unit_model": bubble,
            "gpu_launches": int(launches) * args.steps,
            "pool_high_water_bytes": hw,
            "e2e": {"value": round(e2e, 1), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(2 * tok.nbytes), "d2h_bytes_per_step": 4 * m},
            "roofline": {"bound": "tensor", "kernel": "tcgen05 GEMMs (all K1/K2/K8 launches)",
                         "achieved": round(gemm_tf, 1) if gemm_tf else None, "peak": pk_sust,
                         "unit": "TFLOP/s",
                         "frac": round(gemm_tf / pk_sust, 4) if gemm_tf else None,
                         "traffic": traffic, "traffic_alg_bytes": alg_bytes,
                         "traffic_src": "newest profiles/r*_gemm_ncu_full_v*.jsonl: mean DRAM bytes per "
                                        "launch over the 12 layer GEMM shapes (ncu --set full)",
                         "peak_src": f"bf16_tflops_sustained ({src})",
                         "launches_per_step": int(kcnt[0] / args.steps),
                         "share_of_step": round(kms[0] / args.steps / step_ms, 3)},
            "kernel_classes": {
                "gemm": {"ms_per_step": round(kms[0] / args.steps, 2), "tflops": round(gemm_tf, 1) if gemm_tf else None},
                "attn_fwd": {"ms_per_step": round(kms[1] / args.steps, 2),
                             "tflops": round(kfl[1] / (kms[1] / 1e3) / 1e12, 1) if kms[1] else None},
                "attn_bwd": {"ms_per_step": round(kms[2] / args.steps, 2),
                             "tflops": round(kfl[2] / (kms[2] / 1e3) / 1e12, 1) if kms[2] else None},
                "other": {"ms_per_step": round(kms[3] / args.steps, 2),
                          "launches_per_step": int(kcnt[3] / args.steps)},
                "idle_ms_per_step": round(step_ms - kms.sum() / args.steps, 2)},
            "clocks": clk.summary(),
        }
    rt.close()
    del rt
    if rank == 0 and not args.no_extras and world == 1:
        # in-build baselines on the same kernels (north star): same model,
        # tokens and step; plan peak HBM per stage from the byte model
        comp = {args.strategy: {"tokens_s": round(value, 1),
                                "plan_peak_GiB": round(plan.peak(0)["total_peak"] / 2 ** 30, 2)}}
        for st in ("1f1b", "1f1b_full_recomp", "tpipe_trecomp", "tpipe"):
            if st in comp:
                continue
            comp[st] = quick_measure(st, N, m, dtok, dtgt, args)
        # the paper's 1F1B + R50 baseline (R33): half of each stage's layers
        # recomputed layer-wise in the backward
        comp["1f1b_r50"] = quick_measure("1f1b_full_recomp", N, m, dtok, dtgt, args,
                                         recomp_layers=max(1, c["n_layers"] // max(N, 1) // 2))
        # partial T-Recomp (R25): half of chunk 1's layers regenerated
        r_half = max(1, plan.layers_chunk[0] // 2)
        comp[f"tpipe_trecomp_r{r_half}"] = quick_measure("tpipe_trecomp", N, m, dtok, dtgt, args,
                                                          recomp_layers=r_half)
        # a7: chunk-1 activation offload instead of recompute (R23; bandwidth-bound)
        try:
            # at p = 1 the F(1,i) -> B(1,i) distance is 4 ops: distance 1 offloads every block
            comp["tpipe_act_offload"] = quick_measure("tpipe", N, m, dtok, dtgt, args,
                                                      offload=P.OFFLOAD_ACTIVATIONS,
                                                      act_distance=1 if N == 1 else 0)
        except Exception as e:   # reported, not fatal
            comp["tpipe_act_offload"] = {"error": str(e)[:200]}
        out["compare"] = comp
        for key, dev in (("tpipe_trecomp_offload", False), ("tpipe_trecomp_offload_devopt", True)):
            try:
                comp[key] = measure_offload(N, m, dtok, dtgt, args, comp["tpipe_trecomp"]["ms_per_step"],
                                            device_opt=dev)
            except Exception as e:   # reported, not fatal
                comp[key] = {"error": str(e)[:200]}
        out["host_link_peak"] = host_link_peak()
        try:
            out["pipeline_replay"] = {
                "how": "C2 on one GPU as a p-stage virtual pipeline, every F/B/R op timed with CUDA events "
                       "(TPIPE_STEP_OP_TIMES), measured durations replayed ASAP on p GPUs by "
                       "tpipe_plan_simulate_durations; stage transport not modelled (prediction, not a "
                       "multi-GPU measurement)", **pipeline_replay((8,))}
        except Exception as e:   # reported, not fatal
            out["pipeline_replay"] = {"error": str(e)[:200]}
        out["hbm_kernels"] = {"peak_GBs": hbm, "peak_src": f"hbm_gbs ({src})",
                              "shape": f"M={c['seq_len'] * c['micro_batch']} rows, h={c['hidden']}, "
                                       f"f={c['ffn_hidden']}; adamw 64M params",
                              **hbm_kernels(c, hbm)}
        out["capacity_80GiB"] = {"p": max(N, 8) if N == 1 else N, "shape": "h=4096 a=32 s=8192 V=32000 b=1 m=32",
                                 **capacity(max(N, 8) if N == 1 else N)}
        out["cpu_baseline"] = cpu_baseline(c)
        out["paper_context"] = {
            "note": "the paper's own figures, other hardware (64 BirenTech GPUs, PP8xTP8, 32 GB HBM each, "
                    "P:443, P:471); context, not targets",
            "max_size_vs_1f1b": 2.4, "max_size_vs_1f1b_r50": 1.5,
            "tpipe_all_throughput_vs_1f1b_r50": 0.9758,
            "this_build": "capacity_80GiB (planner, p=8) and bench.py --capacity-run (executed; "
                          + str(latest_capacity_claim()) + ")"}
    if dist:
        dist.barrier()
    return out


def run_reference(args):
    """Reference arm: the oracle (oracle/model.py) as it stands, on host
    cores, same metric/config; each step = a bounded sample (one micro-batch
    fwd+bwd of one layer), reported as model tokens/s."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    from oracle import model as R
    import synth
    c = C2
    h, f, s, a = c["hidden"], c["ffn_hidden"], c["seq_len"], c["n_heads"]
    W = synth.weights(1, h, f, 64, s, seed=1)
    L = R.to64(W)["layers"][0]
    rng = np.random.default_rng(0)
    x = rng.standard_normal((1, s, h))
    dy = rng.standard_normal((1, s, h))

    def step():
        y, cache = R.layer_fwd(x, L, a)
        R.layer_bwd(dy, cache, L, a)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = s * args.steps / dt / c["n_layers"]
    cores = len(os.sched_getaffinity(0))
    sample = (f"per step: 1 micro-batch fwd+bwd of 1 of {c['n_layers']} layers "
              f"(h={h}, s={s}, fp64 NumPy), scaled /L to model tokens/s")
    return {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "tokens/s",
            "n_gpus": max(args.gpus, world), "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt / args.steps * 1e3, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "configs[1]: GPT-3 1.3B, seq 2048",
                                            "model": "gpt3-1.3b", "seq_len": s},
            "cpu_baseline": {"value": round(value, 3), "unit": "tokens/s", "cores": cores,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": round(value, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tpipe", choices=["tpipe", "reference"])
    ap.add_argument("--strategy", default="tpipe", choices=["tpipe", "tpipe_trecomp", "1f1b"])
    ap.add_argument("--no-extras", action="store_true", help="skip capacity sweep and CPU oracle")
    ap.add_argument("--graph", type=int, default=1,
                    help="1: time steps as CUDA-graph replays (TPIPE_STEP_GRAPH) where the plan allows it")
    ap.add_argument("--pipeline-replay", action="store_true",
                    help="measured-op-duration replay of p = 2, 4, 8 stage pipelines (C2)")
    ap.add_argument("--capacity-run", action="store_true",
                    help="executed capacity at a fixed per-stage HBM budget (p=8 virtual pipeline, one GPU)")
    ap.add_argument("--cap-p", type=int, default=0, help="--capacity-run stages (default 8)")
    ap.add_argument("--cap-budget-gib", type=float, default=0, help="--capacity-run per-stage budget (default 20)")
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl"],
                    help="stage transport for N > 1 ranks (CUDA-IPC copy-engine pull, or NCCL send/recv)")
    ap.add_argument("--pp", type=int, default=0,
                    help="pipeline stages when N > 1 (default N); the N / pp replicas are ZeRO-1 data "
                         "parallel (SURVEY NEXT-3)")
    ap.add_argument("--virtual-stages", type=int, default=0,
                    help="run a p-stage virtual pipeline on this one GPU (reported as n_gpus = 1)")
    ap.add_argument("--workload", default="", choices=["", "c3", "c4"],
                    help="throughput at the C3 / C4 model shapes on one GPU (p = 1, auto ladder)")
    ap.add_argument("--oracle-timing", action="store_true",
                    help="fp64 oracle per-layer timing at the C3 / C4 layer shapes (host cores)")
    args = ap.parse_args()
    if args.workload:
        print(json.dumps(run_workload(args)), flush=True)
        return
    if args.oracle_timing:
        print(json.dumps({"oracle_layer_timing": oracle_layer_timing()}), flush=True)
        return
    if args.capacity_run:
        print(json.dumps(run_capacity(args)), flush=True)
        return
    if args.pipeline_replay:
        print(json.dumps({"pipeline_replay": pipeline_replay((2, 4, 8), ("1f1b", "tpipe", "tpipe_trecomp",
                                                                        "1f1b_full_recomp",
                                                                        "interleave",
                                                                        "interleave_trecomp",
                                                                        "1f1b_bal", "tpipe_bal",
                                                                        "tpipe_trecomp_bal",
                                                                        "interleave_bal", "tpipe_v3",
                                                                        "tpipe_trecomp_v3"))}),
              flush=True)
        return
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "tpipe" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        launch_ranks(args)
    out = run_reference(args) if args.impl == "reference" else run_tpipe(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
