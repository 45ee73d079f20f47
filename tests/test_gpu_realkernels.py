"""Parity and bit-exactness where the production kernels run.

* p = 8 virtual pipeline (C1 width, L = 16): fp32 against the fp64 oracle
  (max-rel <= 1e-4) and bf16 (rel-L2 <= 2e-2) for every strategy, including
  T-Recomp with k = 1 delay round (App. B; SURVEY D-3), model-state
  T-Offload at p = 8 and Interleave-1F1B.
* head_dim 128 with production tiles: C_MID (h = 256, a = 2, d = 128) and
  the 2-layer GPT-3 1.3B shape (h = 2048, a = 16, s = 2048, V = 50304) route
  attention to the tcgen05 kernels (fa5::*) and GEMMs to the CTA-pair
  tcgen05 kernels. T-Recomp (full and partial), T-Offload (host and streamed
  device AdamW), activation offload and Interleave-1F1B give gradients and
  updated parameters bit-identical to T-Pipe (BASELINE north_star, R21).
* pool canaries (TPIPE_DEBUG_POOL_CANARY): no kernel writes past the bytes
  the plan gave its buffer, on C1 and C_MID for every strategy; the
  self-test proves the check fires.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from oracle import model as R  # noqa: E402

C1_16 = dict(L=16, h=64, a=4, f=256, V=256, s=32, b=2)
C_MID8 = dict(L=8, h=256, a=2, f=1024, V=512, s=256, b=1)
G13 = dict(L=2, h=2048, a=16, f=8192, V=50304, s=2048, b=1)


def mods():
    from paper_2503_03182_b200 import params, plan, runtime
    return plan, runtime, params


def build(cfg, p, m, strategy, dtype, offload=0, recomp_layers=0, seed=11, debug_flags=0,
          std=0.05):
    P, RT, PR = mods()
    md = P.Model(cfg["L"], cfg["h"], cfg["a"], cfg["f"], cfg["V"], cfg["s"], cfg["b"], dtype)
    # activation offload: distance 1 so that these small shapes really offload
    # (the bandwidth-derived distance, Q12, would keep every block on the device)
    ad = 1 if offload & P.OFFLOAD_ACTIVATIONS else 0
    plan = P.Plan(md, p, m, strategy=strategy, offload=offload, recomp_layers=recomp_layers,
                  act_distance=ad)
    rt = RT.Runtime(plan, stage=-1, lr=1e-3, debug_flags=debug_flags)
    W = synth.weights(cfg["L"], cfg["h"], cfg["f"], cfg["V"], cfg["s"], seed=seed, std=std,
                      bias_std=0.02, ln_jitter=0.05)
    for s in range(p):
        for c in range(1, plan.v + 1):
            rt.set_params(s, c, PR.pack(W, p, plan.v, plan.partition, s, c))
    return plan, rt, W


def max_rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / (np.abs(b).max() + 1e-30))


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))


P8_STRATS = [("tpipe", 0), ("tpipe_trecomp", 0), ("tpipe", 1), ("tpipe_trecomp", 5),
             ("1f1b", 0), ("1f1b_full_recomp", 0), ("interleave", 0), ("interleave_trecomp", 0)]


@pytest.mark.parametrize("strategy,offload", P8_STRATS)
@pytest.mark.parametrize("dtype", [0, 1])
def test_p8_parity(strategy, offload, dtype):
    _P, RT, PR = mods()
    p, m, cfg = 8, 16, C1_16
    plan, rt, W = build(cfg, p, m, strategy, dtype, offload)
    if strategy == "tpipe_trecomp":
        assert plan.k == 1
    tok, tgt = synth.tokens(cfg["V"], m, cfg["b"], cfg["s"], step=0)
    loss = rt.step(tok, tgt, RT.STEP_NO_OPT)
    lref, G = R.step_grads(R.to64(W), tok, tgt, cfg["a"])
    tol, metric = (1e-4, max_rel) if dtype == 0 else (2e-2, rel_l2)
    assert abs(loss - lref) / abs(lref) < (1e-5 if dtype == 0 else 2e-2)
    for s in range(p):
        for c in range(1, plan.v + 1):
            got = PR.unpack(rt.get_grads(s, c), W, p, plan.v, plan.partition, s, c)
            for (k, l), g in got.items():
                ref = G["layers"][l][k] if l is not None else G[k]
                assert metric(g, ref) <= tol, (s, c, k, l)
    st = rt.stats()
    for s in range(p):
        assert st["pool_high_water"][s] == plan.peak(s)["total_peak"]
    rt.close()


def _run(cfg, p, m, strategy, offload=0, recomp_layers=0, steps=2, std=0.05):
    """bf16: step-0 loss and gradients (no optimizer), then `steps` optimizer
    steps from the same initial parameters; returns everything as raw bits."""
    _P, RT, _PR = mods()
    plan, rt, W = build(cfg, p, m, strategy, 1, offload, recomp_layers, std=std)
    tok, tgt = synth.tokens(cfg["V"], m, cfg["b"], cfg["s"], step=0,
                            vocab_eff=50257 if cfg["V"] == 50304 else None)
    loss0 = rt.step(tok, tgt, RT.STEP_NO_OPT)
    grads = [rt.get_grads(s, c).view(np.uint32).copy() for s in range(p) for c in range(1, plan.v + 1)]
    from paper_2503_03182_b200 import params as PR
    for s in range(p):
        for c in range(1, plan.v + 1):
            rt.set_params(s, c, PR.pack(W, p, plan.v, plan.partition, s, c))
    losses = []
    for k in range(steps):
        tok, tgt = synth.tokens(cfg["V"], m, cfg["b"], cfg["s"], step=k,
                                vocab_eff=50257 if cfg["V"] == 50304 else None)
        losses.append(rt.step(tok, tgt, 0))
    params = [rt.get_params(s, c).view(np.uint32).copy() for s in range(p) for c in range(1, plan.v + 1)]
    rt.close()
    return loss0, grads, losses, params


def _assert_same(a, b, what):
    assert a[0] == b[0], (what, "loss", a[0], b[0])
    for x, y in zip(a[1], b[1]):
        assert np.array_equal(x, y), (what, "grads")
    assert a[2] == b[2], (what, "losses")
    for x, y in zip(a[3], b[3]):
        assert np.array_equal(x, y), (what, "params")


CMID_VARIANTS = [("tpipe_trecomp", 0, 0), ("tpipe_trecomp", 0, 1), ("tpipe", 1, 0),
                 ("tpipe", 5, 0), ("tpipe_trecomp", 5, 1), ("tpipe", 2, 0),
                 ("interleave", 0, 0), ("interleave_trecomp", 0, 0)]


@pytest.mark.parametrize("p", [1, 2])
def test_cmid_d128_bitexact_vs_tpipe(p):
    """C_MID (d = 128 -> fa5 tcgen05 attention; tcgen05 GEMMs): every
    recompute / offload variant reproduces T-Pipe bit for bit."""
    m = 4
    ref = _run(C_MID8, p, m, "tpipe")
    for strategy, offload, r in CMID_VARIANTS:
        if p == 1 and strategy.startswith("interleave"):
            continue
        _assert_same(ref, _run(C_MID8, p, m, strategy, offload, r), (strategy, offload, r))


@pytest.mark.parametrize("strategy,offload", [("tpipe_trecomp", 0), ("tpipe", 1), ("tpipe", 5),
                                              ("tpipe", 2)])
def test_gpt13b_shape_bitexact_vs_tpipe(strategy, offload):
    """The bench's layer / vocabulary shape (2 layers of GPT-3 1.3B, p = 1,
    m = 2): CTA-pair GEMMs, fa5 attention at s = 2048."""
    ref = _run(G13, 1, 2, "tpipe", steps=1, std=0.02)
    _assert_same(ref, _run(G13, 1, 2, strategy, offload, steps=1, std=0.02), (strategy, offload))


@pytest.mark.parametrize("cfg,p,m", [(C1_16, 4, 8), (C_MID8, 2, 4)])
@pytest.mark.parametrize("strategy,offload", [("tpipe", 0), ("tpipe_trecomp", 0), ("tpipe", 2),
                                              ("tpipe_trecomp", 5), ("1f1b_full_recomp", 0),
                                              ("interleave_trecomp", 0)])
def test_pool_canaries_clean(cfg, p, m, strategy, offload):
    _P, RT, _PR = mods()
    plan, rt, W = build(cfg, p, m, strategy, 1, offload, debug_flags=RT.DEBUG_POOL_CANARY)
    tok, tgt = synth.tokens(cfg["V"], m, cfg["b"], cfg["s"], step=0)
    rt.step(tok, tgt, 0)
    rt.close()


def test_pool_canary_selftest_fires():
    _P, RT, _PR = mods()
    from paper_2503_03182_b200._lib import TPipeError
    plan, rt, W = build(C1_16, 4, 8, "tpipe", 1,
                        debug_flags=RT.DEBUG_POOL_CANARY | RT.DEBUG_POOL_CANARY_SELFTEST)
    tok, tgt = synth.tokens(C1_16["V"], 8, C1_16["b"], C1_16["s"], step=0)
    with pytest.raises(TPipeError, match="pool canary"):
        rt.step(tok, tgt, 0)
    rt.close()


@pytest.mark.parametrize("strategy", ["tpipe", "tpipe_trecomp"])
def test_duration_aware_partition_step(strategy):
    """R29 (NEXT-5): per-stage layer counts and chunk splits chosen freely —
    fp32 gradients match the oracle, bf16 gradients are bit-identical to the
    uniform partition's (the layer math does not depend on where chunk
    boundaries fall), and the ledger high-water equals the plan peak."""
    P, RT, PR = mods()
    cfg, p, m = C1_16, 4, 8
    part, ch1 = (5, 4, 4, 3), (4, 1, 2, 2)
    tok, tgt = synth.tokens(cfg["V"], m, cfg["b"], cfg["s"], step=1)
    W = synth.weights(cfg["L"], cfg["h"], cfg["f"], cfg["V"], cfg["s"], seed=11, std=0.05,
                      bias_std=0.02, ln_jitter=0.05)
    lref, G = R.step_grads(R.to64(W), tok, tgt, cfg["a"])
    grads = []
    for dtype, sl, c1 in ((0, part, ch1), (1, part, ch1), (1, None, None)):
        md = P.Model(cfg["L"], cfg["h"], cfg["a"], cfg["f"], cfg["V"], cfg["s"], cfg["b"], dtype)
        plan = P.Plan(md, p, m, strategy=strategy, stage_layers=sl, stage_chunk1=c1)
        rt = RT.Runtime(plan, stage=-1)
        for s in range(p):
            for c in (1, 2):
                rt.set_params(s, c, PR.pack(W, p, 2, plan.partition, s, c))
        rt.step(tok, tgt, RT.STEP_NO_OPT)
        g = {}
        for s in range(p):
            for c in (1, 2):
                g.update(PR.unpack(rt.get_grads(s, c), W, p, 2, plan.partition, s, c))
        st = rt.stats()
        assert all(st["pool_high_water"][s] == plan.peak(s)["total_peak"] for s in range(p))
        rt.close()
        if dtype == 0:
            for (k, l), v in g.items():
                ref = G["layers"][l][k] if l is not None else G[k]
                assert max_rel(v, ref) <= 1e-4, (k, l)
        else:
            grads.append(g)
    for k in grads[0]:
        assert np.array_equal(np.asarray(grads[0][k], np.float32).view(np.uint32),
                              np.asarray(grads[1][k], np.float32).view(np.uint32)), k


MC_CASES = [("tpipe", 0), ("tpipe_trecomp", 0), ("interleave_trecomp", 0), ("tpipe", 1), ("tpipe_trecomp", 5)]


@pytest.mark.parametrize("v", [3, 4])
@pytest.mark.parametrize("strategy,offload", MC_CASES)
def test_multichunk_parity(v, strategy, offload):
    """v = 3, 4 chunks per stage (NEXT-4 / NEXT-1, DESIGN R32): fp32 gradients
    and loss vs the oracle; after two optimizer steps (multi-chunk T-Offload
    of chunks 2..v with the host or streamed device AdamW) the bf16
    parameters are bit-identical to the same model at v = 2 (per-layer math
    and per-chunk accumulation order do not depend on the chunking)."""
    P, RT, PR = mods()
    cfg = dict(C1_16, L=4 * v)
    p, m = 2, 4
    W = synth.weights(cfg["L"], cfg["h"], cfg["f"], cfg["V"], cfg["s"], seed=11, std=0.05,
                      bias_std=0.02, ln_jitter=0.05)
    tok, tgt = synth.tokens(cfg["V"], m, cfg["b"], cfg["s"], step=0)
    lref, G = R.step_grads(R.to64(W), tok, tgt, cfg["a"])
    md = P.Model(cfg["L"], cfg["h"], cfg["a"], cfg["f"], cfg["V"], cfg["s"], cfg["b"], 0)
    plan = P.Plan(md, p, m, strategy=strategy, offload=offload, chunks=v)
    rt = RT.Runtime(plan, stage=-1, lr=1e-3)
    for s in range(p):
        for c in range(1, v + 1):
            rt.set_params(s, c, PR.pack(W, p, v, plan.partition, s, c))
    loss = rt.step(tok, tgt, RT.STEP_NO_OPT)
    assert abs(loss - lref) / abs(lref) < 1e-5
    for s in range(p):
        for c in range(1, v + 1):
            for (k, l), g in PR.unpack(rt.get_grads(s, c), W, p, v, plan.partition, s, c).items():
                ref = G["layers"][l][k] if l is not None else G[k]
                assert max_rel(g, ref) <= 1e-4, (s, c, k, l)
    st = rt.stats()
    assert all(st["pool_high_water"][s] == plan.peak(s)["total_peak"] for s in range(p))
    rt.close()
    params = []
    for vv in (v, 2):
        md = P.Model(cfg["L"], cfg["h"], cfg["a"], cfg["f"], cfg["V"], cfg["s"], cfg["b"], 1)
        plan = P.Plan(md, p, m, strategy=strategy, offload=offload, chunks=vv)
        rt = RT.Runtime(plan, stage=-1, lr=1e-3)
        for s in range(p):
            for c in range(1, vv + 1):
                rt.set_params(s, c, PR.pack(W, p, vv, plan.partition, s, c))
        for k in range(2):
            t2, g2 = synth.tokens(cfg["V"], m, cfg["b"], cfg["s"], step=k)
            rt.step(t2, g2, 0)
        d = {}
        for s in range(p):
            for c in range(1, vv + 1):
                d.update(PR.unpack(rt.get_params(s, c), W, p, vv, plan.partition, s, c))
        params.append(d)
        rt.close()
    for key in params[0]:
        assert np.array_equal(np.asarray(params[0][key], np.float32).view(np.uint32),
                              np.asarray(params[1][key], np.float32).view(np.uint32)), key


@pytest.mark.parametrize("strategy,offload,p", [("tpipe", 0, 4), ("tpipe_trecomp", 5, 4), ("tpipe", 2, 2),
                                                ("1f1b_full_recomp", 0, 4), ("interleave_trecomp", 0, 8)])
def test_planned_arena_close_to_peak(strategy, offload, p):
    """The pool lays out every buffer of the plan once (fixed lifetimes):
    the physical arena stays within a few percent of the plan peak (the
    ledger high-water equals the peak exactly), and steps reuse it without
    any run-time placement."""
    _P, RT, _PR = mods()
    cfg = C1_16 if p == 8 else C_MID8
    plan, rt, W = build(cfg, p, 2 * p, strategy, 1, offload)
    tok, tgt = synth.tokens(cfg["V"], 2 * p, cfg["b"], cfg["s"], step=0)
    for _ in range(2):
        rt.step(tok, tgt, 0)
    st = rt.stats()
    peak = sum(plan.peak(s)["total_peak"] for s in range(p))
    assert all(st["pool_high_water"][s] == plan.peak(s)["total_peak"] for s in range(p))
    assert st["pool_overflow_bytes"] == 0
    assert peak <= st["pool_reserved"] <= 1.12 * peak + p * (1 << 20), (st["pool_reserved"], peak)
    rt.close()


@pytest.mark.parametrize("r", [1, 2])
def test_1f1b_partial_recompute_step(r):
    """1F1B + layer-grouped recompute of r of the stage's layers (r = 2 of 4:
    1F1B + R50; DESIGN R33): fp32 gradients vs the oracle; bf16
    gradients and updated parameters bit-identical to plain 1F1B (the
    recomputed layers regenerate the same values with the same kernels)."""
    P, RT, PR = mods()
    cfg, p, m = dict(C1_16, L=8), 2, 4
    W = synth.weights(cfg["L"], cfg["h"], cfg["f"], cfg["V"], cfg["s"], seed=11, std=0.05,
                      bias_std=0.02, ln_jitter=0.05)
    tok, tgt = synth.tokens(cfg["V"], m, cfg["b"], cfg["s"], step=0)
    lref, G = R.step_grads(R.to64(W), tok, tgt, cfg["a"])
    md = P.Model(cfg["L"], cfg["h"], cfg["a"], cfg["f"], cfg["V"], cfg["s"], cfg["b"], 0)
    plan = P.Plan(md, p, m, strategy="1f1b_full_recomp", recomp_layers=r)
    rt = RT.Runtime(plan, stage=-1)
    for s in range(p):
        rt.set_params(s, 1, PR.pack(W, p, 1, plan.partition, s, 1))
    rt.step(tok, tgt, RT.STEP_NO_OPT)
    for s in range(p):
        for (k, l), g in PR.unpack(rt.get_grads(s, 1), W, p, 1, plan.partition, s, 1).items():
            ref = G["layers"][l][k] if l is not None else G[k]
            assert max_rel(g, ref) <= 1e-4, (s, k, l)
    assert all(rt.stats()["pool_high_water"][s] == plan.peak(s)["total_peak"] for s in range(p))
    rt.close()
    ref = _run(dict(cfg), p, m, "1f1b")
    _assert_same(ref, _run(dict(cfg), p, m, "1f1b_full_recomp", recomp_layers=r), ("1f1b_r", r))


def test_config_loader_end_to_end(tmp_path):
    """JSON config -> plan -> runtime -> step gives the same loss and
    gradients as the direct API call (config.py is marshalling only)."""
    import json
    P, RT, PR = mods()
    from paper_2503_03182_b200 import config as CFG
    cfg, p, m = C1_16, 4, 8
    doc = {"model": {"n_layers": cfg["L"], "hidden": cfg["h"], "n_heads": cfg["a"], "ffn_hidden": cfg["f"],
                     "vocab": cfg["V"], "seq_len": cfg["s"], "micro_batch": cfg["b"], "dtype": "bf16"},
           "p": p, "m": m, "strategy": "tpipe_trecomp", "chunks": 2}
    f = tmp_path / "cfg.json"
    f.write_text(json.dumps(doc))
    outs = []
    md = P.Model(cfg["L"], cfg["h"], cfg["a"], cfg["f"], cfg["V"], cfg["s"], cfg["b"], P.BF16)
    for plan in (CFG.load(str(f)), P.Plan(md, p, m, strategy="tpipe_trecomp")):
        rt = RT.Runtime(plan, stage=-1)
        W = synth.weights(cfg["L"], cfg["h"], cfg["f"], cfg["V"], cfg["s"], seed=11, std=0.05,
                          bias_std=0.02, ln_jitter=0.05)
        for s in range(p):
            for c in (1, 2):
                rt.set_params(s, c, PR.pack(W, p, 2, plan.partition, s, c))
        tok, tgt = synth.tokens(cfg["V"], m, cfg["b"], cfg["s"], step=0)
        loss = rt.step(tok, tgt, RT.STEP_NO_OPT)
        outs.append((loss, [rt.get_grads(s, c).view(np.uint32).copy() for s in range(p) for c in (1, 2)]))
        rt.close()
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(a, b)
