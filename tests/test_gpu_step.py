"""Full training-step parity through the C-ABI (tpipe_plan -> tpipe_runtime ->
tpipe_step) against the fp64 oracle (oracle.model), on seeded synthetic
inputs of config C1 shape (BASELINE.json configs[0]).

Bars (BASELINE.json north_star): fp32 mode loss and every
gradient tensor max-relative error <= 1e-4; bf16 mode relative L2 <= 2e-2;
T-Recomp on/off and T-Offload on/off bit-exact; pool ledger high-water ==
plan peak bytes exactly.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from oracle import model as R  # noqa: E402

C1 = dict(n_layers=8, hidden=64, n_heads=4, ffn_hidden=256, vocab=256, seq_len=32, micro_batch=2)


def mods():
    from paper_2503_03182_b200 import params, plan, runtime
    return plan, runtime, params


def build(cfg, p, m, strategy, dtype, offload=0, lr=1e-3, seed=11, recomp_layers=0, stage_layers=None,
          act_distance=None):
    P, RT, PR = mods()
    md = P.Model(cfg["n_layers"], cfg["hidden"], cfg["n_heads"], cfg["ffn_hidden"], cfg["vocab"],
                 cfg["seq_len"], cfg["micro_batch"], dtype)
    if act_distance is None:
        # activation offload at these tiny sizes: the bandwidth-derived distance
        # (Q12) would keep every block on the device; use round 1's fixed 2
        act_distance = 2 if offload & P.OFFLOAD_ACTIVATIONS else 0
    plan = P.Plan(md, p, m, strategy=strategy, offload=offload, recomp_layers=recomp_layers,
                  stage_layers=stage_layers, act_distance=act_distance)
    rt = RT.Runtime(plan, stage=-1, lr=lr)
    W = synth.weights(cfg["n_layers"], cfg["hidden"], cfg["ffn_hidden"], cfg["vocab"],
                      cfg["seq_len"], seed=seed, std=0.05, bias_std=0.02, ln_jitter=0.05)
    for s in range(p):
        for c in range(1, plan.v + 1):
            rt.set_params(s, c, PR.pack(W, p, plan.v, plan.partition, s, c))
    return plan, rt, W


def oracle_grads(cfg, W, tok, tgt):
    return R.step_grads(R.to64(W), tok, tgt, cfg["n_heads"])


def compare(plan, rt, W, G, metric, tol):
    _P, _RT, PR = mods()
    worst = 0.0
    for s in range(plan.p):
        for c in range(1, plan.v + 1):
            got = PR.unpack(rt.get_grads(s, c), W, plan.p, plan.v, plan.partition, s, c)
            for (k, l), g in got.items():
                ref = G["layers"][l][k] if l is not None else G[k]
                err = metric(g, ref)
                worst = max(worst, err)
                assert err <= tol, (s, c, k, l, err)
    return worst


def max_rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / (np.abs(b).max() + 1e-30))


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))


@pytest.mark.parametrize("strategy", ["tpipe", "tpipe_trecomp", "1f1b", "1f1b_full_recomp",
                                      "interleave", "interleave_trecomp"])
@pytest.mark.parametrize("p", [1, 2, 4])
def test_step_fp32_parity(strategy, p):
    _P, RT, _PR = mods()
    m = 8
    plan, rt, W = build(C1, p, m, strategy, 0)
    tok, tgt = synth.tokens(C1["vocab"], m, C1["micro_batch"], C1["seq_len"], step=0)
    loss = rt.step(tok, tgt, RT.STEP_NO_OPT)
    lref, G = oracle_grads(C1, W, tok, tgt)
    assert abs(loss - lref) / abs(lref) < 1e-5
    compare(plan, rt, W, G, max_rel, 1e-4)
    # pool ledger high-water == plan peak (byte-exact)
    st = rt.stats()
    for s in range(p):
        assert st["pool_high_water"][s] == plan.peak(s)["total_peak"]
    assert st["kernel_launches"] > 0


@pytest.mark.parametrize("strategy", ["tpipe", "tpipe_trecomp"])
def test_step_bf16_parity(strategy):
    _P, RT, _PR = mods()
    p, m = 4, 8
    plan, rt, W = build(C1, p, m, strategy, 1)
    tok, tgt = synth.tokens(C1["vocab"], m, C1["micro_batch"], C1["seq_len"], step=0)
    loss = rt.step(tok, tgt, RT.STEP_NO_OPT)
    lref, G = oracle_grads(C1, W, tok, tgt)
    assert abs(loss - lref) / abs(lref) < 2e-2
    compare(plan, rt, W, G, rel_l2, 2e-2)


@pytest.mark.parametrize("dtype", [0, 1])
def test_trecomp_bitexact_vs_tpipe(dtype):
    """T-Recomp regenerates chunk-1 activations with the same kernels, so the
    gradients are bit-identical to T-Pipe's (BASELINE north_star); the
    Interleave-1F1B orders (NEXT-2, with and without T-Recomp) accumulate each
    chunk's gradients in the same micro-batch order, so they match too."""
    _P, RT, _PR = mods()
    p, m = 4, 8
    tok, tgt = synth.tokens(C1["vocab"], m, C1["micro_batch"], C1["seq_len"], step=3)
    out = []
    for strategy in ("tpipe", "tpipe_trecomp", "interleave", "interleave_trecomp"):
        plan, rt, _W = build(C1, p, m, strategy, dtype)
        loss = rt.step(tok, tgt, RT.STEP_NO_OPT)
        out.append((loss, [rt.get_grads(s, c) for s in range(p) for c in (1, 2)]))
    for o in out[1:]:
        assert out[0][0] == o[0]
        for a, b in zip(out[0][1], o[1]):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("dtype", [0, 1])
@pytest.mark.parametrize("p,r", [(1, 1), (1, 3), (2, 1)])
def test_partial_trecomp_bitexact_vs_tpipe(dtype, p, r):
    """Partial T-Recomp (R25): R regenerates chunk-1 layers 1..r into the
    recompute buffer while layers r+1..n1 keep their stash; loss and every
    gradient are bit-identical to T-Pipe's, the updated parameters after one
    optimizer step too, and the pool ledger high-water equals the plan peak."""
    _P, RT, _PR = mods()
    m = 8
    tok, tgt = synth.tokens(C1["vocab"], m, C1["micro_batch"], C1["seq_len"], step=5)
    out = []
    for strategy, rl in (("tpipe", 0), ("tpipe_trecomp", r)):
        plan, rt, _W = build(C1, p, m, strategy, dtype, recomp_layers=rl)
        if rl:
            assert plan.recomp_layers == r < plan.layers_chunk[0]
        loss = rt.step(tok, tgt, RT.STEP_NO_OPT)
        grads = [rt.get_grads(s, c) for s in range(p) for c in (1, 2)]
        rt.step(tok, tgt)
        params = [rt.get_params(s, c) for s in range(p) for c in (1, 2)]
        st = rt.stats()
        for s in range(p):
            assert st["pool_high_water"][s] == plan.peak(s)["total_peak"]
        out.append((loss, grads, params))
        rt.close()
    assert out[0][0] == out[1][0]
    for a, b in zip(out[0][1] + out[0][2], out[1][1] + out[1][2]):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


C_MID = dict(n_layers=4, hidden=256, n_heads=2, ffn_hidden=1024, vocab=512, seq_len=256, micro_batch=1)


@pytest.mark.parametrize("cfg", ["C1", "C_MID"])
@pytest.mark.parametrize("dtype", [0, 1])
def test_side_stream_bitexact(cfg, dtype):
    """Weight-gradient GEMMs on the side stream vs all on one stream: loss,
    gradients and updated parameters bit-identical (C_MID exercises the
    tcgen05 GEMM / attention kernels in bf16)."""
    _P, RT, _PR = mods()
    c = C1 if cfg == "C1" else C_MID
    p, m = 2, 4
    res = []
    try:
        for side in (1, 0):
            RT.set_side_stream(side)
            plan, rt, _W = build(c, p, m, "tpipe", dtype)
            tok, tgt = synth.tokens(c["vocab"], m, c["micro_batch"], c["seq_len"], step=1)
            loss = rt.step(tok, tgt, RT.STEP_NO_OPT)
            grads = [rt.get_grads(s, ch) for s in range(p) for ch in (1, 2)]
            loss2 = rt.step(tok, tgt)
            res.append((loss, loss2, grads, [rt.get_params(s, ch) for s in range(p) for ch in (1, 2)]))
    finally:
        RT.set_side_stream(1)
    assert res[0][0] == res[1][0] and res[0][1] == res[1][1]
    for a, b in zip(res[0][2] + res[0][3], res[1][2] + res[1][3]):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("cfg,dtype,strategy,p", [("C_MID", 1, "tpipe", 1), ("C_MID", 1, "tpipe_trecomp", 2),
                                                   ("C1", 0, "tpipe_trecomp", 4), ("C1", 1, "1f1b", 2)])
def test_graph_step_bitexact(cfg, dtype, strategy, p):
    """TPIPE_STEP_GRAPH (the step's device work captured once as a CUDA graph,
    replayed afterwards; AdamW's per-step hyper-parameters from device memory)
    vs the issued step: losses, gradients (a NO_OPT graph) and parameters after
    3 optimizer steps bit-identical."""
    _P, RT, _PR = mods()
    c = C1 if cfg == "C1" else C_MID
    m = 4
    res = []
    for flags in (0, RT.STEP_GRAPH):
        plan, rt, _W = build(c, p, m, strategy, dtype)
        tok, tgt = synth.tokens(c["vocab"], m, c["micro_batch"], c["seq_len"], step=1)
        l0 = rt.step(tok, tgt, RT.STEP_NO_OPT | flags)
        chunks = [(s, ch) for s in range(p) for ch in range(1, plan.v + 1)]
        grads = [rt.get_grads(s, ch) for s, ch in chunks]
        losses = [l0]
        for step in range(3):
            tok, tgt = synth.tokens(c["vocab"], m, c["micro_batch"], c["seq_len"], step=step + 2)
            losses.append(rt.step(tok, tgt, flags))
        assert rt.stats()["kernel_launches"] > 0
        res.append((losses, grads, [rt.get_params(s, ch) for s, ch in chunks]))
        rt.close()
    assert res[0][0] == res[1][0]
    for a, b in zip(res[0][1] + res[0][2], res[1][1] + res[1][2]):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("dtype", [0, 1])
def test_offload_bitexact(dtype):
    """T-Offload (host AdamW for chunk 2) vs device AdamW: parameters
    after 3 optimizer steps are bit-identical; the step counters and the
    uploaded weights agree."""
    _P, RT, _PR = mods()
    p, m = 4, 8
    res = []
    P = mods()[0]
    for off in (0, P.OFFLOAD_MODEL_STATE, P.OFFLOAD_MODEL_STATE | P.OFFLOAD_DEVICE_OPT):
        plan, rt, _W = build(C1, p, m, "tpipe_trecomp", dtype, offload=off)
        losses = []
        for step in range(3):
            tok, tgt = synth.tokens(C1["vocab"], m, C1["micro_batch"], C1["seq_len"], step=step)
            losses.append(rt.step(tok, tgt))
        res.append((losses, [rt.get_params(s, c) for s in range(p) for c in (1, 2)]))
        st = rt.stats()
        if off:
            assert st["offload_d2h_bytes"] > 0 and st["offload_d2h_ms"] > 0
        assert all(st["pool_high_water"][s] == plan.peak(s)["total_peak"] for s in range(p))
    for r in res[1:]:
        assert res[0][0] == r[0]
        for a, b in zip(res[0][1], r[1]):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_device_opt_offload_multislice_bitexact():
    """Streamed device AdamW (R24) with chunks of 4 slices (the slot reuse and
    the cross-step ordering of the staging area are exercised): parameters
    after 3 steps are bit-identical to the host optimizer's."""
    P, RT, _PR = mods()
    cfg = dict(n_layers=4, hidden=1024, n_heads=8, ffn_hidden=4096, vocab=512, seq_len=64,
               micro_batch=1)
    p, m = 1, 4
    res = []
    for off in (P.OFFLOAD_MODEL_STATE, P.OFFLOAD_MODEL_STATE | P.OFFLOAD_DEVICE_OPT):
        plan, rt, _W = build(cfg, p, m, "tpipe_trecomp", P.BF16, offload=off)
        assert plan.chunk_params(0, 2) > 3 * 8388608
        losses = []
        for step in range(3):
            tok, tgt = synth.tokens(cfg["vocab"], m, 1, cfg["seq_len"], step=step)
            losses.append(rt.step(tok, tgt))
        res.append((losses, [rt.get_params(0, c) for c in (1, 2)]))
        rt.close()
    assert res[0][0] == res[1][0]
    for a, b in zip(res[0][1], res[1][1]):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_adamw_step_matches_oracle_fp32():
    """One full step with the optimizer: new fp32 weights vs the oracle's
    fp64 AdamW applied to the oracle gradients (N-3)."""
    _P, RT, PR = mods()
    p, m, lr = 2, 4, 1e-3
    plan, rt, W = build(C1, p, m, "tpipe", 0, lr=lr)
    tok, tgt = synth.tokens(C1["vocab"], m, C1["micro_batch"], C1["seq_len"], step=0)
    rt.step(tok, tgt)
    _l, G = oracle_grads(C1, W, tok, tgt)
    W64 = R.to64(W)
    for s in range(p):
        for c in (1, 2):
            got = PR.unpack(rt.get_params(s, c), W, p, 2, plan.layers_chunk, s, c)
            for (k, l), w in got.items():
                w0 = W64["layers"][l][k] if l is not None else W64[k]
                g = G["layers"][l][k] if l is not None else G[k]
                ref, _, _ = R.adamw(w0, g, np.zeros_like(g), np.zeros_like(g), 1, lr,
                                    decay=(np.ndim(w0) == 2))
                # step-1 Adam update is ~ lr * sign(g): compare the update itself
                upd, upd_ref = np.asarray(w, np.float64) - w0, ref - w0
                mask = np.abs(g) > 1e-3 * np.abs(g).max()   # |g| >> Adam eps
                assert np.abs(upd - upd_ref)[mask].max() <= 2e-4 * lr + 1e-7, (s, c, k, l)


def test_loss_decreases_bf16():
    """Sanity of the whole step (fwd, bwd, optimizer) at C1: training on a
    fixed batch drives the loss down."""
    _P, RT, _PR = mods()
    p, m = 4, 8
    plan, rt, _W = build(C1, p, m, "tpipe_trecomp", 1, lr=3e-3)
    tok, tgt = synth.tokens(C1["vocab"], m, C1["micro_batch"], C1["seq_len"], step=0)
    losses = [rt.step(tok, tgt) for _ in range(8)]
    assert losses[-1] < losses[0] - 0.1, losses


@pytest.mark.parametrize("dtype", [0, 1])
def test_full_recompute_bitexact_vs_1f1b(dtype):
    """1F1B + full layer-grouped recompute (the in-build baseline)
    regenerates every layer's internals with the same kernels: gradients are
    bit-identical to plain 1F1B."""
    _P, RT, _PR = mods()
    p, m = 2, 4
    tok, tgt = synth.tokens(C1["vocab"], m, C1["micro_batch"], C1["seq_len"], step=5)
    out = []
    for strategy in ("1f1b", "1f1b_full_recomp"):
        plan, rt, _W = build(C1, p, m, strategy, dtype)
        loss = rt.step(tok, tgt, RT.STEP_NO_OPT)
        out.append((loss, [rt.get_grads(s, 1) for s in range(p)]))
        st = rt.stats()
        assert all(st["pool_high_water"][s] == plan.peak(s)["total_peak"] for s in range(p))
    assert out[0][0] == out[1][0]
    for a, b in zip(out[0][1], out[1][1]):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("dtype", [0, 1])
@pytest.mark.parametrize("p", [1, 2, 4])
def test_activation_offload_bitexact(dtype, p):
    """Activation offload (chunk-1 stash -> pinned host -> back, R23) moves
    bytes only: loss and gradients are bit-identical to plain T-Pipe, the
    pool ledger matches the (smaller) plan peak, and bytes actually moved."""
    P, RT, _PR = mods()
    m = 8
    tok, tgt = synth.tokens(C1["vocab"], m, C1["micro_batch"], C1["seq_len"], step=7)
    out = []
    for off in (0, P.OFFLOAD_ACTIVATIONS):
        plan, rt, _W = build(C1, p, m, "tpipe", dtype, offload=off)
        loss = rt.step(tok, tgt, RT.STEP_NO_OPT)
        out.append((loss, [rt.get_grads(s, c) for s in range(p) for c in (1, 2)]))
        st = rt.stats()
        assert all(st["pool_high_water"][s] == plan.peak(s)["total_peak"] for s in range(p))
        if off:
            assert st["offload_d2h_bytes"] > 0 and st["offload_h2d_bytes"] == st["offload_d2h_bytes"]
    assert out[0][0] == out[1][0]
    for a, b in zip(out[0][1], out[1][1]):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_op_times_and_replay():
    """TPIPE_STEP_OP_TIMES records one positive duration per compute op of
    every stage; the measured-duration replay's busy time per stage equals the
    sum of that stage's op times and the makespan bounds it."""
    _P, RT, _PR = mods()
    p, m = 4, 8
    plan, rt, _W = build(C1, p, m, "tpipe_trecomp", 1)
    tok, tgt = synth.tokens(C1["vocab"], m, C1["micro_batch"], C1["seq_len"], step=0)
    rt.step(tok, tgt, RT.STEP_NO_OPT | RT.STEP_OP_TIMES)
    ms = [rt.op_times(s) for s in range(p)]
    for s in range(p):
        assert len(ms[s]) == plan.n_compute_ops(s) == 5 * m
        assert all(x > 0 for x in ms[s])
    mk, busy = plan.simulate_durations(ms)
    for s in range(p):
        assert busy[s] == pytest.approx(sum(ms[s]), rel=1e-6)
        assert mk >= busy[s]
    rt.close()


@pytest.mark.parametrize("strategy,p,part", [("tpipe_trecomp", 2, (5, 3)), ("1f1b", 4, (3, 2, 2, 1)),
                                             ("tpipe", 4, (2, 2, 2, 2))])
def test_partition_step(strategy, p, part):
    """Cost-balanced partition (R27): per-stage layer vector. fp32 gradients
    match the oracle (<= 1e-4), bf16 gradients are bit-identical per tensor to
    the uniform partition's (layer math does not depend on chunk boundaries),
    and the pool ledger high-water equals the plan peak on every stage."""
    _P, RT, PR = mods()
    m = 8
    tok, tgt = synth.tokens(C1["vocab"], m, C1["micro_batch"], C1["seq_len"], step=2)
    plan, rt, W = build(C1, p, m, strategy, 0, stage_layers=part)
    assert [sum(x) for x in plan.partition] == list(part)
    rt.step(tok, tgt, RT.STEP_NO_OPT)
    lref, G = oracle_grads(C1, W, tok, tgt)
    compare(plan, rt, W, G, max_rel, 1e-4)
    st = rt.stats()
    for s in range(p):
        assert st["pool_high_water"][s] == plan.peak(s)["total_peak"]
    rt.close()
    grads = []
    for sl in (part, None):
        plan, rt, W = build(C1, p, m, strategy, 1, stage_layers=sl)
        rt.step(tok, tgt, RT.STEP_NO_OPT)
        g = {}
        for s in range(p):
            for c in range(1, plan.v + 1):
                g.update(PR.unpack(rt.get_grads(s, c), W, p, plan.v, plan.partition, s, c))
        grads.append(g)
        rt.close()
    assert grads[0].keys() == grads[1].keys()
    for k in grads[0]:
        assert np.array_equal(np.asarray(grads[0][k], np.float32).view(np.uint32),
                              np.asarray(grads[1][k], np.float32).view(np.uint32)), k


@pytest.mark.parametrize("dtype", [0, 1])
def test_partition_offload_partial_bitexact(dtype):
    """Features compose: an uneven partition (5, 3) with partial T-Recomp
    (r = 1) and T-Offload of the chunk-2 model states (host AdamW and streamed
    device AdamW) gives parameters after 2 optimizer steps bit-identical to
    plain T-Pipe on the same partition; ledger high-water == plan peak."""
    P = mods()[0]
    p, m = 2, 8
    res = []
    for strat, off, rl in (("tpipe", 0, 0), ("tpipe_trecomp", P.OFFLOAD_MODEL_STATE, 1),
                           ("tpipe_trecomp", P.OFFLOAD_MODEL_STATE | P.OFFLOAD_DEVICE_OPT, 1)):
        plan, rt, _W = build(C1, p, m, strat, dtype, offload=off, recomp_layers=rl, stage_layers=(5, 3))
        losses = []
        for step in range(2):
            tok, tgt = synth.tokens(C1["vocab"], m, C1["micro_batch"], C1["seq_len"], step=step)
            losses.append(rt.step(tok, tgt))
        res.append((losses, [rt.get_params(s, c) for s in range(p) for c in (1, 2)]))
        st = rt.stats()
        assert all(st["pool_high_water"][s] == plan.peak(s)["total_peak"] for s in range(p))
        rt.close()
    for r in res[1:]:
        assert res[0][0] == r[0]
        for a, b in zip(res[0][1], r[1]):
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
