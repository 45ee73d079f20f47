"""Plan parity (CPU): the C++ planner behind tpipe_plan_create must emit the
same per-stage instruction streams and the same byte-exact per-stage peaks
as the independent oracle (oracle/stream.py), for every strategy, several
stage counts and micro-batch counts. Also: the C-ABI library loads and
exports every symbol include/*.h declares."""

import os
import re

import pytest

from oracle import schedule as S
from oracle import stream as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _plan_mod():
    from paper_2503_03182_b200 import plan
    return plan


def declared_symbols():
    names = []
    for hdr in ("tpipe.h", "tpipe_kernels.h"):
        src = open(os.path.join(ROOT, "include", hdr)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"\b(tpipe_\w+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_2503_03182_b200 import LIB_PATH
    L = ctypes.CDLL(LIB_PATH)
    missing = [n for n in declared_symbols() if not hasattr(L, n)]
    assert not missing, missing
    assert len(declared_symbols()) >= 30


def oracle_ops(st):
    return [dict(kind=i.kind, chunk=i.chunk, mb=i.mb, peer=i.peer, channel=tuple(i.channel),
                 msg=i.msg) for i in st]


def live_trace(ops, size_of):
    """cumulative live bytes after each instruction's allocs (before frees)."""
    cur, out = 0, []
    for o in ops:
        for a in o["allocs"]:
            cur += size_of(a)
        out.append(cur)
        for f in o["frees"]:
            cur -= size_of(f)
    return out


CASES = []
for strat in ("tpipe", "tpipe_trecomp", "1f1b", "1f1b_full_recomp"):
    for p in (1, 2, 3, 4, 8):
        for m in (1, 3, 8, 32):
            CASES.append((strat, p, m))
for strat in ("interleave", "interleave_trecomp"):          # NEXT-2 (m % p == 0)
    for p, m in ((1, 3), (2, 8), (3, 6), (4, 8), (4, 32), (8, 8), (8, 32)):
        CASES.append((strat, p, m))


@pytest.mark.parametrize("strategy,p,m", CASES)
@pytest.mark.parametrize("dtype", [T.BF16, T.FP32])
def test_streams_and_peaks_match_oracle(strategy, p, m, dtype):
    P = _plan_mod()
    L = 2 * p if p > 2 else 4
    od = T.ModelDesc(L, 64, 4, 256, 128, 32, 2, dtype)
    pd = P.Model(L, 64, 4, 256, 128, 32, 2, dtype)
    plan = P.Plan(pd, p, m, strategy=strategy)
    st, static = T.build_streams(od, p, m, strategy)
    for s in range(p):
        got, bufs = plan.ops(s)
        want = oracle_ops(st[s])
        strip = [{k: o[k] for k in ("kind", "chunk", "mb", "peer", "channel", "msg")} for o in got]
        assert strip == want, f"stage {s}"
        # allocations: same categories and bytes in the same order
        for g, w in zip(got, st[s]):
            assert [(bufs[a][1], bufs[a][4]) for a in g["allocs"]] == [(c, b) for _n, c, b in w.allocs]
            assert len(g["frees"]) == len(w.frees)
        # identical live-byte trace and peaks
        sizes = {n: b for ins in st[s] for n, _c, b in ins.allocs}
        w_trace = live_trace([dict(allocs=[n for n, _c, _b in i.allocs], frees=i.frees)
                              for i in st[s]], lambda n: sizes[n])
        g_trace = live_trace(got, lambda a: bufs[a][4])
        assert g_trace == w_trace
        r = T.replay(st[s], static[s])
        pk = plan.peak(s)
        assert pk["total_peak"] == r["total_peak"]
        for cat in ("model_state", "io", "act", "recomp_buf", "comm", "workspace"):
            assert pk[cat] == r.get(cat, 0), cat


@pytest.mark.parametrize("p", [2, 4, 8])
def test_offload_streams_match_oracle(p):
    P = _plan_mod()
    od = T.ModelDesc(2 * p, 64, 4, 256, 128, 32, 2, T.BF16)
    pd = P.Model(2 * p, 64, 4, 256, 128, 32, 2, T.BF16)
    plan = P.Plan(pd, p, 16, strategy="tpipe_trecomp", offload=P.OFFLOAD_MODEL_STATE)
    st, static = T.build_streams(od, p, 16, "tpipe_trecomp", offload_model_state=True)
    for s in range(p):
        got, _ = plan.ops(s)
        strip = [{k: o[k] for k in ("kind", "chunk", "mb", "peer", "channel", "msg")} for o in got]
        assert strip == oracle_ops(st[s])
        assert plan.peak(s)["total_peak"] == T.replay(st[s], static[s])["total_peak"]


@pytest.mark.parametrize("p", [1, 2, 4, 8])
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_device_opt_offload_streams_match_oracle(p, dtype):
    """Streamed device AdamW (R24): STREAM_OPT replaces GRAD_D2H / HOST_OPT /
    W_H2D; the double-buffered slice staging is static model-state bytes, so
    the peak is the host-optimizer plan's plus 2 * 12 * min(P, slice)."""
    P = _plan_mod()
    dt = T.BF16 if dtype == "bf16" else T.FP32
    od = T.ModelDesc(2 * p, 64, 4, 256, 128, 32, 2, dt)
    pd = P.Model(2 * p, 64, 4, 256, 128, 32, 2, P.BF16 if dtype == "bf16" else P.FP32)
    flags = P.OFFLOAD_MODEL_STATE | P.OFFLOAD_DEVICE_OPT
    plan = P.Plan(pd, p, 16, strategy="tpipe_trecomp", offload=flags)
    host = P.Plan(pd, p, 16, strategy="tpipe_trecomp", offload=P.OFFLOAD_MODEL_STATE)
    st, static = T.build_streams(od, p, 16, "tpipe_trecomp", offload_model_state=True,
                                 offload_device_opt=True)
    for s in range(p):
        got, _ = plan.ops(s)
        strip = [{k: o[k] for k in ("kind", "chunk", "mb", "peer", "channel", "msg")} for o in got]
        assert strip == oracle_ops(st[s])
        kinds = [o["kind"] for o in got]
        assert kinds.count("STREAM_OPT") == 1
        assert not {"GRAD_D2H", "HOST_OPT", "W_H2D"} & set(kinds)
        assert kinds.count("W_WAIT") == 1
        rep = T.replay(st[s], static[s])
        assert plan.peak(s)["total_peak"] == rep["total_peak"]
        extra = T.sopt_staging_bytes(plan.chunk_params(s, 2))
        assert plan.peak(s)["total_peak"] == host.peak(s)["total_peak"] + extra
    from paper_2503_03182_b200._lib import TPipeError
    with pytest.raises(TPipeError):
        P.Plan(pd, p, 16, strategy="tpipe_trecomp", offload=P.OFFLOAD_DEVICE_OPT)


@pytest.mark.parametrize("strategy", ["tpipe", "tpipe_trecomp", "1f1b", "1f1b_full_recomp",
                                      "interleave", "interleave_trecomp"])
@pytest.mark.parametrize("p", [1, 2, 4, 5, 8, 16])
def test_simulate_matches_oracle(strategy, p):
    """C++ unit-time replay == oracle simulator (makespan and busy time)."""
    P = _plan_mod()
    m = 2 * p + 3 if not strategy.startswith("interleave") else 3 * p
    plan = P.Plan(P.Model(2 * p if p > 1 else 2, 64, 4, 256, 128, 32, 2), p, m, strategy=strategy)
    orders, v, rec, dur = S.strategy_orders(strategy, p, m)
    sim = S.simulate(orders, p, v, dur, rec)
    mk, busy = plan.simulate()
    assert mk == sim["makespan"]
    for s in range(p):
        assert busy[s] == sum(sim["end"][(s, o)] - sim["start"][(s, o)] for o in orders[s])


def test_delay_rounds_and_params():
    P = _plan_mod()
    for p, k in [(3, 0), (8, 1), (10, 0), (16, 0)]:
        plan = P.Plan(P.Model(2 * p, 64, 4, 256, 128, 32, 2), p, 2 * p, strategy="tpipe_trecomp")
        assert plan.k == k == S.delay_rounds(p)
    od = T.ModelDesc(8, 64, 4, 256, 128, 32, 2)
    plan = P.Plan(P.Model(8, 64, 4, 256, 128, 32, 2), 4, 8, strategy="tpipe")
    for s in range(4):
        for c in (1, 2):
            assert plan.chunk_params(s, c) == T.chunk_params(od, 4, 2, s, c)


def test_budget_escalation_and_errors():
    P = _plan_mod()
    from paper_2503_03182_b200._lib import TPipeError
    md = P.Model(16, 64, 4, 256, 128, 32, 2)
    a = P.Plan(md, 8, 32, strategy="tpipe")
    b = P.Plan(md, 8, 32, strategy="tpipe_trecomp")
    c = P.Plan(md, 8, 32, strategy="tpipe_trecomp", offload=P.OFFLOAD_MODEL_STATE)
    pa, pb, pc = (max(x.peak(s)["total_peak"] for s in range(8)) for x in (a, b, c))
    assert pa > pb > pc
    assert P.Plan(md, 8, 32, hbm_budget=pa, strategy="auto").strategy == P.S_TPIPE
    auto = P.Plan(md, 8, 32, hbm_budget=pb, strategy="auto")
    assert (auto.strategy, auto.offload) == (P.S_TPIPE_TRECOMP, 0)
    auto = P.Plan(md, 8, 32, hbm_budget=pc, strategy="auto")
    assert (auto.strategy, auto.offload) == (P.S_TPIPE_TRECOMP, 1)
    with pytest.raises(TPipeError, match="budget"):
        P.Plan(md, 8, 32, hbm_budget=pc - 1, strategy="auto")
    with pytest.raises(TPipeError, match="n_layers"):
        P.Plan(P.Model(15, 64, 4, 256, 128, 32, 2), 8, 32)
    with pytest.raises(TPipeError, match="hidden"):
        P.Plan(P.Model(16, 60, 4, 256, 128, 32, 2), 8, 32)
    with pytest.raises(TPipeError, match="deadlock"):
        P.Plan(md, 8, 32, strategy="tpipe_trecomp", send_window=1)


@pytest.mark.parametrize("strategy,p", [("tpipe", 1), ("tpipe", 4), ("1f1b", 2), ("tpipe", 2)])
def test_param_packing_matches_plan(strategy, p):
    """Packed chunk vectors (params.py) have exactly the
    plan's per-chunk parameter counts and cover every global layer once."""
    import synth
    P = _plan_mod()
    from paper_2503_03182_b200 import params as PR
    L = 8
    plan = P.Plan(P.Model(L, 64, 4, 256, 128, 32, 2), p, 4, strategy=strategy)
    W = synth.weights(L, 64, 256, 128, 32)
    seen = []
    for s in range(p):
        for c in range(1, plan.v + 1):
            flat = PR.pack(W, p, plan.v, plan.layers_chunk, s, c)
            assert flat.size == plan.chunk_params(s, c)
            seen += PR.global_layers(p, plan.v, plan.layers_chunk, s, c)
            back = PR.unpack(flat, W, p, plan.v, plan.layers_chunk, s, c)
            for (k, l), a in back.items():
                ref = W["layers"][l][k] if l is not None else W[k]
                assert (a == ref).all()
    assert sorted(seen) == list(range(L))


@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("dist", [1, 2, 3])
def test_activation_offload_streams_match_oracle(p, dist):
    """Activation offload (R23): identical instruction streams and byte peaks;
    the offloaded plan never needs more HBM than plain T-Pipe."""
    P = _plan_mod()
    L = 2 * p if p > 2 else 4
    od = T.ModelDesc(L, 64, 4, 256, 128, 32, 2, T.BF16)
    pd = P.Model(L, 64, 4, 256, 128, 32, 2, T.BF16)
    plan = P.Plan(pd, p, 16, strategy="tpipe", offload=P.OFFLOAD_ACTIVATIONS, act_distance=dist)
    base = P.Plan(pd, p, 16, strategy="tpipe")
    st, static = T.build_streams(od, p, 16, "tpipe", offload_activations=True, act_distance=dist)
    assert T.deadlock_free(st)
    for s in range(p):
        got, bufs = plan.ops(s)
        strip = [{k: o[k] for k in ("kind", "chunk", "mb", "peer", "channel", "msg")} for o in got]
        assert strip == oracle_ops(st[s])
        r = T.replay(st[s], static[s])
        assert plan.peak(s)["total_peak"] == r["total_peak"]
        assert r["total_peak"] <= base.peak(s)["total_peak"]
    from paper_2503_03182_b200._lib import TPipeError
    with pytest.raises(TPipeError, match="activation offload"):
        P.Plan(pd, p, 16, strategy="tpipe_trecomp", offload=P.OFFLOAD_ACTIVATIONS)


@pytest.mark.parametrize("p", [1, 2, 4, 8])
@pytest.mark.parametrize("n", [4, 6])
@pytest.mark.parametrize("dtype", [T.BF16, T.FP32])
def test_partial_trecomp_streams_match_oracle(p, n, dtype):
    """Partial T-Recomp (R25, NEXT-1): for every r in 1..n1 the planner's
    instruction streams, buffer sizes and per-category peaks equal the
    oracle's; r = n1 is block-wise T-Recomp."""
    P = _plan_mod()
    L = n * p
    od = T.ModelDesc(L, 64, 4, 256, 128, 32, 2, dtype)
    pd = P.Model(L, 64, 4, 256, 128, 32, 2, dtype)
    n1 = T.layers_per_chunk(od, p, 2)[0]
    m = 2 * p + 2
    full = P.Plan(pd, p, m, strategy="tpipe_trecomp")
    assert full.recomp_layers == n1
    for r in range(1, n1 + 1):
        plan = P.Plan(pd, p, m, strategy="tpipe_trecomp", recomp_layers=r)
        assert plan.recomp_layers == r
        st, static = T.build_streams(od, p, m, "tpipe_trecomp", recomp_layers=r)
        for s in range(p):
            got, bufs = plan.ops(s)
            strip = [{k: o[k] for k in ("kind", "chunk", "mb", "peer", "channel", "msg")} for o in got]
            assert strip == oracle_ops(st[s])
            for g, w in zip(got, st[s]):
                assert [(bufs[a][1], bufs[a][4]) for a in g["allocs"]] == [(c, b) for _n, c, b in w.allocs]
                assert len(g["frees"]) == len(w.frees)
            rep = T.replay(st[s], static[s])
            pk = plan.peak(s)
            for cat in ("model_state", "io", "act", "recomp_buf", "comm", "workspace"):
                assert pk[cat] == rep.get(cat, 0), cat
            assert pk["total_peak"] == rep["total_peak"]
            if r == n1:
                assert pk == full.peak(s)
    from paper_2503_03182_b200._lib import TPipeError
    with pytest.raises(TPipeError, match="recomp_layers"):
        P.Plan(pd, p, m, strategy="tpipe_trecomp", recomp_layers=n1 + 1)


def test_auto_escalation_partial_trecomp():
    """The auto ladder spends the least recompute that fits: a budget between
    the r=1 and r=2 peaks selects r=2 (of n1=3), before model-state offload."""
    P = _plan_mod()
    md = P.Model(48, 64, 4, 256, 128, 32, 2)            # p=8: n=6 -> n1=3
    pk = {r: max(P.Plan(md, 8, 32, strategy="tpipe_trecomp", recomp_layers=r).peak(s)["total_peak"]
                 for s in range(8)) for r in (1, 2, 3)}
    tp = max(P.Plan(md, 8, 32, strategy="tpipe").peak(s)["total_peak"] for s in range(8))
    assert tp > pk[1] > pk[2] > pk[3]
    auto = P.Plan(md, 8, 32, hbm_budget=pk[2], strategy="auto")
    assert (auto.strategy, auto.offload, auto.recomp_layers) == (P.S_TPIPE_TRECOMP, 0, 2)
    auto = P.Plan(md, 8, 32, hbm_budget=pk[1], strategy="auto")
    assert auto.recomp_layers == 1
    off = max(P.Plan(md, 8, 32, strategy="tpipe_trecomp", recomp_layers=1,
                     offload=P.OFFLOAD_MODEL_STATE).peak(s)["total_peak"] for s in range(8))
    if off < pk[3]:
        auto = P.Plan(md, 8, 32, hbm_budget=off, strategy="auto")
        assert (auto.offload, auto.recomp_layers) == (P.OFFLOAD_MODEL_STATE, 1)


def test_interleave_needs_m_multiple_of_p_and_simulates():
    """Interleave-1F1B needs m % p == 0 (Megatron order); the C++ unit-time
    replay of Interleave + T-Recomp reproduces D-9's 133 at p=8, m=16."""
    P = _plan_mod()
    from paper_2503_03182_b200._lib import TPipeError
    md = P.Model(16, 64, 4, 256, 128, 32, 2)
    with pytest.raises(TPipeError, match="interleave"):
        P.Plan(md, 8, 12, strategy="interleave")
    mk, _busy = P.Plan(md, 8, 16, strategy="interleave_trecomp").simulate()
    assert mk == 133


@pytest.mark.parametrize("strategy", ["tpipe", "tpipe_trecomp", "1f1b", "1f1b_full_recomp",
                                      "interleave_trecomp"])
@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_simulate_durations_matches_oracle(strategy, p):
    """tpipe_plan_simulate_durations (ASAP replay with per-op durations, used
    to replay measured op times) == the oracle simulator with the same
    durations; with the unit durations it equals tpipe_plan_simulate."""
    import random
    P = _plan_mod()
    m = 2 * p
    plan = P.Plan(P.Model(2 * p if p > 1 else 2, 64, 4, 256, 128, 32, 2), p, m, strategy=strategy)
    orders, v, rec, dur = S.strategy_orders(strategy, p, m)
    rng = random.Random(p * 31 + len(strategy))
    ms = [[rng.randint(1, 40) / 8.0 for _ in orders[s]] for s in range(p)]
    mk, busy = plan.simulate_durations(ms)
    idx = {(s, op): j for s in range(p) for j, op in enumerate(orders[s])}
    sim = S.simulate(orders, p, v, lambda s, op: ms[s][idx[(s, op)]], rec)
    assert mk == pytest.approx(sim["makespan"], abs=1e-9)
    for s in range(p):
        assert busy[s] == pytest.approx(sum(ms[s]), abs=1e-9)
    unit = [[float(dur.get("B1", dur["B"]) if (op[0] == "B" and op[1] == 1) else dur[op[0]])
             for op in orders[s]] for s in range(p)]
    assert plan.simulate_durations(unit)[0] == plan.simulate()[0]


PARTITIONS = [(4, (3, 3, 2, 2)), (4, (2, 2, 2, 4)), (2, (5, 3)), (8, (3, 3, 3, 3, 3, 3, 4, 2))]


@pytest.mark.parametrize("p,part", PARTITIONS)
@pytest.mark.parametrize("strategy", ["tpipe", "tpipe_trecomp", "1f1b", "1f1b_full_recomp",
                                      "interleave_trecomp"])
def test_partition_streams_match_oracle(p, part, strategy):
    """Cost-balanced partition (R27, SURVEY D-12): a per-stage layer vector;
    instruction streams, buffer sizes and per-category peaks equal the
    oracle's; chunk parameter counts follow the per-stage layers."""
    P = _plan_mod()
    L = sum(part)
    m = 2 * p
    od = T.ModelDesc(L, 64, 4, 256, 128, 32, 2, T.BF16, stage_layers=part)
    pd = P.Model(L, 64, 4, 256, 128, 32, 2, P.BF16)
    plan = P.Plan(pd, p, m, strategy=strategy, stage_layers=part)
    st, static = T.build_streams(od, p, m, strategy)
    for s in range(p):
        got, bufs = plan.ops(s)
        strip = [{k: o[k] for k in ("kind", "chunk", "mb", "peer", "channel", "msg")} for o in got]
        assert strip == oracle_ops(st[s])
        for g, w in zip(got, st[s]):
            assert [(bufs[a][1], bufs[a][4]) for a in g["allocs"]] == [(c, b) for _n, c, b in w.allocs]
        rep = T.replay(st[s], static[s])
        pk = plan.peak(s)
        for cat in ("model_state", "io", "act", "recomp_buf", "comm", "workspace"):
            assert pk[cat] == rep.get(cat, 0), cat
        for c in range(1, plan.v + 1):
            assert plan.chunk_params(s, c) == T.chunk_params(od, p, plan.v, s, c)
        assert sum(plan.partition[s]) == part[s]
    from paper_2503_03182_b200._lib import TPipeError
    with pytest.raises(TPipeError, match="stage_layers"):
        P.Plan(pd, p, m, strategy=strategy, stage_layers=list(part[:-1]) + [part[-1] + 1])


def test_partition_partial_trecomp_matches_oracle():
    """Partial T-Recomp with a partition: stage s recomputes min(r, n1(s))."""
    P = _plan_mod()
    part = (6, 4, 2, 4)
    od = T.ModelDesc(16, 64, 4, 256, 128, 32, 2, T.BF16, stage_layers=part)
    pd = P.Model(16, 64, 4, 256, 128, 32, 2, P.BF16)
    for r in (1, 2, 3):
        plan = P.Plan(pd, 4, 8, strategy="tpipe_trecomp", recomp_layers=r, stage_layers=part)
        st, static = T.build_streams(od, 4, 8, "tpipe_trecomp", recomp_layers=r)
        for s in range(4):
            assert plan.peak(s)["total_peak"] == T.replay(st[s], static[s])["total_peak"]


@pytest.mark.parametrize("p,part,chunk1", [(4, (5, 4, 4, 3), (4, 1, 2, 2)), (2, (7, 5), (3, 4)),
                                           (8, (2, 2, 3, 2, 2, 3, 2, 2), (1, 1, 2, 1, 1, 1, 1, 1))])
@pytest.mark.parametrize("strategy", ["tpipe", "tpipe_trecomp", "interleave_trecomp"])
def test_partition_chunk_split_streams_match_oracle(p, part, chunk1, strategy):
    """Duration-aware partition (R29): per-stage chunk-1
    layer counts; streams, buffer sizes and peaks equal the oracle's."""
    P = _plan_mod()
    L = sum(part)
    m = 2 * p
    od = T.ModelDesc(L, 64, 4, 256, 128, 32, 2, T.BF16, stage_layers=part, stage_chunk1=chunk1)
    pd = P.Model(L, 64, 4, 256, 128, 32, 2, P.BF16)
    plan = P.Plan(pd, p, m, strategy=strategy, stage_layers=part, stage_chunk1=chunk1)
    assert [x[0] for x in plan.partition] == list(chunk1)
    st, static = T.build_streams(od, p, m, strategy)
    for s in range(p):
        got, bufs = plan.ops(s)
        strip = [{k: o[k] for k in ("kind", "chunk", "mb", "peer", "channel", "msg")} for o in got]
        assert strip == oracle_ops(st[s])
        for g, w in zip(got, st[s]):
            assert [(bufs[a][1], bufs[a][4]) for a in g["allocs"]] == [(c, b) for _n, c, b in w.allocs]
        assert plan.peak(s)["total_peak"] == T.replay(st[s], static[s])["total_peak"]
    from paper_2503_03182_b200._lib import TPipeError
    with pytest.raises(TPipeError, match="stage_chunk1"):
        P.Plan(pd, p, m, strategy=strategy, stage_layers=part,
               stage_chunk1=[part[0]] + list(chunk1[1:]))


@pytest.mark.parametrize("strategy", ["tpipe", "tpipe_trecomp", "1f1b", "1f1b_full_recomp",
                                      "interleave_trecomp"])
@pytest.mark.parametrize("p,dp", [(1, 2), (2, 2), (4, 2), (2, 4), (1, 8)])
@pytest.mark.parametrize("dtype", [T.BF16, T.FP32])
def test_dp_zero1_streams_match_oracle(strategy, p, dp, dtype):
    """DP x PP with ZeRO-1 (NEXT-3, R31): DP_WAIT before each chunk's first
    forward, DP_OPT instead of OPT, model-state bytes with the optimizer
    states of one shard; streams and peaks equal the oracle's."""
    P = _plan_mod()
    L = 2 * p if p > 2 else 4
    m = 2 * p
    od = T.ModelDesc(L, 64, 4, 256, 128, 32, 2, dtype)
    pd = P.Model(L, 64, 4, 256, 128, 32, 2, dtype)
    plan = P.Plan(pd, p, m, strategy=strategy, dp=dp)
    assert plan.dp == dp
    st, static = T.build_streams(od, p, m, strategy, dp=dp)
    for s in range(p):
        got, bufs = plan.ops(s)
        strip = [{k: o[k] for k in ("kind", "chunk", "mb", "peer", "channel", "msg")} for o in got]
        assert strip == oracle_ops(st[s])
        kinds = [o["kind"] for o in got]
        assert "OPT" not in kinds and kinds.count("DP_OPT") == plan.v and kinds.count("DP_WAIT") == plan.v
        rep = T.replay(st[s], static[s])
        pk = plan.peak(s)
        for cat in ("model_state", "io", "act", "recomp_buf", "comm", "workspace"):
            assert pk[cat] == rep.get(cat, 0), cat
    # ZeRO-1 saves (1 - 1/dp) of the optimizer-state bytes (12 B/param bf16, 8 fp32)
    one = P.Plan(pd, p, m, strategy=strategy)
    for s in range(p):
        saved = one.peak(s)["model_state"] - plan.peak(s)["model_state"]
        per = 12 if dtype == T.BF16 else 8
        n = sum(one.chunk_params(s, c) for c in range(1, one.v + 1))
        assert saved >= per * n * (1 - 1 / dp) - per * 64 * one.v
    from paper_2503_03182_b200._lib import TPipeError
    if strategy.startswith("tpipe"):
        with pytest.raises(TPipeError, match="ZeRO-1"):
            P.Plan(pd, p, m, strategy=strategy, dp=dp, offload=P.OFFLOAD_MODEL_STATE)


@pytest.mark.parametrize("p,r", [(1, 1), (1, 2), (2, 1), (2, 2), (4, 1), (4, 2), (8, 1)])
@pytest.mark.parametrize("dtype", [T.BF16, T.FP32])
def test_1f1b_partial_recompute_matches_oracle(p, r, dtype):
    """1F1B + layer-grouped recompute of the r shallowest layers per stage
    (r = n/2: the paper's 1F1B + R50 baseline; DESIGN R33): streams
    and bytes equal the oracle's, the stash follows r inputs + (n - r) full
    layers, and the unit replay of R50 takes 7(m+p-1) (D-5)."""
    P = _plan_mod()
    L = 4 * p
    m = 2 * p + 2
    od = T.ModelDesc(L, 64, 4, 256, 128, 32, 2, dtype)
    pd = P.Model(L, 64, 4, 256, 128, 32, 2, dtype)
    plan = P.Plan(pd, p, m, strategy="1f1b_full_recomp", recomp_layers=r)
    assert plan.recomp_layers == r
    st, static = T.build_streams(od, p, m, "1f1b_full_recomp", recomp_layers=r)
    for s in range(p):
        got, bufs = plan.ops(s)
        strip = [{k: o[k] for k in ("kind", "chunk", "mb", "peer", "channel", "msg")} for o in got]
        assert strip == oracle_ops(st[s])
        rep = T.replay(st[s], static[s])
        pk = plan.peak(s)
        for cat in ("model_state", "io", "act", "recomp_buf", "comm", "workspace"):
            assert pk[cat] == rep.get(cat, 0), cat
    z = T.sizes(od, p, 1, min(1, p - 1), 1, full_recomp=True, ckpt_layers=r)
    full = T.sizes(od, p, 1, min(1, p - 1), 1)
    es = 2 if dtype == T.BF16 else 4
    M, h = 64, 64
    assert z["stash"] == full["stash"] - r * (full["layer_stash"] - M * h * es)
    if r * 2 == L // p:
        assert plan.simulate()[0] == 7 * (m + p - 1)
