"""v > 2 chunks per stage (SURVEY NEXT-4 and the NEXT-1 remainder; DESIGN R32).

The paper evaluates T-Pipe / Interleave-1F1B + T-Recomp at several chunk
counts (Fig. E56) and multi-chunk T-Offload (model-state
reduction 33.33% / 44% / 49.09% at 2 / 3 / 4 chunks) but gives the v > 2
T-Pipe order only as figures. Reading (R32): D-11's generalisation of the
slot table with period 3v; T-Recomp regenerates chunk 1; T-Offload moves
chunks 2..v. Pins:
* the general recurrence reproduces D-1 exactly at v = 2;
* collision-free (every stage's slot times distinct) for v = 3, 4, p <= 16;
* ASAP makespan 3v(m+p-1) units (one unit = one chunk forward = T_fwd/v:
  the same bubble as 1F1B in real time, D-11) for p >= 4; p = 2, 3 within +3v;
* send window: W = v is deadlock-free and reaches the unconstrained
  makespan; W = 2 deadlocks T-Pipe at v = 4 (the v - 1 chunk turnarounds share
  the wrap channel);
* multi-chunk T-Offload: (v-1)/v x 12/18 of the model-state bytes leave HBM
  on a stage with equal chunks: 1/3, 4/9, 1/2 (P:569's 33.33%, 44%, and
  "near-maximal" 49.09%; SURVEY D-8);
* planner streams and bytes equal the oracle's for v = 3, 4.
"""

import pytest

from oracle import schedule as S
from oracle import stream as T


@pytest.mark.parametrize("p", list(range(1, 17)))
def test_general_slots_reduce_to_d1(p):
    for m in (1, p, 2 * p + 1):
        assert S.tpipe_slots_general(p, m, 2) == S.tpipe_slots(p, m)


@pytest.mark.parametrize("v", [3, 4])
@pytest.mark.parametrize("p", list(range(1, 17)))
def test_slots_collision_free_and_makespan(v, p):
    for m in (1, p, 2 * p + 1, 4 * p):
        sl = S.tpipe_slots(p, m, v)
        for s in range(p):
            ts = [t for (ss, _k, _c, _i), t in sl.items() if ss == s]
            assert len(set(ts)) == len(ts)
        mk = S.simulate(S.tpipe_orders(p, m, v=v), p, v)["makespan"]
        if p >= 4:
            assert mk == 3 * v * (m + p - 1)
        else:
            assert abs(mk - 3 * v * (m + p - 1)) <= 3 * v


@pytest.mark.parametrize("v", [3, 4])
@pytest.mark.parametrize("p", [2, 3, 4, 8, 16])
def test_send_window_v(v, p):
    d = T.ModelDesc(2 * v * p, 64, 4, 256, 256, 32, 2, T.BF16)
    for strat in ("tpipe", "tpipe_trecomp", "interleave", "interleave_trecomp"):
        st, _ = T.build_streams(d, p, 4 * p, strat, chunks=v)          # default W = v
        assert T.deadlock_free(st) and T.fifo_consistent(st)
    orders = S.tpipe_orders(p, 4 * p, v=v)
    assert S.simulate(orders, p, v, window=v)["makespan"] == S.simulate(orders, p, v)["makespan"]
    if v == 4:
        st, _ = T.build_streams(d, p, 4 * p, "tpipe", chunks=v, window=2)
        assert not T.deadlock_free(st)


@pytest.mark.parametrize("v,frac", [(2, 1 / 3), (3, 4 / 9), (4, 1 / 2)])
def test_multichunk_offload_fraction(v, frac):
    p = 4
    d = T.ModelDesc(4 * v * p, 64, 4, 256, 256, 32, 2, T.BF16)
    s = 1                                      # a middle stage: equal chunks, no emb / head
    full = sum(T.model_state_bytes(d, T.chunk_params(d, p, v, s, c), False) for c in range(1, v + 1))
    off = sum(T.model_state_bytes(d, T.chunk_params(d, p, v, s, c), c >= 2) for c in range(1, v + 1))
    assert (full - off) / full == pytest.approx(frac, rel=1e-12)


def oracle_ops(st):
    return [dict(kind=i.kind, chunk=i.chunk, mb=i.mb, peer=i.peer, channel=tuple(i.channel),
                 msg=i.msg) for i in st]


def _plan_mod():
    from paper_2503_03182_b200 import plan
    return plan


CASES = [(st, v, p, off) for v in (3, 4) for p in (1, 2, 4)
         for st, off in (("tpipe", 0), ("tpipe_trecomp", 0), ("interleave", 0), ("interleave_trecomp", 0),
                         ("tpipe", 1), ("tpipe_trecomp", 5))]


@pytest.mark.parametrize("strategy,v,p,offload", CASES)
def test_planner_multichunk_streams_match_oracle(strategy, v, p, offload):
    P = _plan_mod()
    L = 2 * v * p
    m = 2 * p
    od = T.ModelDesc(L, 64, 4, 256, 256, 32, 2, T.BF16)
    pd = P.Model(L, 64, 4, 256, 256, 32, 2, P.BF16)
    plan = P.Plan(pd, p, m, strategy=strategy, chunks=v, offload=offload)
    assert plan.v == v and plan.W == max(2, v)
    assert all(len(x) == v and sum(x) == 2 * v for x in plan.partition)
    st, static = T.build_streams(od, p, m, strategy, chunks=v, offload_model_state=bool(offload & 1),
                                 offload_device_opt=bool(offload & 4))
    for s in range(p):
        got, bufs = plan.ops(s)
        strip = [{k: o[k] for k in ("kind", "chunk", "mb", "peer", "channel", "msg")} for o in got]
        assert strip == oracle_ops(st[s])
        rep = T.replay(st[s], static[s])
        pk = plan.peak(s)
        for cat in ("model_state", "io", "act", "recomp_buf", "comm", "workspace"):
            assert pk[cat] == rep.get(cat, 0), cat
        for c in range(1, v + 1):
            assert plan.chunk_params(s, c) == T.chunk_params(od, p, v, s, c)
