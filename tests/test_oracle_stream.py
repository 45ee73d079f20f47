"""Pins for the oracle's byte-level instruction streams (oracle/stream.py)."""

import pytest

from oracle import schedule as S
from oracle import stream as T

C1 = T.ModelDesc(8, 64, 4, 256, 256, 32, 2, T.BF16)


def desc(L, dtype=T.BF16):
    return T.ModelDesc(L, 64, 4, 256, 256, 32, 2, dtype)


@pytest.mark.parametrize("strategy", ["tpipe", "tpipe_trecomp", "1f1b", "1f1b_full_recomp",
                                      "interleave", "interleave_trecomp"])
@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_stream_invariants(strategy, p):
    """Deadlock-free with W=2 (static acyclicity, D-14), channel FIFO
    consistency, every transient byte released at step end."""
    d = desc(2 * p if p > 4 else 8)
    st, static = T.build_streams(d, p, 8, strategy)
    assert T.deadlock_free(st)
    assert T.fifo_consistent(st)
    for s in range(p):
        r = T.replay(st[s], static[s])
        assert r["final"] == sum(b for _n, _c, b in static[s])


def test_send_window_one_deadlocks_trecomp_p8():
    """SURVEY D-14: W=1 deadlocks T-Recomp at p=8 (k=1); W=2 does not."""
    d = desc(16)
    st, _ = T.build_streams(d, 8, 32, "tpipe_trecomp", window=1)
    assert not T.deadlock_free(st)
    st, _ = T.build_streams(d, 8, 32, "tpipe_trecomp", window=2)
    assert T.deadlock_free(st)


@pytest.mark.parametrize("p", [4, 8])
def test_bytes_match_blocks(p):
    """The byte replay of a middle stage's activations (stash + chunk input)
    equals the block replay (P:611 blocks) times the per-chunk stash bytes."""
    d = desc(2 * p)                       # one layer per chunk
    m = 4 * p
    st, static = T.build_streams(d, p, m, "tpipe")
    z = T.sizes(d, p, 2, 1, 1)
    block_bytes = z["stash"] + z["act"]
    orders = S.tpipe_orders(p, m)
    for s in range(1, p - 1):
        r = T.replay(st[s], static[s])
        _pk, tot = S.block_replay(orders[s], "tpipe")
        assert r["act"] == tot * block_bytes


def test_model_state_offload_one_third():
    """T-Offload of chunk 2 (of 2) cuts model-state memory by 33.33%:
    12 of 18 B/param move to host for half the params (SURVEY D-8)."""
    d = desc(16)
    P1 = T.chunk_params(d, 8, 2, 3, 1)
    P2 = T.chunk_params(d, 8, 2, 3, 2)
    assert P1 == P2
    full = T.model_state_bytes(d, P1, False) + T.model_state_bytes(d, P2, False)
    off = T.model_state_bytes(d, P1, False) + T.model_state_bytes(d, P2, True)
    assert (full - off) * 3 == full


def test_trecomp_bytes_below_tpipe():
    """T-Recomp's stage-0 peak bytes are below T-Pipe's."""
    d = desc(16)
    a = T.replay(*[x[0] for x in T.build_streams(d, 8, 32, "tpipe")])
    b = T.replay(*[x[0] for x in T.build_streams(d, 8, 32, "tpipe_trecomp")])
    assert b["total_peak"] < a["total_peak"]


# ---------------------------------------------------------------- partial T-Recomp (R25)
def _kept_live_count(order, upto):
    """Chunk-1 micro-batches whose forward has started and whose backward has
    not ended after the first `upto` compute ops of the stage's order (the
    P:611 lifespan F(1,i) start -> B(1,i) end), counted from the schedule."""
    started = {op[2] for op in order[:upto] if op[0] == "F" and op[1] == 1}
    ended = {op[2] for op in order[:upto] if op[0] == "B" and op[1] == 1}
    return len(started - ended)


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("n", [4, 6])
def test_partial_trecomp_kept_stash_follows_schedule(p, n):
    """Partial T-Recomp of r of the n1 chunk-1 layers: after every compute op
    of the T-Recomp order (oracle.schedule, independent of the stream
    builder), the live kept-stash bytes equal (n1 - r) x per-layer stash x the
    number of chunk-1 micro-batches inside their F -> B lifespan, and the
    recompute buffer holds at most one micro-batch's r layers (P:666's one
    buffer block)."""
    d = desc(n * p)
    n1 = T.layers_per_chunk(d, p, 2)[0]
    m = 2 * p + 1
    orders = S.strategy_orders("tpipe_trecomp", p, m)[0]
    for r in range(1, n1):
        st, _static = T.build_streams(d, p, m, "tpipe_trecomp", recomp_layers=r)
        for s in range(p):
            z = T.sizes(d, p, 2, s, 1)
            keep, rec = T.partial_trecomp_split(z, n1, r)
            assert keep == (n1 - r) * z["layer_stash"] and keep + rec == z["stash"]
            live = {}
            k = 0
            for ins in st[s]:
                for name, _cat, b in ins.allocs:
                    live[name] = b
                if ins.kind in ("F", "B", "R"):
                    k += 1
                    kept = sum(b for nm, b in live.items() if nm[0] == "STASH" and nm[1] == 1)
                    rbuf = [b for nm, b in live.items() if nm[0] == "RBUF"]
                    assert kept == keep * _kept_live_count(orders[s], k - (ins.kind == "B"))
                    assert len(rbuf) <= 1 and all(b == rec for b in rbuf)
                for name in ins.frees:
                    live.pop(name)


@pytest.mark.parametrize("p", [1, 4, 8])
def test_partial_trecomp_endpoints(p):
    """r = n1 is exactly block-wise T-Recomp; peaks are non-increasing in r,
    and r = 1 already stores less than plain T-Pipe whenever more than one
    chunk-1 block is in flight (m >= 2p)."""
    d = desc(6 * p)
    n1 = T.layers_per_chunk(d, p, 2)[0]
    m = 4 * p
    full, fst = T.build_streams(d, p, m, "tpipe_trecomp")
    same, sst = T.build_streams(d, p, m, "tpipe_trecomp", recomp_layers=n1)
    assert [[(i.key(), i.allocs, i.frees) for i in x] for x in full] == \
        [[(i.key(), i.allocs, i.frees) for i in x] for x in same]
    tp, tst = T.build_streams(d, p, m, "tpipe")
    for s in range(p):
        pk = [T.replay(*[x[s] for x in T.build_streams(d, p, m, "tpipe_trecomp", recomp_layers=r)])
              ["total_peak"] for r in range(1, n1 + 1)]
        assert pk == sorted(pk, reverse=True)
        if p > 1:
            assert pk[0] < T.replay(tp[s], tst[s])["total_peak"]
    with pytest.raises(ValueError):
        T.build_streams(d, p, m, "tpipe_trecomp", recomp_layers=n1 + 1)


@pytest.mark.parametrize("p", [4, 8])
def test_interleave_bytes_match_blocks(p):
    """Interleave-1F1B byte replay of a middle stage's activations equals the
    block replay (P:210 pin m_a(1 + (p-1)/(pv)) lives there) times the
    per-chunk stash + input bytes; with T-Recomp the chunk-2 blocks plus the
    one recompute buffer match the (p+1)-block D-9 count."""
    d = desc(2 * p)
    m = 2 * p
    z = T.sizes(d, p, 2, 1, 1)
    st, static = T.build_streams(d, p, m, "interleave")
    orders = S.interleave_orders(p, m, 2)
    for s in range(1, p - 1):
        r = T.replay(st[s], static[s])
        _pk, tot = S.block_replay(orders[s], "interleave")
        assert r["act"] == tot * (z["stash"] + z["act"])
    st, static = T.build_streams(d, p, m, "interleave_trecomp")
    orders = S.strategy_orders("interleave_trecomp", p, m)[0]
    for s in range(1, p - 1):
        r = T.replay(st[s], static[s])
        pk, _tot = S.block_replay(orders[s], "tpipe_trecomp")
        assert r["recomp_buf"] == pk["buf"] * z["stash"]
