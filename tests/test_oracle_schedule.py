"""Pins for oracle Part 1 (schedule simulator) against the paper's closed forms,
independently derived golden vectors and brute force. CPU only.

Each test cites the PAPER.md line (P:n) whose statement it checks.
"""

import itertools
import math
import os
from fractions import Fraction

import pytest

from oracle import schedule as S

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def run(strategy, p, m, k=None, window=None):
    orders, v, rec, dur = S.strategy_orders(strategy, p, m, k=k)
    sim = S.simulate(orders, p, v, dur, rec, window=window)
    return orders, sim


def cdiv(a, b):
    return -((-a) // b)


# ------------------------------------------------------------- T-Pipe (App. A)
@pytest.mark.parametrize("p", list(range(1, 17)) + [24, 40])
def test_tpipe_makespan_and_bubble(p):
    """warmup 2p + steady 6(m-1) + cooldown 4p = 6(m+p-1) T_unit;
    bubble 6(p-1) per stage -> ratio (p-1)/(m+p-1)."""
    for m in sorted({1, 2, max(1, p // 2), p, 2 * p} if p <= 16 else {2 * p}):
        orders, sim = run("tpipe", p, m)
        assert sim["makespan"] == 6 * (m + p - 1)
        for s in range(p):
            busy = sum(sim["end"][(s, op)] - sim["start"][(s, op)] for op in orders[s])
            assert busy == 6 * m
            bubble = Fraction(sim["makespan"] - busy, sim["makespan"])
            assert bubble == Fraction(p - 1, m + p - 1)


@pytest.mark.parametrize("p", range(3, 41))
def test_tpipe_stage0_chunk_peaks(p):
    """stage-0 peak blocks ceil(2/3 + a + b + p/2) (chunk 1) and
    ceil((3p-2)/6) (chunk 2), a=ceil((p-3)/6), b=ceil((2p-3)/6); steady state
    (m = 2p)."""
    a, b = cdiv(p - 3, 6), cdiv(2 * p - 3, 6)
    want_c1 = math.ceil(Fraction(2, 3) + a + b + Fraction(p, 2))
    want_c2 = cdiv(3 * p - 2, 6)
    orders = S.tpipe_orders(p, 2 * p)
    peaks, _tot = S.block_replay(orders[0], "tpipe")
    assert (peaks["c1"], peaks["c2"]) == (want_c1, want_c2)


@pytest.mark.parametrize("p", [3, 4, 5, 6, 7, 8, 9, 12, 16, 24])
def test_tpipe_intervals(p):
    """T_fwd_interval = (3 + 6 ceil((p-3)/6) - p) T_unit between the
    chunk-1 forward end (stage p-1) and chunk-2 forward start (stage 0);
    T_bwd_interval = (3 + 6 ceil((2p-3)/6) - 2p) between chunk-2 backward end
    (stage 0) and chunk-1 backward start (stage p-1). Steady state, m = 4p."""
    m = 4 * p
    _o, sim = run("tpipe", p, m)
    i = 2 * p
    a, b = cdiv(p - 3, 6), cdiv(2 * p - 3, 6)
    fwd = sim["start"][(0, ("F", 2, i))] - sim["end"][(p - 1, ("F", 1, i))]
    bwd = sim["start"][(p - 1, ("B", 1, i))] - sim["end"][(0, ("B", 2, i))]
    assert fwd == 3 + 6 * a - p
    assert bwd == 3 + 6 * b - 2 * p


@pytest.mark.parametrize("p", [3, 4, 5, 6, 8, 9, 12, 16])
def test_tpipe_lifespan_chunk2(p):
    """T_life_chunk2 = T_fwd_chunk2 + T_bwd_chunk2 - 2 T_unit = 3p-2
    (stage 0, F(0,2,i) start -> B(0,2,i) start), steady state (m = 4p,
    i = 2p+1: at p = 5 the warmup transient lasts ~p microbatches)."""
    _o, sim = run("tpipe", p, 4 * p)
    i = 2 * p + 1
    life = sim["start"][(0, ("B", 2, i))] - sim["start"][(0, ("F", 2, i))]
    assert life == 3 * p - 2


@pytest.mark.parametrize("p", [2, 3, 4, 5, 6, 8, 9, 12, 16])
def test_offload_windows_eq5_eq7(p):
    """App. D: Eq. 5 cooldown window (p - ceil((2p-3)/6) - 1) T_bwd/(2p)
    = 2(p-b-1) T_unit idle between B(s,2,m) end and B(s,1,m) start; Eq. 7
     warmup window (p - ceil((p-3)/6) - 1) T_fwd/(2p) idle between
    F(s,1,1) end and F(s,2,1) start. Checked at every stage."""
    m = 2 * p
    _o, sim = run("tpipe", p, m)
    a, b = cdiv(p - 3, 6), cdiv(2 * p - 3, 6)
    for s in range(p):
        w5 = S.idle_between(sim, s, sim["end"][(s, ("B", 2, m))], sim["start"][(s, ("B", 1, m))])
        w7 = S.idle_between(sim, s, sim["end"][(s, ("F", 1, 1))], sim["start"][(s, ("F", 2, 1))])
        assert w5 == max(0, 2 * (p - b - 1))
        assert w7 == p - a - 1


def test_tpipe_75_percent_limit():
    """T-Pipe peak activation -> 75% m_a for large p
    (SPEC S:392 asks p=120 within (0.74, 0.78))."""
    for p in (40, 120):
        orders = S.tpipe_orders(p, 2 * p)
        _peaks, tot = S.block_replay(orders[0], "tpipe")
        frac = tot / (2 * p)
        assert 0.74 < frac < 0.78, (p, frac)


def test_golden_tpipe_p4_m8():
    """Independent survey-session vector G-1 (tests/golden/tpipe_p4_m8.txt)."""
    gold = {}
    for line in open(os.path.join(GOLD, "tpipe_p4_m8.txt")):
        if line.startswith("#") or not line.strip():
            continue
        k, v = line.split(":", 1)
        gold[k.strip()] = v.split()
    orders, sim = run("tpipe", 4, 8)
    for s in (0, 3):
        got = [f"{op[0]}{op[1]}.{op[2]}@{sim['start'][(s, op)]}" for op in orders[s]]
        assert got == gold[f"stage{s}"]
    assert sim["makespan"] == int(gold["makespan"][0])
    for s, want in enumerate(gold["peaks"]):
        pk, tot = S.block_replay(orders[s], "tpipe")
        assert (pk["c1"], pk["c2"], tot) == tuple(int(x) for x in want.split(","))


# ------------------------------------------------------------- T-Recomp (App. B/C)
@pytest.mark.parametrize("p", list(range(3, 18)) + [24, 27, 32, 40, 41])
def test_trecomp_appendix_c(p):
    """App. C: chunk-2 lifespan (3p + ceil((p-1)/2) - 2) T_unit, steady
    period 7 T_unit, stage-0 total = floor(p/2) + 1 blocks incl. the
    recompute buffer, makespan <= [6p + 7(m-1)] T_unit."""
    m = 4 * p
    orders, sim = run("tpipe_trecomp", p, m)
    i = 2 * p + 1                       # steady state
    life = sim["start"][(0, ("B", 2, i))] - sim["start"][(0, ("F", 2, i))]
    assert life == 3 * p + cdiv(p - 1, 2) - 2
    assert sim["start"][(0, ("F", 2, i + 1))] - sim["start"][(0, ("F", 2, i))] == 7
    pk, tot = S.block_replay(orders[0], "tpipe_trecomp")
    assert tot == p // 2 + 1
    assert pk["buf"] == 1
    assert sim["makespan"] <= 6 * p + 7 * (m - 1)
    # no deep-layer penalty: chunk-2 peak never exceeds T-Pipe's
    pk0, _ = S.block_replay(S.tpipe_orders(p, m)[0], "tpipe")
    assert pk["c2"] <= pk0["c2"]


@pytest.mark.parametrize("p", list(range(3, 18)) + [24, 27, 32, 36, 40, 41])
def test_delay_rounds_minimal(p):
    """App. B: the printed constraint's k removes the inter-chunk
    conflict (lifespan equals App. C, no backward waits), and k-1 does not.
    (The prose 'k=1 for 8<=p<=40', disagrees: DESIGN.md R3.)"""
    k = S.delay_rounds(p)
    m = 4 * p
    i = 2 * p + 1
    formula = 3 * p + cdiv(p - 1, 2) - 2
    _o, sim = run("tpipe_trecomp", p, m, k=k)
    life = sim["start"][(0, ("B", 2, i))] - sim["start"][(0, ("F", 2, i))]
    assert life == formula
    if k >= 1:
        _o2, sim2 = run("tpipe_trecomp", p, m, k=k - 1)
        life2 = sim2["start"][(0, ("B", 2, i))] - sim2["start"][(0, ("F", 2, i))]
        assert life2 > formula or sim2["makespan"] > sim["makespan"]


def test_delay_rounds_values():
    """P:643-652 evaluated by hand (SURVEY D-3 table)."""
    table = {3: 0, 7: 0, 8: 1, 9: 1, 10: 0, 12: 0, 13: 1, 16: 0, 17: 0, 18: 1,
             26: 1, 27: 2, 31: 1, 32: 2, 33: 2, 35: 1, 36: 2, 39: 2, 40: 1, 41: 2}
    for p, k in table.items():
        assert S.delay_rounds(p) == k, p


def test_golden_trecomp_p4_m8():
    """Independent survey-session vector G-2 (tests/golden/trecomp_p4_m8.txt)."""
    orders, sim = run("tpipe_trecomp", 4, 8)
    got = [f"{op[0]}{op[1]}.{op[2]}@{sim['start'][(0, op)]}" for op in orders[0]]
    excerpt = "F2.4@22 R1.1@23 B1.1@24 F1.6@26 B2.3@27".split()
    j = got.index(excerpt[0])
    assert got[j:j + len(excerpt)] == excerpt
    assert sim["makespan"] == 71
    pk, tot = S.block_replay(orders[0], "tpipe_trecomp")
    assert (pk["c2"], pk["buf"], tot) == (2, 1, 3)
    totals = [S.block_replay(orders[s], "tpipe_trecomp")[1] for s in range(4)]
    ck = [S.block_replay(orders[s], "tpipe_trecomp")[0]["ckpt"] for s in range(4)]
    assert totals == [3, 2, 2, 1] and ck == [5, 5, 4, 4]


def test_fig8a_activation_ratio():
    """T-Recomp cuts activation 16.61 GB -> 6.39 GB at PP8; the unit
    model's stage-0 ratio is 5/13 (SURVEY D-8)."""
    _p1, t1 = S.block_replay(S.tpipe_orders(8, 32)[0], "tpipe")
    _p2, t2 = S.block_replay(S.tpipe_orders(8, 32, recomp=True)[0], "tpipe_trecomp")
    assert (t1, t2) == (13, 5)
    assert abs(t2 / t1 - 6.39 / 16.61) < 0.002


@pytest.mark.parametrize("p", [4, 8, 16])
def test_layer_grouped_trecomp_is_worse(p):
    """P:343-345 / Fig. 6(b,c): recompute fused into B1 (layer-grouped) breaks
    the period: makespan strictly above block-wise T-Recomp."""
    m = 4 * p
    _o, lg = run("tpipe_layer_grouped", p, m)
    _o, bw = run("tpipe_trecomp", p, m)
    assert lg["makespan"] > bw["makespan"]
    assert lg["makespan"] > 6 * p + 7 * (m - 1)


# ------------------------------------------------------------- baselines
@pytest.mark.parametrize("p", [1, 2, 3, 4, 8])
def test_1f1b(p):
    """1F1B stage-s peak (p-s) m_a/p, i.e. 2(p-s) blocks of m_a/(2p),
    makespan 6(m+p-1); 1F1B+R=50% takes 7(m-1+p) T_unit; full layer-
    grouped recompute 8(m+p-1)."""
    for m in (p, 2 * p, 4 * p):
        orders, sim = run("1f1b", p, m)
        assert sim["makespan"] == 6 * (m + p - 1)
        for s in range(p):
            _pk, tot = S.block_replay(orders[s], "1f1b")
            assert tot == 2 * (p - s)
        _o, r50 = run("1f1b_r50", p, m)
        assert r50["makespan"] == 7 * (m + p - 1)
        _o, full = run("1f1b_full_recomp", p, m)
        assert full["makespan"] == 8 * (m + p - 1)


@pytest.mark.parametrize("p", [2, 4, 8])
def test_interleave(p):
    """Interleave-1F1B (v chunks) peak activation m_a(1 + (p-1)/(pv))
    at stage 0 and bubble 1/v of 1F1B's."""
    for v in (2, 3):
        m = 2 * p
        orders = S.interleave_orders(p, m, v)
        dur = {"F": 1, "B": 2, "R": 1}           # T_unit = T_fwd/(vp)
        sim = S.simulate(orders, p, v, dur)
        busy = 3 * v * m
        onef1b_bubble = 3 * v * (p - 1)           # (p-1)(T_fwd+T_bwd)/p in these units
        assert sim["makespan"] - busy == Fraction(onef1b_bubble, v)
        _pk, tot = S.block_replay(orders[0], "interleave")
        assert Fraction(tot, v * p) == 1 + Fraction(p - 1, p * v)


# ------------------------------------------------------------- invariants
@pytest.mark.parametrize("strategy", ["tpipe", "tpipe_trecomp", "1f1b"])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 8, 16])
def test_invariants(strategy, p):
    """|F| = |B| = p v m; every channel FIFO-consistent (D-14)."""
    m = 2 * p
    orders, v, _r, _d = S.strategy_orders(strategy, p, m)
    nF = sum(1 for o in orders for op in o if op[0] == "F")
    nB = sum(1 for o in orders for op in o if op[0] == "B")
    assert nF == nB == p * v * m
    for ch, (snd, rcv) in S.channel_sequences(orders, p, v).items():
        assert snd == rcv, ch


def test_send_window():
    """SURVEY D-14: W=1 deadlocks T-Recomp at p=8 (k=1); W=2 is deadlock-free
    and reaches the unconstrained makespan for p <= 16."""
    with pytest.raises(S.Deadlock):
        run("tpipe_trecomp", 8, 32, window=1)
    for p in range(3, 17):
        for strat in ("tpipe", "tpipe_trecomp"):
            _o, free = run(strat, p, 2 * p)
            _o, w2 = run(strat, p, 2 * p, window=2)
            assert w2["makespan"] == free["makespan"], (strat, p)


def test_random_durations_deadlock_free():
    """SURVEY D-16: with W=2 the orders execute under arbitrary positive
    durations (no deadlock), and block peaks are duration-independent by
    construction of the replay."""
    import random
    rng = random.Random(7)
    for p in (4, 8):
        for strat in ("tpipe", "tpipe_trecomp"):
            orders, v, rec, _d = S.strategy_orders(strat, p, 4 * p)
            for _ in range(5):
                table = {}

                def dur(s, op, table=table):
                    return table.setdefault((s, op), rng.randint(1, 9))
                S.simulate(orders, p, v, dur, rec, window=2)


# ------------------------------------------------------------- brute force (D-10)
def _longest_path_makespan(orders, p, v, dur):
    """Independent recount: ASAP start = longest path in the DAG of program
    order + data edges (topological order by repeated relaxation)."""
    nodes = [(s, op) for s in range(p) for op in orders[s]]
    preds = {n: [] for n in nodes}
    for s in range(p):
        for a, b in zip(orders[s], orders[s][1:]):
            preds[(s, b)].append((s, a))
    for (s, op) in nodes:
        preds[(s, op)] += S.data_deps(s, op, p, v, False)
    finish = {}

    def f(n):
        if n not in finish:
            finish[n] = max([f(x) for x in preds[n]] + [0]) + dur[n[1][0]]
        return finish[n]
    return max(f(n) for n in nodes)


def _all_orders(p, m, v):
    """Every per-stage order that is FIFO per (kind, chunk) and respects the
    same-stage deps (SURVEY D-10: 14 per stage at m=2, 196 / 2,744 combos)."""
    def stage_orders():
        kinds = [("F", c) for c in range(1, v + 1)] + [("B", c) for c in range(1, v + 1)]
        seqs = []

        def rec(cnt, seq):
            if len(seq) == 2 * v * m:
                seqs.append(list(seq))
                return
            for kd in kinds:
                i = cnt[kd] + 1
                if i > m:
                    continue
                if kd[0] == "B" and cnt[("F", kd[1])] < i:
                    continue
                # chain F1(i) < F2(i) < B2(i) < B1(i): any other same-stage
                # order is a transitive self-dependency (deadlock)
                if kd[0] == "F" and kd[1] > 1 and cnt[("F", kd[1] - 1)] < i:
                    continue
                if kd[0] == "B" and kd[1] < v and cnt[("B", kd[1] + 1)] < i:
                    continue
                cnt[kd] += 1
                seq.append((kd[0], kd[1], i))
                rec(cnt, seq)
                seq.pop()
                cnt[kd] -= 1
        rec({kd: 0 for kd in kinds}, [])
        return seqs
    per = stage_orders()
    return itertools.product(per, repeat=p)


@pytest.mark.parametrize("p,m,want_min", [(2, 2, 15), (3, 2, 21), (2, 3, 21)])
def test_brute_force(p, m, want_min):
    """SURVEY D-10: over all FIFO per-stage orders (v=2, F=1, B=2) the
    simulator agrees with an independent longest-path recount; the minimum
    makespan is 15 / 21; T-Pipe reaches 6(m+p-1), not claimed optimal."""
    v = 2
    dur = {"F": 1, "B": 2}
    best = None
    n = 0
    for orders in _all_orders(p, m, v):
        orders = list(orders)
        try:
            sim = S.simulate(orders, p, v, dur)
        except S.Deadlock:
            continue
        n += 1
        assert sim["makespan"] == _longest_path_makespan(orders, p, v, dur)
        best = sim["makespan"] if best is None else min(best, sim["makespan"])
    assert best == want_min
    assert n > 0
    tp = S.simulate(S.tpipe_orders(p, m), p, v, dur)["makespan"]
    assert tp == 6 * (m + p - 1) and tp >= best


@pytest.mark.parametrize("p", [2, 3, 4, 8, 16])
def test_interleave_trecomp_d9(p):
    """P:367 / SURVEY D-9: Interleave-1F1B + block-wise T-Recomp of chunk 1
    holds (p+1) blocks = (p+1)/(2p) m_a at stage 0 (-> 50%, vs plain
    interleave's m_a(1 + (p-1)/(2p))); at p=8, m=16 its unit-model makespan is
    133 vs 7(m+p-1) = 161 for 1F1B + 50% layer recompute."""
    m = 2 * p
    orders, v, rec, dur = S.strategy_orders("interleave_trecomp", p, m)
    assert v == 2 and rec
    for s in range(p):
        lst = orders[s]
        assert sum(op[0] == "R" for op in lst) == m
        for n, op in enumerate(lst):
            if op[0] == "B" and op[1] == 1:
                assert lst[n - 1] == ("R", 1, op[2])
    _pk, tot = S.block_replay(orders[0], "tpipe_trecomp")
    assert Fraction(tot, 2 * p) == Fraction(p + 1, 2 * p)
    sim = S.simulate(orders, p, v, dur, rec)
    if p == 8:
        assert sim["makespan"] == 133
        r50 = S.simulate(*[S.strategy_orders("1f1b_r50", p, m)[i] for i in (0,)], p, 1,
                         S.strategy_orders("1f1b_r50", p, m)[3])
        assert r50["makespan"] == 7 * (m + p - 1) == 161
