"""Oracle Part 1 — exact integer unit-time pipeline schedule simulator.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``). Shares no code with the
C++ planner in ``paper_2503_03182_b200/csrc/plan``.

Unit model (Appendix A): T_bwd = 2 T_fwd, T_unit = T_fwd/(2p),
one chunk-task activation block = m_a/(2p). At v=2 a chunk forward F lasts 1
T_unit, a chunk backward B lasts 2, a block-wise recompute R lasts 1.
At v=1 (1F1B) a stage holds two blocks' worth of layers: F=2, B=4.

Ops are tuples ``(kind, chunk, mb)`` with kind in {'F','B','R'}, chunk 1..v
(1 = shallow), mb 1..m. Stage s owns global layer block (c-1)p+s for chunk c
(P:210 layout, reused by T-Pipe P:306).

Schedules
---------
* T-Pipe (Fig. 5 is unreadable, App. A P:611-636 gives only closed
  forms). Reading (R1): a closed-form slot table,
  each stage executes its ops sorted by slot time, ASAP under data deps.
* T-Recomp block-wise (Fig. 6(d); App. C). Reading (D-2, R2):
  insert R(s,1,i) immediately before B(s,1,i); chunk-1 stash released at F end,
  its input kept as checkpoint; one recompute buffer block live R start ->
  B end; chunk 2 delayed k rounds with k from App. B as printed
  (``delay_rounds``), NOT the prose "k=1 for 8<=p<=40".
* 1F1B (DAPPLE): warmup min(p-s-1, m) forwards, then 1F1B, then drain.
* 1F1B + layer-grouped recompute ratio R: B grows by
  R*F (full: B=6, R=50%: B=5).
* T-Pipe + layer-grouped T-Recomp (the paper's NEGATIVE design, P:343-345,
  Fig. 6(b)): recompute fused into B(s,1,i) (B1 = 3).
* Interleave-1F1B (Megatron virtual pipeline), for the paper's
  m_a(1+(p-1)/(pv)) and bubble/v statements.
* Interleave-1F1B + T-Recomp (Fig. 6(e)):
  the interleave order with R(s,1,i) inserted immediately before B(s,1,i),
  chunk 1 (the chunk with the poorest temporal locality) recomputed
  block-wise exactly as in T-Recomp (R26).
"""

from __future__ import annotations

from collections import defaultdict


class Deadlock(RuntimeError):
    """No stage can make progress (SPEC S:331 'DeadlockError')."""


def cdiv(n: int, d: int) -> int:
    """Ceiling division for possibly negative integers (App. A uses ceil of
    (p-3)/6, negative for p<3)."""
    return -((-n) // d)


def tpipe_ab(p: int):
    """a = ceil((p-3)/6), b = ceil((2p-3)/6): App. A interval terms."""
    return cdiv(p - 3, 6), cdiv(2 * p - 3, 6)


def delay_rounds(p: int) -> int:
    """Appendix B, as printed: min k in N with
    T_fwd_interval - dT_fwd_interval + 7k >= 0, where
    T_fwd_interval = 3 + 6 ceil((p-3)/6) - p
    dT_fwd_interval = ceil((p-1)/2) - ceil((p-3)/6) - 1.
    Defined for p >= 3; below that there is no conflict and k = 0."""
    if p < 3:
        return 0
    a = cdiv(p - 3, 6)
    fwd_interval = 3 + 6 * a - p
    delta = cdiv(p - 1, 2) - a - 1
    k = 0
    while fwd_interval - delta + 7 * k < 0:
        k += 1
    return k


# --------------------------------------------------------------------------
# Per-stage orders
# --------------------------------------------------------------------------

def tpipe_slots(p: int, m: int, v: int = 2) -> dict:
    """D-1 slot table; keys (stage, kind, chunk, mb).

    v > 2 (D-11's generalisation, DESIGN R32): the slot period
    per micro-batch is 3v units;
      F(s,1,i)   = 3v(i-1) + s
      F(0,c+1,i) = the first t >= F(0,c,i) + p with t = 3c (mod 3v)
      B(0,v,i)   = F(0,v,i) + 3p - 2          (= F(p-1,v,i) + 1 + 2(p-1))
      B(0,c-1,i) = the first t >= B(0,c,i) + 2p with t = B(0,c,i) + 3 (mod 3v)
      F(s,c,i)   = F(0,c,i) + s,   B(s,c,i) = B(0,c,i) - 2s.
    At v = 2 this is exactly D-1 (a = ceil((p-3)/6), b = ceil((2p-3)/6))."""
    if v == 2:
        a, b = tpipe_ab(p)
        t = {}
        for i in range(1, m + 1):
            for s in range(p):
                t[(s, "F", 1, i)] = 6 * (i - 1) + s
                t[(s, "F", 2, i)] = 6 * (i - 1) + 3 + 6 * a + s
            for s in range(p):
                t[(s, "B", 2, i)] = t[(p - 1, "F", 2, i)] + 1 + 2 * (p - 1 - s)
            for s in range(p):
                t[(s, "B", 1, i)] = t[(0, "B", 2, i)] + 3 + 6 * b - 2 * s
        return t
    return tpipe_slots_general(p, m, v)


def tpipe_slots_general(p: int, m: int, v: int) -> dict:
    """The period-3v slot table of tpipe_slots for any v >= 1 (written from
    the recurrences, not from D-1's closed form; equal to it at v = 2)."""
    per = 3 * v

    def first_at_least(lo, residue):
        return lo + ((residue - lo) % per)

    t = {}
    for i in range(1, m + 1):
        f0 = {1: per * (i - 1)}
        for ch in range(1, v):
            f0[ch + 1] = first_at_least(f0[ch] + p, 3 * ch)
        b0 = {v: f0[v] + 3 * p - 2}
        for ch in range(v, 1, -1):
            b0[ch - 1] = first_at_least(b0[ch] + 2 * p, b0[ch] + 3)
        for s in range(p):
            for ch in range(1, v + 1):
                t[(s, "F", ch, i)] = f0[ch] + s
                t[(s, "B", ch, i)] = b0[ch] - 2 * s
    return t


def tpipe_orders(p: int, m: int, recomp: bool = False, k: int | None = None,
                 layer_grouped: bool = False, v: int = 2):
    """T-Pipe per-stage compute order (v=2).

    recomp=True: block-wise T-Recomp (R before each B1, chunk-1 forwards run k
    microbatches ahead == chunk 2 delayed k rounds).
    layer_grouped=True: the negative design (recompute fused into B1, no R op,
    no delay) for P:345's dependency conflict.
    """
    slots = tpipe_slots(p, m, v)
    if recomp and k is None:
        # App. B's delay analysis is for two chunks; v > 2 runs undelayed (R32)
        k = delay_rounds(p) if v == 2 else 0
    if not recomp:
        k = 0
    orders = []
    for s in range(p):
        ops = sorted((t, kind, c, i) for (ss, kind, c, i), t in slots.items() if ss == s)
        lst = [(kind, c, i) for (_, kind, c, i) in ops]
        assert len({t for (t, *_rest) in ops}) == len(ops), "slot collision"
        if k:
            relabeled = []
            n = 0
            for op in lst:
                if op[0] == "F" and op[1] == 1:
                    n += 1
                    if n + k <= m:
                        relabeled.append(("F", 1, n + k))
                else:
                    relabeled.append(op)
            lst = [("F", 1, i) for i in range(1, min(k, m) + 1)] + relabeled
        if recomp:
            out = []
            for op in lst:
                if op[0] == "B" and op[1] == 1:
                    out.append(("R", 1, op[2]))
                out.append(op)
            lst = out
        orders.append(lst)
    return orders


def onef1b_orders(p: int, m: int):
    """1F1B (DAPPLE): warmup min(p-s-1, m) forwards, steady 1F1B, drain."""
    orders = []
    for s in range(p):
        w = min(p - s - 1, m)
        lst = [("F", 1, i) for i in range(1, w + 1)]
        for i in range(1, m - w + 1):
            lst.append(("F", 1, w + i))
            lst.append(("B", 1, i))
        for i in range(m - w + 1, m + 1):
            lst.append(("B", 1, i))
        orders.append(lst)
    return orders


def interleave_trecomp_orders(p: int, m: int, v: int = 2):
    """Interleave-1F1B + block-wise T-Recomp of chunk 1 (DESIGN R26):
    R(s,1,i) right before each B(s,1,i) of the interleave order."""
    out = []
    for lst in interleave_orders(p, m, v):
        withr = []
        for op in lst:
            if op[0] == "B" and op[1] == 1:
                withr.append(("R", 1, op[2]))
            withr.append(op)
        out.append(withr)
    return out


def interleave_orders(p: int, m: int, v: int):
    """Interleave-1F1B (Megatron virtual pipeline). Requires m % p == 0.
    Virtual forward index q -> chunk (q mod pv)//p + 1, mb (q//(pv))p + q mod p + 1;
    backward chunk mirrored. Warmup 2(p-s-1) + (v-1)p virtual forwards."""
    assert m % p == 0
    total = m * v

    def f_op(q):
        return ("F", (q % (p * v)) // p + 1, (q // (p * v)) * p + q % p + 1)

    def b_op(q):
        return ("B", v - (q % (p * v)) // p, (q // (p * v)) * p + q % p + 1)

    orders = []
    for s in range(p):
        w = min(2 * (p - s - 1) + (v - 1) * p, total)
        lst = [f_op(q) for q in range(w)]
        for q in range(total - w):
            lst.append(f_op(w + q))
            lst.append(b_op(q))
        for q in range(total - w, total):
            lst.append(b_op(q))
        orders.append(lst)
    return orders


# --------------------------------------------------------------------------
# Dependencies, messages, simulation
# --------------------------------------------------------------------------

def data_deps(s: int, op, p: int, v: int, recomputed: bool):
    """Data-flow edges: F(s,c,i) <- F(s-1,c,i); F(0,c,i) <-
    F(p-1,c-1,i); B mirrors in reverse; B needs its own F (and R if any)."""
    kind, c, i = op
    if kind == "F":
        if s > 0:
            return [(s - 1, ("F", c, i))]
        if c > 1:
            return [(p - 1, ("F", c - 1, i))]
        return []
    if kind == "R":
        return [(s, ("F", c, i))]
    d = [(s, ("F", c, i))]
    if recomputed and c == 1:
        d.append((s, ("R", c, i)))
    if s < p - 1:
        d.append((s + 1, ("B", c, i)))
    elif c < v:
        d.append((0, ("B", c + 1, i)))
    return d


def message_of(s: int, op, p: int, v: int):
    """If op's output crosses stages, return (channel, dst_stage, consumer_op).
    Channels are FIFO per (kind, src, dst) (SURVEY §8(c) comm semantics):
    'A' = activations (forward), 'G' = activation grads (backward)."""
    kind, c, i = op
    if kind == "F":
        if s < p - 1:
            dst, cons = s + 1, ("F", c, i)
        elif c < v:
            dst, cons = 0, ("F", c + 1, i)
        else:
            return None
        ch = ("A", s, dst)
    elif kind == "B":
        if s > 0:
            dst, cons = s - 1, ("B", c, i)
        elif c > 1:
            dst, cons = p - 1, ("B", c - 1, i)
        else:
            return None
        ch = ("G", s, dst)
    else:
        return None
    if dst == s:          # p == 1: local hand-off, no channel
        return None
    return ch, dst, cons


def channel_sequences(orders, p: int, v: int):
    """Per channel: (sender production order, receiver consumption order)."""
    send = defaultdict(list)
    for s, lst in enumerate(orders):
        for op in lst:
            msg = message_of(s, op, p, v)
            if msg:
                ch, dst, cons = msg
                send[ch].append(cons[1:])  # (chunk, mb) of the message
    recv = defaultdict(list)
    for ch in send:
        _, src, dst = ch
        for op in orders[dst]:
            for dsrc, dop in data_deps(dst, op, p, v, False):
                if dsrc == src and dsrc != dst:
                    prod_msg = message_of(src, dop, p, v)
                    if prod_msg and prod_msg[0] == ch:
                        recv[ch].append(op[1:])
    return {ch: (send[ch], recv[ch]) for ch in send}


def default_durations(v: int, layer_grouped_b1: bool = False, b_extra: int = 0):
    if v == 1:
        return {"F": 2, "B": 4 + b_extra, "R": 2}
    return {"F": 1, "B": 2, "R": 1, "B1": 3 if layer_grouped_b1 else 2}


def simulate(orders, p: int, v: int, dur=None, recomputed: bool = False,
             window: int | None = None):
    """ASAP execution of fixed per-stage orders (SPEC S:308-372 'sim').

    Start(op) = max(stage free, end of data deps [+ start of window deps]).
    window=W adds the send-window edge (SURVEY D-14): the producer of message
    j+W on a channel may not start before the consumer of message j starts.
    ``dur`` maps kind -> units, or a callable (stage, op) -> units.
    Returns dict with 'start', 'end' ({(s, op): t}) and 'makespan'.
    Raises Deadlock if no stage can progress.
    """
    if dur is None:
        dur = default_durations(v)
    if callable(dur):
        dfun = dur
    else:
        def dfun(s, op):
            if op[0] == "B" and op[1] == 1 and "B1" in dur:
                return dur["B1"]
            return dur[op[0]]

    wdeps = defaultdict(list)
    if window:
        seqs = channel_sequences(orders, p, v)
        for ch, (snd, _rcv) in seqs.items():
            _, src, dst = ch
            for j in range(window, len(snd)):
                # producer (on src) of message j waits for the consumer (on
                # dst) of message j-W to have started
                prod_op = _producer(src, ch, snd[j], p, v)
                cons_op = _consumer(ch, snd[j - window], p, v)
                wdeps[(src, prod_op)].append((dst, cons_op))

    pos = [0] * p
    free = [0] * p
    start, end = {}, {}
    n_total = sum(len(x) for x in orders)
    done = 0
    while done < n_total:
        progress = False
        for s in range(p):
            while pos[s] < len(orders[s]):
                op = orders[s][pos[s]]
                deps = data_deps(s, op, p, v, recomputed)
                sdeps = wdeps.get((s, op), [])
                if all(d in end for d in deps) and all(d in start for d in sdeps):
                    t0 = max([free[s]] + [end[d] for d in deps] + [start[d] for d in sdeps])
                    start[(s, op)] = t0
                    end[(s, op)] = t0 + dfun(s, op)
                    free[s] = end[(s, op)]
                    pos[s] += 1
                    done += 1
                    progress = True
                else:
                    break
        if not progress and done < n_total:
            raise Deadlock(f"stuck at positions {pos}")
    return {"start": start, "end": end, "makespan": max(end.values()) if end else 0}


def _producer(src, ch, cm, p, v):
    c, i = cm
    if ch[0] == "A":
        # message carries input of (c,i) at dst; producer on src
        if src == p - 1 and ch[2] == 0:
            return ("F", c - 1, i)
        return ("F", c, i)
    if src == 0 and ch[2] == p - 1:
        return ("B", c + 1, i)
    return ("B", c, i)


def _consumer(ch, cm, p, v):
    c, i = cm
    return ("F", c, i) if ch[0] == "A" else ("B", c, i)


# --------------------------------------------------------------------------
# Block-level memory replay (order-determined, P:611 block = m_a/(2p))
# --------------------------------------------------------------------------

def block_replay(order, strategy: str):
    """Instruction-granular replay of one stage's order: at each op, allocs
    happen at op start, frees at op end; returns per-category peaks and the
    simultaneous total peak (activation blocks + recompute buffer; the
    T-Recomp checkpoints are reported separately as 'ckpt').

    strategy: 'tpipe' | 'tpipe_trecomp' | '1f1b' | '1f1b_full_recomp' |
              '1f1b_r50' | 'interleave'.
    Block units: m_a/(2p) per chunk task at v=2; a 1F1B microbatch on one
    stage is 2 blocks (m_a/p). Interleave uses m_a/(vp) per chunk task.
    """
    live = defaultdict(int)
    peak = defaultdict(int)
    peak_total = 0

    def bump():
        nonlocal peak_total
        for kk, vv in live.items():
            peak[kk] = max(peak[kk], vv)
        tot = sum(vv for kk, vv in live.items() if kk != "ckpt")
        peak_total = max(peak_total, tot)

    for kind, c, i in order:
        alloc, free = [], []
        if strategy in ("tpipe", "interleave"):
            if kind == "F":
                alloc = [f"c{c}"]
            elif kind == "B":
                free = [f"c{c}"]
        elif strategy == "tpipe_trecomp":
            if kind == "F" and c == 1:
                alloc, free = ["c1", "ckpt"], ["c1"]
            elif kind == "F":
                alloc = ["c2"]
            elif kind == "R":
                alloc = ["buf"]
            elif kind == "B" and c == 1:
                free = ["buf", "ckpt"]
            elif kind == "B":
                free = ["c2"]
        elif strategy == "1f1b":
            if kind == "F":
                alloc = ["c1", "c1"]
            elif kind == "B":
                free = ["c1", "c1"]
        elif strategy == "1f1b_r50":
            if kind == "F":
                alloc = ["c1"]          # half of the 2 blocks retained
            elif kind == "B":
                alloc, free = ["buf"], ["c1", "buf"]
        elif strategy == "1f1b_full_recomp":
            if kind == "F":
                alloc = ["ckpt"]
            elif kind == "B":
                alloc, free = ["buf"], ["ckpt", "buf"]
        else:
            raise ValueError(strategy)
        for x in alloc:
            live[x] += 1
        bump()
        for x in free:
            live[x] -= 1
            assert live[x] >= 0
    assert all(vv == 0 for vv in live.values()), "memory not released at step end"
    return dict(peak), peak_total


def idle_between(sim, s, t0, t1):
    """Idle time of stage s within [t0, t1) given simulated start/end."""
    busy = 0
    for (ss, _op), st in sim["start"].items():
        if ss != s:
            continue
        en = sim["end"][(ss, _op)]
        lo, hi = max(st, t0), min(en, t1)
        if hi > lo:
            busy += hi - lo
    return (t1 - t0) - busy


def strategy_orders(strategy: str, p: int, m: int, k: int | None = None, v: int = 2):
    """Convenience: (orders, v, recomputed, durations) for a named strategy;
    v = chunks per stage for the T-Pipe and Interleave strategies."""
    if strategy == "tpipe":
        return tpipe_orders(p, m, v=v), v, False, default_durations(2)
    if strategy == "tpipe_trecomp":
        return tpipe_orders(p, m, recomp=True, k=k, v=v), v, True, default_durations(2)
    if strategy == "tpipe_layer_grouped":
        return (tpipe_orders(p, m, layer_grouped=True), 2, False,
                default_durations(2, layer_grouped_b1=True))
    if strategy == "1f1b":
        return onef1b_orders(p, m), 1, False, default_durations(1)
    if strategy == "1f1b_r50":
        return onef1b_orders(p, m), 1, False, default_durations(1, b_extra=1)
    if strategy == "1f1b_full_recomp":
        return onef1b_orders(p, m), 1, False, default_durations(1, b_extra=2)
    if strategy == "interleave":
        return interleave_orders(p, m, v), v, False, default_durations(2)
    if strategy == "interleave_trecomp":
        return interleave_trecomp_orders(p, m, v), v, True, default_durations(2)
    raise ValueError(strategy)
