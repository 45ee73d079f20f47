"""Duration-aware T-Pipe (DESIGN R29).

The T-Pipe slot order (D-1) assumes equal chunk durations on every stage
(P:611 unit model). With the LM head on the last stage's deep chunk (SURVEY
D-12: 1.9 layer-forwards at the GPT-3 1.3B shape) they are not equal, and the
R27 partition alone made T-Pipe lose to a balanced 1F1B at p = 4 (DESIGN §5c:
0.95x). The planner's `balance` option now searches per-stage layer counts AND
chunk splits on the modeled ASAP replay of T-Pipe's own order.

Pins (independent of the planner's code):
* replay parity: the oracle simulator (oracle/schedule.simulate) run on the
  same order with durations from the FLOP model gives the planner's makespan;
* exhaustive search: on a small instance, no partition / split in the whole
  space beats the planner's choice by more than 1%;
* the D-12 gap closes: at p = 4 (C2) T-Pipe's modeled step equals a balanced
  1F1B's; at p = 8 it is within 3%.
"""

import itertools

import pytest

from oracle import schedule as S
from paper_2503_03182_b200 import plan as P

C2 = dict(h=2048, a=16, f=8192, V=50304, s=2048, b=1)


def layer_flops(c):
    M = c["b"] * c["s"]
    return 2 * M * (4 * c["h"] ** 2 + 2 * c["h"] * c["f"]) + \
        4 * c["b"] * c["a"] * (c["s"] * (c["s"] + 1) / 2) * (c["h"] // c["a"])


def head_flops(c):
    return 2 * c["b"] * c["s"] * c["V"] * c["h"]


def model(L, c=C2):
    return P.Model(L, c["h"], c["a"], c["f"], c["V"], c["s"], c["b"], P.BF16)


def oracle_makespan(strategy, p, m, part, c=C2, flops=1e15):
    """oracle.schedule.simulate of the strategy's order with F = layers of
    the chunk (+ the head on the last stage's last chunk) x layer time, B = 2F."""
    orders = S.strategy_orders(strategy, p, m)[0]
    v = 1 if strategy == "1f1b" else 2
    tl, th = layer_flops(c) / flops, head_flops(c) / flops

    def dur(s, op):
        kind, ch, _i = op
        f = part[s][ch - 1] * tl + (th if (s == p - 1 and ch == v) else 0.0)
        return 2 * f if kind == "B" else f
    return S.simulate(orders, p, v, dur)["makespan"]


@pytest.mark.parametrize("strategy", ["tpipe", "1f1b", "interleave"])
@pytest.mark.parametrize("p", [2, 4, 8])
def test_planner_makespan_equals_oracle_replay(strategy, p):
    pl = P.Plan(model(24), p, 32, strategy=strategy, balance=True)
    assert pl.est_step_s == pytest.approx(oracle_makespan(strategy, p, 32, pl.partition), rel=1e-9)


def test_p4_tpipe_no_longer_loses_to_balanced_1f1b():
    md = model(24)
    tp = P.Plan(md, 4, 32, strategy="tpipe", balance=True)
    fb = P.Plan(md, 4, 32, strategy="1f1b", balance=True)
    assert tp.balanced and fb.balanced
    assert tp.est_step_s <= fb.est_step_s * (1 + 1e-9)
    # the R27 closed form alone (ceil/floor chunk splits) left T-Pipe behind
    r27 = P.Plan(md, 4, 32, strategy="tpipe", stage_layers=[7, 7, 7, 3])
    assert r27.est_step_s > 1.05 * fb.est_step_s
    p8t = P.Plan(md, 8, 32, strategy="tpipe", balance=True)
    p8f = P.Plan(md, 8, 32, strategy="1f1b", balance=True)
    assert p8t.est_step_s <= 1.03 * p8f.est_step_s


def test_search_near_exhaustive_optimum():
    """p = 4, L = 12, m = 8 (C2 layer shape): every composition of 12 layers
    into 4 stages (>= 2 each) and every chunk split, simulated by the oracle;
    the planner's steepest-descent choice is within 1% of the best."""
    p, L, m = 4, 12, 8
    best = None
    for comp in itertools.product(range(2, 7), repeat=p):
        if sum(comp) != L:
            continue
        for splits in itertools.product(*[range(1, n) for n in comp]):
            part = [(a, n - a) for a, n in zip(splits, comp)]
            mk = oracle_makespan("tpipe", p, m, part)
            if best is None or mk < best:
                best = mk
    pl = P.Plan(model(L), p, m, strategy="tpipe", balance=True)
    got = oracle_makespan("tpipe", p, m, pl.partition)
    assert got <= best * 1.01
