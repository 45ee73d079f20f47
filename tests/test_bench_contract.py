"""CPU checks of bench.py's contract: the reference arm (the fp64 oracle,
DESIGN.md §10) prints one JSON line with the driver's keys, and the planner's
capacity sweep (SURVEY D-13) gives T-Pipe-ALL >= 2x the 1F1B model size at a
fixed 80 GiB per-GPU budget (the north star's size target, byte model)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, check=True).stdout.strip().splitlines()
    assert len(out) == 1
    d = json.loads(out[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "tokens/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_capacity_sweep_size_target():
    sys.path.insert(0, ROOT)
    import bench
    cap = bench.capacity(8)
    assert cap["tpipe_all"]["max_params_B"] >= 2 * cap["1f1b"]["max_params_B"]
    assert cap["tpipe_trecomp"]["max_layers"] > cap["tpipe"]["max_layers"] >= cap["1f1b"]["max_layers"]
    # plain Interleave-1F1B stores more than 1F1B; with T-Recomp it stores less
    assert cap["interleave"]["max_layers"] < cap["1f1b"]["max_layers"] < cap["interleave_trecomp"]["max_layers"]


def test_balanced_partition_and_choice():
    """R27: the balanced split keeps every stage >= v layers, sums to L and
    lowers the largest stage cost (head counted in layer-equivalents); the
    planner picks a partition only when its cost model predicts >= 3% gain."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2503_03182_b200 import plan as P
    c = bench.C2
    hl = 6 * c["hidden"] * c["vocab"] / (72 * c["hidden"] ** 2 + 6 * c["seq_len"] * c["hidden"])
    for p in (2, 4, 8):
        for v in (1, 2):
            part = bench.balanced_partition(24, p, v, hl)
            assert sum(part) == 24 and min(part) >= v and len(part) == p
            cost = max(max(part[:-1]), part[-1] + hl)
            assert cost <= max(24 // p, 24 // p + hl)
    # the choice itself now lives in the planner (tpipe_plan_opts.balance, R28/R29)
    md = P.Model(24, 2048, 16, 8192, 50304, 2048, 1, P.BF16)
    assert P.Plan(md, 8, 32, strategy="tpipe", balance=True).balanced
    assert not P.Plan(md, 1, 32, strategy="tpipe", balance=True).balanced


def test_gpus_n_without_ranks_refuses():
    """`bench.py --gpus N` outside torchrun launches N ranks itself, or — on a
    box with fewer than N GPUs (here: none) — exits 2 with a clear error
    instead of printing a one-GPU virtual-pipeline number labelled N GPUs."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 2
    assert r.stdout.strip() == ""
    assert "needs 2 GPUs" in r.stderr and "--virtual-stages" in r.stderr
