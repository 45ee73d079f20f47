"""JSON config ingestion (SPEC's load_config maps onto
tpipe_plan_create). Validation errors name the offending field."""

import json
import os
import subprocess
import sys

import pytest

from paper_2503_03182_b200 import config as CFG, plan as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = {"model": {"n_layers": 8, "hidden": 64, "n_heads": 4, "ffn_hidden": 256, "vocab": 256,
                  "seq_len": 32, "micro_batch": 2}, "p": 4, "m": 8}


def cfg(**kw):
    d = json.loads(json.dumps(BASE))
    d.update(kw)
    return d


def test_defaults_and_equivalence_with_direct_call():
    plan = CFG.load(cfg(strategy="tpipe_trecomp"))
    ref = P.Plan(P.Model(8, 64, 4, 256, 256, 32, 2, P.BF16), 4, 8, strategy="tpipe_trecomp")
    assert plan.strategy == ref.strategy and plan.v == 2 and plan.k == ref.k
    for s in range(4):
        assert plan.ops(s)[0] == ref.ops(s)[0]
        assert plan.peak(s) == ref.peak(s)


def test_all_options_roundtrip(tmp_path):
    c = cfg(strategy="tpipe", chunks=2, offload=["model_state", "device_opt"], dp=2,
            recompute={"layers": 0}, partition={"stage_layers": [2, 2, 2, 2], "stage_chunk1": [1, 1, 1, 1]},
            cost_model={"host_link_bps": 4e10})
    c["offload"] = []            # dp > 1 excludes model-state offload (R31)
    f = tmp_path / "c.json"
    f.write_text(json.dumps(c))
    plan = CFG.load(str(f))
    assert plan.dp == 2 and plan.partition == [(1, 1)] * 4
    s = CFG.summary(plan)
    assert s["strategy"] == "tpipe" and len(s["peak_bytes"]) == 4 and s["unit_makespan"] > 0


@pytest.mark.parametrize("bad,field", [
    ({"p": 0}, "p"), ({"m": "8"}, "m"), ({"strategy": "gpipe"}, "strategy"),
    ({"chunks": 5}, "chunks"), ({"offload": ["everything"]}, "offload"),
    ({"hbm_budget_gib": -1}, "hbm_budget_gib"), ({"bogus": 1}, "bogus"),
    ({"partition": {"stage_layers": [8]}}, "partition.stage_layers"),
    ({"cost_model": {"device_flops": "fast"}}, "cost_model.device_flops"),
])
def test_validation_names_field(bad, field):
    with pytest.raises(CFG.ConfigError) as e:
        CFG.load(cfg(**bad))
    assert e.value.field == field


def test_model_field_errors():
    c = cfg()
    del c["model"]["hidden"]
    with pytest.raises(CFG.ConfigError, match="model.hidden"):
        CFG.load(c)
    c = cfg()
    c["model"]["dtype"] = "fp8"
    with pytest.raises(CFG.ConfigError, match="model.dtype"):
        CFG.load(c)


def test_budget_escalation_and_cli(tmp_path):
    c = cfg(strategy="auto", hbm_budget_gib=0.0005)
    with pytest.raises(Exception, match="no escalation fits"):
        CFG.load(c)
    c = cfg(strategy="auto", hbm_budget_gib=1)
    f = tmp_path / "c.json"
    f.write_text(json.dumps(c))
    out = subprocess.run([sys.executable, "-m", "paper_2503_03182_b200.config", str(f)], cwd=ROOT,
                         capture_output=True, text=True, check=True).stdout
    assert json.loads(out)["strategy"] == "tpipe"
    f.write_text("{not json")
    r = subprocess.run([sys.executable, "-m", "paper_2503_03182_b200.config", str(f)], cwd=ROOT,
                       capture_output=True, text=True)
    assert r.returncode == 2 and "cannot parse" in r.stderr
