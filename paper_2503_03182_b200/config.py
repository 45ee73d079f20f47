"""JSON configuration -> tpipe_plan_create (config ingestion,
SPEC S:65-73 maps onto the planner's C-ABI call). Marshalling and validation
only; every decision is the planner's (include/tpipe.h).

Schema (all keys optional except model / p / m):

    {
      "model": {"n_layers": 24, "hidden": 2048, "n_heads": 16, "ffn_hidden": 8192,
                "vocab": 50304, "seq_len": 2048, "micro_batch": 1, "dtype": "bf16"},
      "p": 8,                      # pipeline stages
      "m": 32,                     # micro-batches per step (per replica)
      "dp": 1,                     # data-parallel replicas (ZeRO-1, DESIGN R31)
      "hbm_budget_gib": 80,        # per-GPU budget; 0 / absent = none
      "strategy": "auto",          # tpipe | tpipe_trecomp | 1f1b | 1f1b_full_recomp |
                                   # interleave | interleave_trecomp | auto
      "chunks": 2,                 # 2, 3, 4 (0 with auto: try all)
      "recompute": {"layers": 0, "delay_rounds": -1},
      "offload": ["model_state", "device_opt", "activations"],
      "act_distance": 0, "send_window": 0,
      "partition": {"balance": false, "stage_layers": [...], "stage_chunk1": [...]},
      "cost_model": {"host_link_bps": 0, "host_adam_params_per_s": 0, "device_flops": 0}
    }

Errors raise ConfigError naming the offending field (SPEC's ValidationError).
`python -m paper_2503_03182_b200.config cfg.json` prints the plan summary.
"""

from __future__ import annotations

import json
import sys

from . import plan as P


class ConfigError(ValueError):
    """Invalid configuration; `field` names the offending key."""

    def __init__(self, field: str, msg: str):
        super().__init__(f"{field}: {msg}")
        self.field = field


MODEL_KEYS = ("n_layers", "hidden", "n_heads", "ffn_hidden", "vocab", "seq_len", "micro_batch")
OFFLOAD = {"model_state": P.OFFLOAD_MODEL_STATE, "activations": P.OFFLOAD_ACTIVATIONS,
           "device_opt": P.OFFLOAD_DEVICE_OPT}
TOP_KEYS = {"model", "p", "m", "dp", "hbm_budget_gib", "strategy", "chunks", "recompute", "offload",
            "act_distance", "send_window", "partition", "cost_model"}


def _int(d, key, field, lo=None, default=None):
    if key not in d:
        if default is None:
            raise ConfigError(field, "required")
        return default
    v = d[key]
    if isinstance(v, bool) or not isinstance(v, int):
        raise ConfigError(field, f"must be an integer, got {v!r}")
    if lo is not None and v < lo:
        raise ConfigError(field, f"must be >= {lo}, got {v}")
    return v


def parse(cfg: dict) -> dict:
    """Validate a config dict; returns the normalised keyword arguments of
    plan.Plan plus model / p / m."""
    if not isinstance(cfg, dict):
        raise ConfigError("<root>", "must be a JSON object")
    unknown = set(cfg) - TOP_KEYS
    if unknown:
        raise ConfigError(sorted(unknown)[0], "unknown key")
    md = cfg.get("model")
    if not isinstance(md, dict):
        raise ConfigError("model", "required object")
    for k in md:
        if k not in MODEL_KEYS and k != "dtype":
            raise ConfigError(f"model.{k}", "unknown key")
    mvals = {k: _int(md, k, f"model.{k}", lo=1) for k in MODEL_KEYS}
    dt = md.get("dtype", "bf16")
    if dt not in ("bf16", "fp32"):
        raise ConfigError("model.dtype", "must be 'bf16' or 'fp32'")
    model = P.Model(*(mvals[k] for k in MODEL_KEYS), P.BF16 if dt == "bf16" else P.FP32)
    p = _int(cfg, "p", "p", lo=1)
    m = _int(cfg, "m", "m", lo=1)
    kw = {"dp": _int(cfg, "dp", "dp", lo=1, default=1)}
    budget = cfg.get("hbm_budget_gib", 0)
    if not isinstance(budget, (int, float)) or isinstance(budget, bool) or budget < 0:
        raise ConfigError("hbm_budget_gib", "must be a number >= 0")
    kw["hbm_budget"] = int(budget * 2 ** 30)
    strat = cfg.get("strategy", "tpipe")
    if strat != "auto" and strat not in P.STRATEGY:
        raise ConfigError("strategy", f"one of {sorted(P.STRATEGY) + ['auto']}")
    kw["strategy"] = strat
    kw["chunks"] = _int(cfg, "chunks", "chunks", lo=0, default=0 if strat == "auto" else 2)
    if kw["chunks"] not in (0, 2, 3, 4) or (kw["chunks"] == 0 and strat != "auto"):
        raise ConfigError("chunks", "must be 2, 3 or 4 (0 only with strategy auto)")
    rec = cfg.get("recompute", {})
    if not isinstance(rec, dict):
        raise ConfigError("recompute", "must be an object")
    kw["recomp_layers"] = _int(rec, "layers", "recompute.layers", lo=0, default=0)
    kw["delay_rounds"] = _int(rec, "delay_rounds", "recompute.delay_rounds", lo=-1, default=-1)
    off = cfg.get("offload", [])
    if not isinstance(off, list) or any(o not in OFFLOAD for o in off):
        raise ConfigError("offload", f"list of {sorted(OFFLOAD)}")
    flags = 0
    for o in off:
        flags |= OFFLOAD[o]
    kw["offload"] = flags if (off or strat != "auto") else 0
    kw["act_distance"] = _int(cfg, "act_distance", "act_distance", lo=0, default=0)
    kw["send_window"] = _int(cfg, "send_window", "send_window", lo=0, default=0)
    part = cfg.get("partition", {})
    if not isinstance(part, dict):
        raise ConfigError("partition", "must be an object")
    kw["balance"] = bool(part.get("balance", False))
    for k in ("stage_layers", "stage_chunk1"):
        if k in part:
            v = part[k]
            if not isinstance(v, list) or len(v) != p or any(isinstance(x, bool) or not isinstance(x, int)
                                                             for x in v):
                raise ConfigError(f"partition.{k}", f"list of {p} integers")
            kw[k] = v
    cm = cfg.get("cost_model", {})
    if not isinstance(cm, dict):
        raise ConfigError("cost_model", "must be an object")
    for k in ("host_link_bps", "host_adam_params_per_s", "device_flops"):
        v = cm.get(k, 0)
        if not isinstance(v, (int, float)) or isinstance(v, bool) or v < 0:
            raise ConfigError(f"cost_model.{k}", "must be a number >= 0")
        kw[k] = float(v)
    return {"model": model, "p": p, "m": m, **kw}


def load(src) -> "P.Plan":
    """A plan from a JSON file path, JSON text or dict (the planner validates
    the rest: its TPipeError messages name the field)."""
    if isinstance(src, dict):
        cfg = src
    else:
        try:
            text = open(src).read() if not str(src).lstrip().startswith("{") else str(src)
            cfg = json.loads(text)
        except (OSError, json.JSONDecodeError) as e:
            raise ConfigError("<document>", f"cannot parse: {e}") from None
    a = parse(cfg)
    model, p, m = a.pop("model"), a.pop("p"), a.pop("m")
    return P.Plan(model, p, m, **a)


def summary(plan: "P.Plan") -> dict:
    names = ["1f1b", "1f1b_full_recomp", "tpipe", "tpipe_trecomp", "interleave", "interleave_trecomp"]
    mk, _busy = plan.simulate()
    return {"strategy": names[plan.strategy], "chunks": plan.v, "dp": plan.dp, "offload": plan.offload,
            "recomp_layers": plan.recomp_layers, "delay_rounds": plan.k, "send_window": plan.W,
            "partition": [list(x) for x in plan.partition], "params": plan.params_total,
            "peak_bytes": [plan.peak(s)["total_peak"] for s in range(plan.p)],
            "unit_makespan": mk, "est_step_s": plan.est_step_s,
            "est_exposed_offload_s": plan.est_exposed_offload_s}


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    if len(argv) != 1:
        print("usage: python -m paper_2503_03182_b200.config CONFIG.json", file=sys.stderr)
        return 2
    try:
        print(json.dumps(summary(load(argv[0]))))
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    return 0


if __name__ == "__main__":
    sys.exit(main())
