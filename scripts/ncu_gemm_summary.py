"""Summarise an `ncu --set full` capture of the 12 layer GEMM shapes
(scripts/gemm_shapes_once.py) into the jsonl bench.py's gemm_traffic() reads:

  ncu -i rep.ncu-rep --page raw --csv > raw.csv
  python scripts/ncu_gemm_summary.py raw.csv shapes.jsonl > profiles/rN_gemm_ncu_full_vK.jsonl

shapes.jsonl = the stdout of gemm_shapes_once.py (kernel order = capture order)."""
import csv
import json
import sys


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
data = [r for r in rows[2:] if len(r) == len(hdr)]   # row 1 = units
units = rows[1]
shapes = [json.loads(l) for l in open(sys.argv[2]) if l.startswith("{")]
col = {h: i for i, h in enumerate(hdr)}
PREF = ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")
tensor_col = next((h for h in PREF if h in hdr), None)
out, dram_tot, alg_tot = [], 0.0, 0.0
for sh, r in zip(shapes, data):
    t = num(r[col["gpu__time_duration.sum"]])
    tu = units[col["gpu__time_duration.sum"]]
    us = t / 1e3 if tu == "nsecond" else t * 1e3 if tu == "msecond" else t
    def bytes_of(name):
        v, u = num(r[col[name]]), units[col[name]]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    dram = bytes_of("dram__bytes_read.sum") + bytes_of("dram__bytes_write.sum")
    d = {"kernel": sh["kernel"], "grid": r[col["launch__grid_size"]] if "launch__grid_size" in col else None,
         "us": round(us, 3), "tflops_cold": round(sh["flops"] / (us * 1e-6) / 1e12, 1),
         "dram_MB": round(dram / 1e6, 1), "alg_MB": round(sh["alg_bytes"] / 1e6, 1),
         "traffic_over_alg": round(dram / sh["alg_bytes"], 2)}
    if tensor_col:
        d["tensor_active_pct"] = round(num(r[col[tensor_col]]), 1)
    out.append(d)
    dram_tot += dram
    alg_tot += sh["alg_bytes"]
for d in out:
    print(json.dumps(d))
print(json.dumps({"summary": True, "launches": len(out), "mean_dram_bytes": int(dram_tot / len(out)),
                  "mean_alg_bytes": int(alg_tot / len(out)), "tensor_metric": tensor_col}))
