"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel:
python scripts/launch_summary.py launches.csv [header-comment] [last-N-launches]"""
import csv, sys, collections

path = sys.argv[1]
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    us = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v if unit == "us" else v / 1e3
    rows.append((r["Kernel Name"], us))
if len(sys.argv) > 3:
    rows = rows[-int(sys.argv[3]):]
tot = sum(u for _, u in rows)
agg = collections.defaultdict(lambda: [0, 0.0])
for k, u in rows:
    agg[k][0] += 1
    agg[k][1] += u
if len(sys.argv) > 2:
    print("# " + sys.argv[2])
print(f"# launches {len(rows)}  total {tot / 1e3:.1f} ms")
print(f"{'share':>7} {'count':>6} {'avg_us':>9}  kernel")
for k, (n, u) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    name = k if len(k) < 90 else k[:87] + "..."
    print(f"{100 * u / tot:6.2f}% {n:6d} {u / n:9.1f}  {name}")
