"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) as markdown.

  python tools/launch_summary.py launches.csv "title"
"""
import csv
import sys
from collections import defaultdict

path, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
rows = []
with open(path) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
    rows.append((r["Kernel Name"], v * scale))
agg = defaultdict(lambda: [0, 0.0])
for name, us in rows:
    key = name.split("(")[0].replace("void ", "")[:60]
    agg[key][0] += 1
    agg[key][1] += us
tot = sum(v[1] for v in agg.values())
print(f"# {title}\n")
print("ncu `gpu__time_duration.sum`, `--clock-control none`; per-launch times are cold-cache and serialised.\n")
print("| kernel | launches | total ms | share |\n|---|---|---|---|")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| {k} | {n} | {us / 1e3:.3f} | {100 * us / tot:.1f}% |")
print(f"\nTotal {len(rows)} launches, {tot / 1e3:.2f} ms.")
