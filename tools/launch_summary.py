"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) as a markdown
table: launches, total us and share per kernel. Usage: launch_summary.py launches.csv [steps]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
ix = {k: j for j, k in enumerate(h)}
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
d = defaultdict(lambda: [0, 0.0])
for r in rows[i + 1:]:
    if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]].replace(",", "")) * scale[r[ix["Metric Unit"]]]
    name = r[ix["Kernel Name"]].split("(")[0]
    d[name][0] += 1
    d[name][1] += v
tot = sum(v[1] for v in d.values())
print(f"| kernel | launches | total us | us per step (/{steps:g}) | share |")
print("|---|---|---|---|---|")
for k, v in sorted(d.items(), key=lambda x: -x[1][1]):
    print(f"| `{k}` | {v[0]} | {v[1]:.1f} | {v[1] / steps:.1f} | {v[1] / tot:.1%} |")
print(f"\nTotal kernel time {tot / 1e3:.3f} ms over {sum(v[0] for v in d.values())} launches.")
