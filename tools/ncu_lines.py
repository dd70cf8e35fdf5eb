"""Aggregate an ncu '--page source --csv --print-source cuda,sass' export by CUDA source
line: warp-stall samples (all) and the top stall reasons. Usage:
  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv
  python tools/ncu_lines.py s.csv [top]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
fname = None
hdr = None
agg = defaultdict(lambda: defaultdict(float))
src = {}
total = 0.0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name",) or len(r) < len(hdr):
        continue
    if r[2] != "-":  # sass row inside a line; skip (line rows have Address '-')
        continue
    key = (fname, int(r[0]))
    src[key] = r[1][:70]
    for i, h in enumerate(hdr):
        if i < 4:
            continue
        if h.startswith("stall_") and "Not Issued" not in h or h == "Warp Stall Sampling (All Samples)":
            try:
                v = float(r[i])
            except ValueError:
                continue
            agg[key][h] += v
for k in agg:
    total += agg[k]["Warp Stall Sampling (All Samples)"]
items = sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])
print(f"total samples {total:.0f}")
for k, d in items[:top]:
    s = d["Warp Stall Sampling (All Samples)"]
    if s == 0:
        break
    reasons = sorted(((v, h[6:]) for h, v in d.items() if h.startswith("stall_")), reverse=True)[:3]
    rs = " ".join(f"{h}:{v / s:.0%}" for v, h in reasons if v > 0)
    print(f"{s / total:6.1%} {k[0]}:{k[1]:<4} {src[k]:<70} {rs}")
