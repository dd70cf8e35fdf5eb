"""Per-source-line executed warp instructions from an ncu source export (cuda,sass):
  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv
  python tools/ncu_inst.py s.csv [file-filter] [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
filt = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
fname = None
hdr = None
agg = defaultdict(float)
src = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ix = {h: i for i, h in enumerate(hdr)}
        continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-":
        continue
    key = (fname, int(r[0]))
    src[key] = r[1][:90]
    try:
        agg[key] += float(r[ix["Instructions Executed"]])
    except ValueError:
        pass
tot = sum(agg.values())
print("total warp instructions", tot)
sel = [(k, v) for k, v in agg.items() if filt in k[0] and v > 0]
for k, v in sorted(sel, key=lambda x: -x[1])[:top]:
    print(f"{v:7.0f} {k[0]}:{k[1]:<5} {src[k]}")
