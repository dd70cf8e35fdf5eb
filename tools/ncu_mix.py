"""Opcode mix (warp instructions executed) of an ncu report's source page:
  python tools/ncu_mix.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
ex = h.index("Instructions Executed")
c = Counter()
for r in rows[2:]:
    if len(r) != len(h):
        continue
    ins = r[1].strip()
    op = ins.split()[1] if ins.startswith("@") else ins.split()[0]
    c[op.split(".")[0]] += int(r[ex] or 0)
tot = sum(c.values())
print(f"total warp instructions {tot}")
for op, v in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{op:12s} {v:12d} {v / tot:6.1%}")
