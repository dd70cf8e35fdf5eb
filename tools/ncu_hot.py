"""Top SASS instructions by warp-stall samples of an ncu report (source page), with the
instructions before each for context:  python tools/ncu_hot.py report.ncu-rep [top] [ctx]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 3
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
body = [r for r in rows[2:] if len(r) == len(h)]
si = h.index("Warp Stall Sampling (All Samples)")
ex = h.index("Instructions Executed")
tot = sum(int(r[si] or 0) for r in body)
print(f"{len(body)} instructions, {tot} samples")
order = sorted(range(len(body)), key=lambda i: -int(body[i][si] or 0))
for i in order[:top]:
    print(f"--- {int(body[i][si])} samples ({int(body[i][si]) / tot:.1%}), exec {body[i][ex]}")
    for j in range(max(0, i - ctx), i + 1):
        print(f"   {j:5d} {body[j][si]:>6s} {body[j][1].strip()}")
