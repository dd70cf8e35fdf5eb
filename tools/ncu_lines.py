"""Warp-stall samples of an ncu report aggregated by CUDA source line, through the
nvdisasm -gi line table of the kernel in the library that was profiled.
  python tools/ncu_lines.py report.ncu-rep lib.so kernel_substring [top]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, lib, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
body = [r for r in rows[2:] if len(r) == len(h)]
si, ai = h.index("Warp Stall Sampling (All Samples)"), h.index("Address")
ex = h.index("Instructions Executed")
base = int(body[0][ai], 16)
samples = {int(r[ai], 16) - base: (int(r[si] or 0), int(r[ex] or 0)) for r in body}

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
lines_of = {}
for cub in sorted(os.listdir(tmp)):
    dis = subprocess.run(["nvdisasm", "-gi", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    sec = None
    cur_inner = cur_outer = None
    in_block = False
    for ln in dis.splitlines():
        m = re.match(r"\s*\.section\s+\.text\.(\S+),", ln)
        if m:
            sec = m.group(1).rstrip(",")
            continue
        if sec is None or kname not in sec:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
        if m:  # the first annotation of a block is the innermost frame, the last the kernel's
            here = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            if not in_block:
                cur_inner = here
                in_block = True
            cur_outer = here if not m.group(3) else f"{os.path.basename(m.group(3))}:{m.group(4)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_inner:
            in_block = False
            lines_of[int(m.group(1), 16)] = (cur_inner, cur_outer)
    if lines_of:
        break
agg_in, agg_out = collections.Counter(), collections.Counter()
exe = collections.Counter()
tot = 0
for off, (s, e) in samples.items():
    li, lo = lines_of.get(off, ("?", "?"))
    agg_in[li] += s
    agg_out[lo] += s
    exe[li] += e
    tot += s
print(f"{tot} samples; mapped offsets {len(lines_of)}")
print("-- by innermost line")
for k, v in agg_in.most_common(top):
    print(f"{v:7d} {v / max(tot, 1):6.1%}  exec {exe[k]:10d}  {k}")
tot_e = sum(exe.values())
print(f"-- by executed instructions (innermost line), {tot_e} total")
for k, v in exe.most_common(top):
    print(f"{v:10d} {v / max(tot_e, 1):6.1%}  samples {agg_in[k]:6d}  {k}")
print("-- by outermost (kernel-file) line")
for k, v in agg_out.most_common(top // 2):
    print(f"{v:7d} {v / max(tot, 1):6.1%}  {k}")
