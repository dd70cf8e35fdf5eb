"""SASS instruction census of the placement kernels (cuobjdump -sass of the sm_100a
object): memory-path mnemonics (LDGSTS = Ampere cp.async, UBLKCP / UTMALDG = Hopper+ bulk
/ tensor copies, SYNCS = mbarrier ops), FP64 pipe (DADD / DMUL / DFMA), local memory
(LDL / STL = spills or local arrays) and barriers. Static counts (instructions in the
binary, not executions). Usage: sass_census.py [object] > profiles/.../sass_census.md"""
import re
import subprocess
import sys
from collections import Counter

obj = sys.argv[1] if len(sys.argv) > 1 else "paper_2512_16896_b200/csrc/build/sb_place.o"
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True, check=True).stdout
KEYS = ["LDGSTS", "UBLKCP", "UTMALDG", "SYNCS", "LDG", "STG", "LDS", "STS", "LDL", "STL",
        "DADD", "DMUL", "DFMA", "BAR", "ATOMG", "REDG", "SHFL"]
funcs = {}
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = Counter()
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if cur and m:
        op = m.group(1)
        funcs[cur][op] += 1
        funcs[cur]["_total"] += 1


def short(name):
    m = re.search(r"\d(k_[a-z0-9_]+?)(?:I|E)", name)
    base = m.group(1) if m else name
    targs = re.findall(r"Lb([01])E|Li(\d+)E", name)
    args = ",".join(a or b for a, b in targs)
    return f"{base}<{args}>" if args else base


print("| kernel | instrs | " + " | ".join(KEYS) + " |")
print("|---|---|" + "---|" * len(KEYS))
for f, c in sorted(funcs.items()):
    if "k_place" not in f and "k_wide" not in f and "k_fast" not in f:
        continue
    print(f"| `{short(f)}` | {c['_total']} | " + " | ".join(str(c[k]) for k in KEYS) + " |")
