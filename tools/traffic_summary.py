"""DRAM traffic of one warm generation, per kernel and per placement, from an ncu CSV of
  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,\
dram__bytes_write.sum --clock-control none --csv python tools/one_step.py <config>
(ncu flushes the caches before every kernel: cold-cache bytes, an upper bound for the
pipelined run). Writes a JSON summary; bench.py reads its `dram_bytes_per_launch` as the
roofline's `traffic` (one "launch" = one placement's kernel chain).
Usage: traffic_summary.py traffic.csv config placements out.json"""
import csv
import json
import sys
from collections import defaultdict

path, cfg, placements, out = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
rows = list(csv.reader(open(path)))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
ix = {k: j for j, k in enumerate(h)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
per = defaultdict(lambda: {"launches": 0, "us": 0.0, "read": 0.0, "write": 0.0})
seen = set()
for r in rows[i + 1:]:
    if len(r) < len(h):
        continue
    name = r[ix["Kernel Name"]].split("(")[0]
    m = r[ix["Metric Name"]]
    v = float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1.0)
    d = per[name]
    if (r[ix["ID"]], name) not in seen:
        seen.add((r[ix["ID"]], name))
        d["launches"] += 1
    if m == "gpu__time_duration.sum":
        d["us"] += v
    elif m == "dram__bytes_read.sum":
        d["read"] += v
    elif m == "dram__bytes_write.sum":
        d["write"] += v
tot_r = sum(d["read"] for d in per.values())
tot_w = sum(d["write"] for d in per.values())
res = {"config": cfg, "placements": placements, "source": path.split("/")[-1],
       "dram_read_bytes_per_step": round(tot_r), "dram_write_bytes_per_step": round(tot_w),
       "dram_bytes_per_launch": round((tot_r + tot_w) / placements),
       "dram_write_bytes_per_launch": round(tot_w / placements),
       "kernels": {k: {"launches": d["launches"], "us": round(d["us"], 1),
                       "dram_read": round(d["read"]), "dram_write": round(d["write"])}
                   for k, d in sorted(per.items(), key=lambda x: -x[1]["us"])}}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "kernels"}))
for k, d in list(res["kernels"].items())[:12]:
    print(f"{k[:60]:60s} n={d['launches']:4d} {d['us']:9.1f} us  R {d['dram_read'] / 1e6:9.1f} MB  W {d['dram_write'] / 1e6:8.1f} MB")
