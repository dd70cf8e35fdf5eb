"""Summarise an `ncu --set full` report of k_place into profiles/ncu_k_place_<cfg>.json
(the bench's `roofline.traffic` source) and print a markdown table.
  python tools/ncu_summary.py gpurun_out/prof_X.ncu-rep <config> [out.json]"""
import csv
import io
import json
import subprocess
import sys

rep, cfg = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else f"profiles/ncu_k_place_{cfg}.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
want = {
    "dram_read": "dram__bytes_read.sum", "dram_write": "dram__bytes_write.sum",
    "duration": "gpu__time_duration.sum",
    "fp64_pipe_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread", "ipc": "sm__inst_executed.avg.per_cycle_active",
    "l2_hit": "lts__t_sector_hit_rate.pct", "l1_hit": "l1tex__t_sector_hit_rate.pct",
}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
         "msecond": 1e3, "us": 1.0, "ns": 1e-3, "ms": 1e3}
ix = {k: h.index(v) for k, v in want.items() if v in h}
launches = []
for r in rows[2:]:
    d = {}
    for k, i in ix.items():
        try:
            val = float(r[i].replace(",", ""))
        except ValueError:
            continue
        d[k] = val * scale.get(units[i], 1.0) if k in ("dram_read", "dram_write", "duration") else val
    d["kernel"] = r[h.index("Kernel Name")] if "Kernel Name" in h else ""
    launches.append(d)
n = len(launches)
avg = lambda k: sum(l.get(k, 0.0) for l in launches) / max(n, 1)
summary = {
    "config": cfg, "report": rep, "launches_profiled": n,
    "dram_bytes_per_launch": round(avg("dram_read") + avg("dram_write")),
    "dram_read_bytes_per_launch": round(avg("dram_read")),
    "dram_write_bytes_per_launch": round(avg("dram_write")),
    "duration_us_per_launch_cold": round(avg("duration"), 2),
    "fp64_pipe_pct_of_peak": round(avg("fp64_pipe_pct"), 2),
    "warps_active_pct": round(avg("warps_active_pct"), 2),
    "registers_per_thread": launches[0].get("regs") if launches else None,
    "l2_hit_pct": round(avg("l2_hit"), 1), "l1_hit_pct": round(avg("l1_hit"), 1),
}
json.dump(summary, open(out, "w"), indent=1)
print(f"| launch | duration us (cold) | DRAM read MB | DRAM write MB | FP64 pipe % | warps active % |")
print("|---|---|---|---|---|---|")
for i, l in enumerate(launches):
    print(f"| {i} | {l.get('duration', 0):.1f} | {l.get('dram_read', 0) / 1e6:.2f} | {l.get('dram_write', 0) / 1e6:.2f} "
          f"| {l.get('fp64_pipe_pct', 0):.2f} | {l.get('warps_active_pct', 0):.1f} |")
print(json.dumps(summary))
