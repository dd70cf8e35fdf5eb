"""Key numbers of an ncu --set full report (one or more launches):
  python tools/ncu_brief.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram_read"),
        ("dram__bytes_write.sum", "dram_write"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
        ("launch__occupancy_limit_registers", "occ_lim_regs"),
        ("sm__inst_executed.avg.per_cycle_active", "ipc"),
        ("lts__t_sector_hit_rate.pct", "l2_hit_%"), ("l1tex__t_sector_hit_rate.pct", "l1_hit_%"),
        ("smsp__inst_executed.sum", "warp_inst"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
        ("lts__t_sectors_srcunit_tex_op_read.sum", "l2_read_sectors"),
        ("local_load", None)]


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        print("kernel:", r[h.index("Kernel Name")][:90])
        for k, name in KEYS:
            if name and k in h:
                print(f"  {name:16s} {r[h.index(k)]:>16s} {units[h.index(k)]}")
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio"):
                try:
                    stalls.append((float(r[i]), k.split("stalled_")[1][:-6]))
                except ValueError:
                    pass
            elif k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), "pc:" + k.split("stalled_")[1]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("  stalls:", ", ".join(f"{n}={v:g}" for v, n in stalls[:12]))


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        main(rep)
