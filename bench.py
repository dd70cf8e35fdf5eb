#!/usr/bin/env python
"""Benchmark: collision-free scenes/sec and candidate collision checks/sec (BASELINE.json).

A step is one full generation pass (every placement, every attempt round) over the
config's N variations per GPU, through the C ABI (libscenebatch_b200.so).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4_clutter] [--impl ours|reference]

Default workload: C4 (262,144 variations x 100 sphere-set objects), the largest
single-GPU configuration BASELINE.json names (its `metric` is not quoted on any config).
N>1 runs under torchrun (one rank per GPU): instances are sharded by contiguous
variation ranges (weak scaling: N_per_gpu fixed); the only exchange is the fast-path
per-round count all-gather (8 bytes per rank per round) and a relation placement's
instance-0 anchor state, both through the library's native communicator (sb_comm: no
torch.distributed, no NCCL on the data path).
`value` times results resident in HBM (CUDA events on the engine stream, L2 flushed
between steps); `e2e` times the same call with the results copied to pinned host memory.
--impl reference times the reference itself (oracle/_ref/libsbref.so: its own sources
compiled in place + the Appendix-C driver) on the host cores; that process builds its
scene with the reference's own mesh constructors and never maps this package's library.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import struct
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "collision-free scenes/sec and candidate collision checks/sec at 1/2/4/8 B200"

WORKLOADS = {
    "c1_tabletop": ("tabletop: 1 table, 10 cuboids, 1024 variations/GPU, 64 candidates/object",
                    lambda n: __import__("paper_2512_16896_b200.scenes", fromlist=["x"]).tabletop_boxes(n), 1024),
    "c2_mixed": ("tabletop: 25 mixed cuboid+sphere-set objects, on/next-to relations, "
                 "16384 variations/GPU, 64 candidates/object",
                 lambda n: __import__("paper_2512_16896_b200.scenes", fromlist=["x"]).tabletop_mixed(n), 16384),
    "c3_kitchen": ("kitchen: 3 supports incl. container interior, 50 objects, 65536 variations/GPU, "
                   "256 candidates/object",
                   lambda n: __import__("paper_2512_16896_b200.scenes", fromlist=["x"]).kitchen(n), 65536),
    "c4_clutter": ("dense clutter: 100 32-sphere-set objects on one table, 262144 variations/GPU",
                   lambda n: __import__("paper_2512_16896_b200.scenes", fromlist=["x"]).dense_clutter(n), 262144),
    "c5_sweep100": ("scale sweep point: 100 cuboids, 1048576 variations/GPU",
                    lambda n: __import__("paper_2512_16896_b200.scenes", fromlist=["x"]).scale_sweep(n, 100), 1 << 20),
    "c5_sweep10": ("scale sweep point: 10 cuboids, 1048576 variations/GPU",
                   lambda n: __import__("paper_2512_16896_b200.scenes", fromlist=["x"]).scale_sweep(n, 10), 1 << 20),
}


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML every 20 ms in a
    thread (nvidia-smi -lms 200 as the fallback when pynvml is unavailable)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int, period_s: float = 0.02):
        self.device = device
        self.period = period_s
        self.proc = None
        self.nvml = None
        self.lines = []
        self.samples = []  # (sm_mhz, max_mhz, set of reasons)
        self._stop = threading.Event()

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            idx = self.device
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                try:
                    idx = int(vis.split(",")[self.device])
                except (ValueError, IndexError):
                    pass
            self.nvml = (N, N.nvmlDeviceGetHandleByIndex(idx))
        except Exception:
            self.nvml = None
        if self.nvml is not None:
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _poll(self):
        N, h = self.nvml
        bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), float(mx), {k for k, b in bits.items() if r & b}))
            except Exception:
                pass
            self._stop.wait(self.period)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        self._stop.set()
        if self.nvml is None and self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        if self.nvml is not None:
            self.t.join(timeout=2)
            src = "nvml, every 20 ms"
        else:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            src = "nvidia-smi -lms 200"
            for ln in self.lines:
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    rs = {n for n, v in zip(self.NAMES, parts[2:6]) if v.lower() in ("active", "1")}
                    self.samples.append((float(parts[0]), float(parts[1]), rs))
                except ValueError:
                    continue
        sm = [a for a, _, _ in self.samples]
        mx = [b for _, b, _ in self.samples]
        reasons = set().union(*[r for _, _, r in self.samples]) if self.samples else set()
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_min_mhz": min(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "source": src}


def fp64_peak(device: int):
    """Measured FP64 pipe peak (GFLOP/s) for DADD / DMUL / DFMA (tools/fp64_peak.cu)."""
    path = os.path.join(ROOT, "tools", "libfp64peak.so")
    L = C.CDLL(path)
    L.sb_fp64_peak_gflops.restype = C.c_double
    L.sb_fp64_peak_gflops.argtypes = [C.c_int, C.c_int]
    return {"dadd": L.sb_fp64_peak_gflops(0, device), "dmul": L.sb_fp64_peak_gflops(1, device),
            "dfma": L.sb_fp64_peak_gflops(2, device)}


# Algorithmic FP64 operation counts: every op of the reference's
# expression trees, counted from the kernel's own work counters.
FLOPS = {
    "checked": 150,   # sample (sqrt, barycentric ~14) + point->world 15 + pose compose 84
                      # (shim Mat4 product rows 0-2) + candidate box 30 + inverse 18 - reuse
    "broad": 6,       # 6 comparisons per enabled object (counted as FP64 ops)
    "narrow": 84,     # other_in_cand = inv * pose (3x4 shim product)
    "nodes": 36,      # transform_aabb of the B node box (30) + 6 overlap comparisons
    "pairs": 46,      # first-plane test of tri_tri_intersect (the cost every pair pays)
}


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2512_16896_b200 as pkg

    desc, factory, n_default = WORKLOADS[args.config]
    n_per = args.n or n_default
    n_total = n_per * world
    scene = factory(n_total)
    # one process per GPU (local_rank modulo the visible devices, so a 2-rank run can also be
    # exercised on a single GPU)
    device = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(device)

    shard = comm = None
    if world > 1:
        # the engine's exchange is native (sb_comm: TCP bootstrap at MASTER_ADDR /
        # MASTER_PORT + 1, count boards mapped over NVLink / NVSwitch by CUDA IPC); the same
        # communicator provides the timing barrier and the max-over-ranks reduction
        comm = pkg.Comm(rank, world, device=device)
        shard = comm.shard(n_total)
    t0 = time.time()
    eng = pkg.Engine(scene, shard, device=device)
    cold_s = time.time() - t0
    P = len(scene.placements)

    # pinned host result buffers for the end-to-end leg
    acc = torch.empty((P, n_per), dtype=torch.int16).pin_memory()
    valid = torch.empty(n_per, dtype=torch.uint8).pin_memory()
    poses = torch.empty((P, n_per, 16), dtype=torch.float64).pin_memory()
    res = pkg._capi.sb_result(C.cast(acc.data_ptr(), C.POINTER(C.c_int16)),
                              C.cast(poses.data_ptr(), C.POINTER(C.c_double)),
                              C.cast(valid.data_ptr(), C.POINTER(C.c_uint8)))
    d2h = acc.numel() * 2 + valid.numel() + poses.numel() * 8
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{device}")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            comm.barrier()

    seed = 1
    for _ in range(args.warmup):
        eng.generate(seed, download=False)
    clocks = ClockSampler(device)
    clocks.start()
    step_ms, check_ms, check_launches, launches = [], [], [], []
    phases = {}
    agg = {}
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        r = eng.generate(seed, with_poses=False, download=False)
        barrier()
        total, chk, nchk = eng.last_timing()
        step_ms.append(total)
        check_ms.append(chk)
        check_launches.append(nchk)
        launches.append(eng.last_launches())
        for k, v in eng.phase_profile().items():
            phases[k] = phases.get(k, 0.0) + v / args.steps
        for k, v in r.stats.items():
            agg[k] = agg.get(k, 0) + v
    # end-to-end: same call, results D2H into pinned host memory, wall clock
    e2e_ms = []
    for _ in range(max(3, min(args.steps, 7))):
        flush.zero_()
        barrier()
        t = time.perf_counter()
        eng.generate_into(seed, res)
        barrier()
        e2e_ms.append((time.perf_counter() - t) * 1e3)
    clk = clocks.stop()

    K = args.steps
    mine = {"time_ms": sum(step_ms), "e2e_ms": statistics.median(e2e_ms),
            "valid": agg["valid_instances"] / K, "checks": agg["candidate_checks"] / K}
    if world > 1:
        keys = ("time_ms", "e2e_ms", "valid", "checks")
        bits = comm.allgather([struct.unpack("<Q", struct.pack("<d", float(mine[k])))[0] for k in keys])
        vals = [struct.unpack("<d", struct.pack("<Q", b))[0] for b in bits]
        per_rank = [dict(zip(keys, vals[4 * r:4 * r + 4])) for r in range(world)]
        time_ms = max(d["time_ms"] for d in per_rank)  # device time, max over ranks
        e2e = max(d["e2e_ms"] for d in per_rank)
        valid_sum = sum(d["valid"] for d in per_rank)
        checks_sum = sum(d["checks"] for d in per_rank)
    else:
        time_ms, e2e, valid_sum, checks_sum = (mine["time_ms"], mine["e2e_ms"], mine["valid"],
                                               mine["checks"])
    if rank != 0:
        return None
    ms_step = time_ms / K
    value = valid_sum / (ms_step * 1e-3)

    # Roofline of the dominant kernel, k_place (one cooperative launch per placement: every
    # attempt round's sample + compose + broad + narrow + accept). Algorithmic units are
    # SURVEY.md 8(d)'s: bytes = every placed object's pose (96 B) + world box (48 B) + enable
    # bit (1 B) read once per (instance, placement) + 150 B written per accepted candidate;
    # FP64 ops from the kernel's own work counters (FLOPS above). The binding roofline
    # (larger time at peak) is reported as `roofline`, the other as `roofline_secondary`.
    per = {k: agg.get(v, 0) / K for k, v in (("checked", "candidate_checks"),
                                              ("broad", "broad_phase_tests"),
                                              ("narrow", "narrow_phase_tests"),
                                              ("nodes", "node_pair_tests"),
                                              ("pairs", "triangle_pair_tests"),
                                              ("accepted", "accepted_candidates"))}
    flops = sum(FLOPS[k] * per[k] for k in FLOPS)
    n_fixed = len(scene.fixed)
    bytes_ = n_per * sum((n_fixed + k) * 145 for k in range(P)) + 150 * per["accepted"]
    k_ms = sum(check_ms) / K
    n_launch = sum(check_launches) / K
    peaks = fp64_peak(device)
    fp64_peak_tf = peaks["dadd"] / 1e3  # no-FMA build: one flop per FP64 instruction
    mp_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    measured = json.load(open(mp_path)) if os.path.exists(mp_path) else None
    hbm_peak = measured["hbm_gbs"] if measured else 6650.0
    hbm_src = "of measured (MEASURED_PEAKS.json hbm_gbs)" if measured else "of fallback (B200_PROFILING.md)"
    achieved_tf = flops / (k_ms * 1e-3) / 1e12 if k_ms > 0 else 0.0
    achieved_gbs = bytes_ / (k_ms * 1e-3) / 1e9 if k_ms > 0 else 0.0
    # dram__bytes_read.sum + dram__bytes_write.sum per launch (= per placement chain) from
    # the committed ncu capture of one warm generation (tools/gpu_traffic.sh)
    traffic = None
    prof_json = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(prof_json):
        traffic = json.load(open(prof_json)).get("dram_bytes_per_launch")
    hbm = {"bound": "hbm", "achieved": round(achieved_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
           "frac": round(achieved_gbs / hbm_peak, 5), "traffic": traffic,
           "peak_source": hbm_src, "algorithmic_bytes_per_launch": round(bytes_ / max(n_launch, 1)),
           "traffic_source": f"profiles/traffic_{args.config}.json" if traffic else None}
    if traffic and k_ms > 0 and n_launch > 0:
        # what the DRAM really moves: the per-instance occupancy grid and the shared-memory
        # tile state skip most of SURVEY 8(d)'s per-object reads, so `achieved` (algorithmic
        # bytes) overstates the DRAM use; this is the measured traffic over the same time
        dram_gbs = traffic * n_launch / (k_ms * 1e-3) / 1e9
        hbm.update({"dram_achieved": round(dram_gbs, 1), "dram_frac": round(dram_gbs / hbm_peak, 5),
                    "traffic_vs_algorithmic": round(traffic / max(bytes_ / max(n_launch, 1), 1), 4),
                    "note": "achieved/frac use SURVEY 8(d)'s algorithmic bytes (every placed "
                            "object's pose+box+enable read per instance and placement); the "
                            "occupancy grid reads only the candidate cells' objects, so frac can "
                            "exceed 1 -- dram_achieved/dram_frac are the measured DRAM bytes "
                            "(ncu, cold caches) over the same time; the chain is latency-bound"})
    fp64 = {"bound": "fp64", "achieved": round(achieved_tf, 3), "peak": round(fp64_peak_tf, 3),
            "unit": "TFLOP/s", "frac": round(achieved_tf / fp64_peak_tf, 5) if fp64_peak_tf > 0 else None,
            "peak_source": "measured in this run: DADD rate, tools/fp64_peak.cu (no-FMA build)",
            "algorithmic_flops_per_launch": round(flops / max(n_launch, 1))}
    t_hbm = bytes_ / (hbm_peak * 1e9)
    t_fp64 = flops / (fp64_peak_tf * 1e12) if fp64_peak_tf > 0 else 0.0
    primary, secondary = (hbm, fp64) if t_hbm >= t_fp64 else (fp64, hbm)
    # One "launch" here is one placement's kernel chain on the engine stream. The chains are
    # timed by CUDA events on that stream around the whole generation (per-placement events
    # would break the programmatic-launch edges between the kernels; SB_PLACE_EVENTS=1 puts
    # them back), so kernel_ms_per_step also holds the run's reset / grid-init kernels: FIFO placements of large batches run round 0 as k_fast_init +
    # k_wide_scan + k_wide_sample + k_wide_filter + k_wide_narrow + k_wide_accept +
    # k_wide_scan + k_wide_spread and later rounds in the persistent k_place; other
    # placements are one k_place (or k_place_instances). Per-kernel shares: the committed
    # ncu launch list (profiles/).
    for r in (primary, secondary):
        r.update({"kernel": "placement kernel chain (k_wide_* round 0 + persistent k_place; "
                            "per-kernel shares in profiles/ launch lists)",
                  "kernel_ms_per_step": round(k_ms, 4), "launches_per_step": n_launch,
                  "share_of_step": round(k_ms / ms_step, 4)})
    line = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "collision-free scenes/s",
        "checks_per_s": round(checks_sum / (ms_step * 1e-3), 1),
        "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic scene of the named shape, seeded (no assets/network); run_seed 1",
        "config": workload_config(args, world, scene),
        "valid_fraction": round(valid_sum / n_total, 4),
        "l2": "flushed (256 MiB write) between timed steps",
        "cold_start_s": round(cold_s, 3),
        "roofline": primary,
        "roofline_secondary": secondary,
        "fp64_peaks_gflops": {k: round(v, 1) for k, v in peaks.items()},
        "work_per_step": {k: round(v) for k, v in per.items()},
        "e2e": {"value": round(valid_sum / (e2e * 1e-3), 1), "unit": "collision-free scenes/s",
                "ms_per_step": round(e2e, 4), "h2d_bytes_per_step": 8,
                "d2h_bytes_per_step": int(d2h),
                "path": "sb_engine_generate with pinned host sb_result (accepted, valid, poses)"},
        "gpu_launches": round(statistics.mean(launches)) * K,
        "phase_profile_per_step": {k: round(v, 4) for k, v in phases.items()},
        "clocks": clk,
    }
    if not args.no_cpu_baseline and world == 1:  # rank 0 at N=1 only
        line["cpu_baseline"] = cpu_baseline(args)
    return line


def workload_config(args, world, scene):
    """The `config` object, identical in both arms (--impl ours / reference)."""
    desc, _, n_default = WORKLOADS[args.config]
    n_per = args.n or n_default
    return {"workload": f"{args.config}: {desc}", "n_instances_per_gpu": n_per,
            "n_instances_total": n_per * world, "placements": len(scene.placements),
            "candidates_per_object": scene.attempts,
            "parallelism": f"dp{world} (variation shards)"}


# Variations per reference step: a bounded sample of the workload (the same scene, fewer
# variations), so `--steps K --warmup W` of the CPU reference ends within minutes. Per-
# variation CPU work does not depend on N (the fast path's shared stream only orders the
# draws), so scenes/s over the sample is the reference's rate on the workload.
REF_SAMPLE = {"c1_tabletop": 1024, "c2_mixed": 16384, "c3_kitchen": 8192, "c4_clutter": 8192,
              "c5_sweep100": 32768, "c5_sweep10": 262144}


def reference_scene(args, n):
    """The workload's scene built with the reference's own mesh constructors and
    support-surface extraction (oracle/_ref: trimesh.cpp make_box / make_cylinder /
    make_sphere, transform_point; surface.cpp extract_support_surfaces)."""
    from oracle import oracle as O
    from paper_2512_16896_b200 import scenes
    from paper_2512_16896_b200.world import TriMesh

    prims = {"extract_support_surfaces": lambda m, mode: [
                 (poly, frame.reshape(4, 4).T)
                 for poly, frame, _, _ in O.extract_support_surfaces(m.vertices, m.triangles, mode)],
             "make_box": lambda sx, sy, sz: TriMesh(*O.make_box(sx, sy, sz)),
             "make_cylinder": lambda r, h, seg=32: TriMesh(*O.make_cylinder(r, h, seg)),
             "make_sphere": lambda r, st=12, sl=16: TriMesh(*O.make_sphere(r, st, sl)),
             "transformed": lambda m, pose: TriMesh(O.transformed_vertices(m.vertices, pose),
                                                    m.triangles.copy())}
    with scenes.mesh_source(**prims):
        return WORKLOADS[args.config][1](n)


def time_reference(scene, steps, warmup, threads):
    """Warm generation passes of the reference (RefEngine: cold part outside the timer)."""
    from oracle import oracle as O

    eng = O.RefEngine(scene, threads)
    for _ in range(warmup):
        eng.generate(1)
    times, valid, checks = [], 0, 0
    for _ in range(steps):
        t = time.perf_counter()
        r = eng.generate(1)
        times.append(time.perf_counter() - t)
        valid += r["stats"]["valid_instances"]
        checks += r["stats"]["candidate_checks"]
    eng.close()
    return sum(times), valid, checks


def cpu_baseline(args, budget_s=12.0):
    """The reference (oracle/_ref) on the host cores, rank 0 at N=1: warm passes over a
    bounded sample of the workload for about `budget_s` seconds."""
    threads = os.cpu_count() or 1
    n = args.cpu_n or min(REF_SAMPLE[args.config], WORKLOADS[args.config][2], 4096)
    scene = reference_scene(args, n)
    total = valid = checks = passes = 0
    while total < budget_s and passes < 50:
        dt, v, c = time_reference(scene, 1, 1 if passes == 0 else 0, threads)
        total += dt
        valid += v
        checks += c
        passes += 1
    return {"value": round(valid / total, 1), "unit": "collision-free scenes/s",
            "checks_per_s": round(checks / total, 1), "cores": threads, "kind": "reference",
            "sample": f"{passes} warm generation pass(es) of the workload's scene at {n} "
                      f"variations ({total:.1f} s timed, ThreadPool({threads}))"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path on this host (rank 0 only)."""
    if rank != 0:
        return None
    desc, _, n_default = WORKLOADS[args.config]
    n_cfg = args.n or n_default
    n = min(n_cfg, args.ref_n or REF_SAMPLE[args.config])
    scene = reference_scene(args, n)
    threads = os.cpu_count() or 1
    total, valid, checks = time_reference(scene, args.steps, args.warmup, threads)
    value = valid / total
    sample = (f"each step: one warm generation pass of the workload's scene over {n} of its "
              f"{n_cfg} variations per GPU (bounded sample; ThreadPool({threads}))")
    return {
        "impl": "reference", "metric": METRIC, "value": round(value, 1),
        "unit": "collision-free scenes/s", "checks_per_s": round(checks / total, 1),
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic scene of the named shape, seeded (no assets/network); run_seed 1",
        "config": workload_config(args, world, scene),
        "valid_fraction": round(valid / (n * args.steps), 4),
        "sample": sample,
        "cpu_baseline": {"value": round(value, 1), "unit": "collision-free scenes/s",
                         "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": round(value, 1), "unit": "collision-free scenes/s",
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4_clutter", choices=sorted(WORKLOADS))
    ap.add_argument("--n", type=int, default=0, help="variations per GPU (default: config's)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-n", type=int, default=0)
    ap.add_argument("--ref-n", type=int, default=0,
                    help="--impl reference: variations per step (default: REF_SAMPLE)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        # rank 0 alone times the reference; no process group, nothing of this package's
        # library is loaded in this process
        line = run_reference(args, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    line = run_ours(args, rank, world, local_rank)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
