"""Throughput of the widened components against the reference on the host cores (same
inputs): standalone PositionSampler.sample (FIFO path), BatchedSceneGraph.world_poses
(batched FK, depth 5), ReachMap4D build and query_batch. One JSON line per component:
`device` = wall clock of the host-buffer C-ABI call (H2D + kernel + D2H) after warm-up,
median of 5; `device_resident` = the *_device variant on device buffers, CUDA events on
its stream; `reference` = the reference's own call (1 thread unless stated)."""
import json
import math
import os
import statistics
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import torch

import paper_2512_16896_b200 as pkg
from oracle import oracle as O
from tests import graph_cases as G
from tests import reach_cases as RC
from tests import sampler_cases as S

THREADS = os.cpu_count() or 8


def med(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return statistics.median(ts)


def dev_time(fn, reps=10):
    st = torch.cuda.Stream()
    fn(st)
    st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn(st)
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps


def cm(p):
    return np.ascontiguousarray(np.swapaxes(p, -1, -2)).reshape(p.shape[:-2] + (16,))


def line(name, units, dev_s, ref_s, unit, extra=None):
    d = {"component": name, "unit": unit, "device": round(units / dev_s, 1),
         "reference": round(units / ref_s, 1), "speedup": round(ref_s / dev_s, 1),
         "reference_threads": 1}
    d.update(extra or {})
    print(json.dumps(d), flush=True)


# ---- PositionSampler.sample, FIFO path: 1M active instances per call
n = 1 << 20
sup = np.tile(np.eye(4), (n, 1, 1))
sup[:, :3, 3] = np.random.default_rng(0).uniform(-1, 1, (n, 3))
act = np.arange(n, dtype=np.uint32)
D = S.DeviceAdapter(pkg, 3)
R = S.RefAdapter(O, 3)
D.prepare([S.RECT], n, 1, False)
R.prepare([S.RECT], n, 1, False)
ds = med(lambda: D.sample(sup, act, 0))
rs = med(lambda: R.sample(sup, act, 0), reps=3)
dsup = torch.tensor(cm(sup), device="cuda")
dact = torch.tensor(act.astype(np.int32), device="cuda")
dpos = torch.empty((n, 3), dtype=torch.float64, device="cuda")
dpl = torch.empty(n, dtype=torch.uint8, device="cuda")
dr = dev_time(lambda st: D.s.sample_device(dsup.data_ptr(), dact.data_ptr(), n, 0, dpos.data_ptr(),
                                            dpl.data_ptr(), st.cuda_stream))
line("PositionSampler.sample (FIFO, 1M active)", n, ds, rs, "positions/s",
     {"device_resident": round(n / dr, 1)})

# ---- BatchedSceneGraph.world_poses of a depth-5 node, 1M instances
n = 1 << 20
gd, gr = pkg.BatchedSceneGraph(n), O.RefGraph(n)
rng = np.random.default_rng(1)
parent_d = parent_r = 0
for k in range(5):
    e = G.rigid(rng, n)
    parent_d_new = gd.add_node(parent_d, f"n{k}")
    parent_r_new = gr.add_node(parent_r, f"n{k}")
    gd.set_edge_batch(parent_d, parent_d_new, e)
    gr.set_edge_batch(parent_r, parent_r_new, e)
    parent_d, parent_r = parent_d_new, parent_r_new
ds = med(lambda: gd.world_poses(parent_d))
rs = med(lambda: gr.world_poses(parent_r), reps=3)
dout = torch.empty((n, 16), dtype=torch.float64, device="cuda")
dr = dev_time(lambda st: gd.world_poses_device(parent_d, dout.data_ptr(), st.cuda_stream))
line("BatchedSceneGraph.world_poses (depth 5, 1M)", n, ds, rs, "poses/s",
     {"device_resident": round(n / dr, 1),
      "hbm_gbs": round(n * (5 * 96 + 128) / dr / 1e9, 1)})

# ---- ReachMap4D: build (2M FK samples) and query_batch (1M)
ch = RC.arm()
t = time.perf_counter()
Rm = O.RefReachMap.build(ch, 2_000_000, 0.02, math.pi / 8, seed=3, threads=THREADS)
rb = time.perf_counter() - t
db = med(lambda: pkg.ReachMap4D.build(ch, 2_000_000, 0.02, math.pi / 8, seed=3), reps=3)
d = {"component": "ReachMap4D.build (2M FK samples)", "unit": "samples/s",
     "device": round(2e6 / db, 1), "reference": round(2e6 / rb, 1), "speedup": round(rb / db, 1),
     "reference_threads": THREADS}
print(json.dumps(d), flush=True)
Dm = pkg.ReachMap4D.build(ch, 2_000_000, 0.02, math.pi / 8, seed=3)
n = 1 << 20
B, T = RC.bases(n, 1), RC.targets(n, 1)
ds = med(lambda: Dm.query_batch(B, T))
rs = med(lambda: Rm.query_batch(B, T), reps=3)
db, dt = torch.tensor(cm(B), device="cuda"), torch.tensor(T, device="cuda")
dq = torch.empty(n, dtype=torch.uint8, device="cuda")
dr = dev_time(lambda st: Dm.query_batch_device(db.data_ptr(), dt.data_ptr(), n, dq.data_ptr(),
                                               None, st.cuda_stream))
line("ReachMap4D.query_batch (1M)", n, ds, rs, "queries/s", {"device_resident": round(n / dr, 1)})
