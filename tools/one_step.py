"""One warm generation of a bench workload between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists and captures:
  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file x.csv \
      python tools/one_step.py c4_clutter [n]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2512_16896_b200 as pkg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4_clutter"
desc, factory, n_default = bench.WORKLOADS[cfg]
n = int(sys.argv[2]) if len(sys.argv) > 2 else n_default
eng = pkg.Engine(factory(n))
eng.generate(1, with_poses=False, download=False)
import torch  # noqa: E402

torch.cuda.synchronize()
torch.cuda.profiler.start()
r = eng.generate(1, with_poses=False, download=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(cfg, n, eng.last_timing(), r.stats)
