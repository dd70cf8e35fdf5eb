# Host-side overhead of one generate call (C2): Python wrapper vs the C++ call vs device time.
# Run with SB_HOST_TIMES=1 for the C++ breakdown (enqueue / wait / after).
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import paper_2512_16896_b200 as pkg
from paper_2512_16896_b200 import _capi as A, scenes

eng = pkg.Engine(scenes.tabletop_mixed(16384))
L = A.lib()
st = A.sb_run_stats()
for _ in range(6):
    t = time.perf_counter()
    rc = L.sb_engine_generate(eng._h, 1, None, C.byref(st))
    t1 = time.perf_counter()
    print("raw ctypes call %.1f us (rc %d), device %.1f us, py t %.1f t1 %.1f" % (
        (t1 - t) * 1e6, rc, eng.last_timing()[0] * 1e3, t * 1e6, t1 * 1e6), file=sys.stderr)
for _ in range(3):
    t = time.perf_counter()
    eng.generate(1, with_poses=False, download=False)
    print("Engine.generate %.1f us" % ((time.perf_counter() - t) * 1e6), file=sys.stderr)
