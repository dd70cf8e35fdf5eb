# Region-kernel stage cycles per instance (needs SB_LIB_PATH=.../libscenebatch_b200_prof.so).
import ctypes as C
import sys

sys.path.insert(0, ".")
import paper_2512_16896_b200 as pkg
from paper_2512_16896_b200 import _capi as A, scenes

sc = scenes.tabletop_mixed(16384) if (len(sys.argv) < 2 or sys.argv[1] == "c2") else scenes.kitchen(65536)
eng = pkg.Engine(sc)
eng.generate(1, with_poses=False, download=False)
out = (C.c_uint64 * 8)()
A.check(A.lib().sb_debug_region_profile(out))
eng.generate(1, with_poses=False, download=False)
A.check(A.lib().sb_debug_region_profile(out))
v = list(out)
n = max(1, v[7])
names = ["anchor", "band/bounds", "arc", "orient+clips", "dedupe+area", "tri+fan", "table"]
print("instances", n, {k: round(v[i] / n) for i, k in enumerate(names)}, "regions_ms", round(eng.phase_profile()["regions_ms"], 3))
