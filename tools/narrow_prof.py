# Narrow-phase cycle breakdown (needs SB_LIB_PATH=.../libscenebatch_b200_prof.so).
import ctypes as C, sys, time
sys.path.insert(0, ".")
import paper_2512_16896_b200 as pkg
from paper_2512_16896_b200 import _capi as A, scenes
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
sc = scenes.scale_sweep(65536, 100) if cfg == "c5" else scenes.tabletop_mixed(16384)
eng = pkg.Engine(sc)
eng.generate(1, with_poses=False, download=False)
out = (C.c_uint64 * 8)()
A.check(A.lib().sb_debug_narrow_profile(out))
eng.generate(1, with_poses=False, download=False)
A.check(A.lib().sb_debug_narrow_profile(out))
v = list(out); pairs = max(1, v[5])
names = ["M", "B nodes+leaf", "walk rows", "walk", "-", "-", "filter1", "filter2+rest"]
print(cfg, "pairs", pairs, {n: round(v[i] / pairs) for i, n in enumerate(names) if n != "-"})
