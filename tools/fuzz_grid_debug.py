# Inspect a failing occupancy-grid fuzz seed: which placements / instances differ and how.
import sys
sys.path.insert(0, ".")
import importlib.util
import numpy as np
spec = importlib.util.spec_from_file_location("f", "tests/test_gpu_fuzz.py")
f = importlib.util.module_from_spec(spec)
spec.loader.exec_module(f)
import paper_2512_16896_b200 as pkg
from oracle import oracle as O
seed = int(sys.argv[1])
sc = f.random_scene(pkg, 5000 + seed, n_range=(33, 49), sizes=(64, 300))
g = pkg.Engine(sc).generate(seed + 1)
w = O.generate(sc, seed + 1, threads=8)
print("valid", g.valid.sum(), w["valid"].sum(), "stats", {k: (g.stats[k], w["stats"][k]) for k in ("candidate_checks", "narrow_phase_tests", "rounds")})
d = np.argwhere(g.accepted != w["accepted"])
print("n objects", len(sc.placements), "N", sc.n_instances, "mismatches", len(d))
for p, i in d[:8]:
    pl = sc.placements[p]
    print(" placement", p, "inst", i, "got", g.accepted[p, i], "ref", w["accepted"][p, i], "rel", pl.relation, "orient", pl.orientation, "ratio", pl.ratio_on_support)
