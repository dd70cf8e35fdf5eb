# Isolated narrow-phase latency: ONE warp runs warp_collide on one (candidate, object)
# pair through the world API check_batch (needs SB_LIB_PATH=.../libscenebatch_b200_prof.so).
# Prints per-stage cycles (no contention from other warps) for a few pair kinds.
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2512_16896_b200 as pkg
from paper_2512_16896_b200 import _capi as A, scenes
from paper_2512_16896_b200.world import make_box, translation

names = ["M", "B nodes+leaf", "walk rows", "walk", "-", "-", "filter1", "filter2+rest"]


def run(label, mesh_a, mesh_b, pose_b, pose_a, reps=20):
    W = pkg.CollisionWorld(1)
    ga = W.register_geometry(mesh_a)
    gb = W.register_geometry(mesh_b)
    ob = W.add_object("b", gb)
    W.update_transform(ob, 0, pose_b)
    W.set_enabled(ob, [0], True)
    out = (C.c_uint64 * 8)()
    A.check(A.lib().sb_debug_narrow_profile(out))  # reset
    free = None
    for _ in range(reps):
        free, _ = W.check_batch(ga, pose_a[None], [0])
    A.check(A.lib().sb_debug_narrow_profile(out))
    v = list(out)
    calls = max(1, v[5])
    print(f"{label:28s} free={int(free[0])} calls={calls}",
          {n: round(v[i] / calls) for i, n in enumerate(names) if n != "-"})
    W.close()


rng = scenes.Pcg32(5)
ss_a = scenes.sphere_set(rng)
ss_b = scenes.sphere_set(rng)
box = make_box(0.08, 0.08, 0.08)
box2 = make_box(0.1, 0.06, 0.08)
# overlapping sphere sets (hit), near-miss sphere sets (AABB overlap, no hit), boxes
run("sphere-set same mesh hit", ss_a, ss_a, translation(0.0, 0.0, 0.0), translation(0.004, 0.0, 0.0))
run("sphere-set hit?", ss_a, ss_b, translation(0.0, 0.0, 0.0), translation(0.005, 0.0, 0.0))
run("sphere-set aabb-only", ss_a, ss_b, translation(0.0, 0.0, 0.0), translation(0.055, 0.055, 0.0))
run("box-box hit", box, box2, translation(0.0, 0.0, 0.041), translation(0.05, 0.0, 0.041))
run("box-box coplanar touch", box, box2, translation(0.0, 0.0, 0.041), translation(0.0899, 0.0, 0.041))
run("box-box apart", box, box2, translation(0.0, 0.0, 0.041), translation(0.3, 0.0, 0.041))
