import math, sys, numpy as np
sys.path.insert(0, ".")
import paper_2512_16896_b200 as pkg
from paper_2512_16896_b200 import _capi as A, scenes
from oracle import oracle as O
base = scenes.tabletop_boxes(1024, n_objects=8, table=(1.6, 1.2))
rels = {
    2: pkg.Relation(anchor=1, distance_type=A.SB_DIST_GREATER, direction=A.SB_DIR_FRONT, distance=0.2, angle_threshold=math.pi / 3),
    3: pkg.Relation(anchor=0, distance_type=A.SB_DIST_EQUAL, direction=A.SB_DIR_VECTOR, direction_vector=(0.3, -0.4), distance=0.3, frame=A.SB_FRAME_LOCAL),
    5: pkg.Relation(anchor=4, distance_type=A.SB_DIST_LESS, distance=0.35),
    6: pkg.Relation(anchor=2, direction=A.SB_DIR_RIGHT, frame=A.SB_FRAME_LOCAL),
}
for k, r in rels.items(): base.placements[k].relation = r
base.placements[4].orientation = A.SB_ORIENT_FACE_TO; base.placements[4].face_target = 0
base.placements[7].orientation = A.SB_ORIENT_FIXED
got = pkg.Engine(base).generate(3)
want = O.generate(base, 3, threads=8)
ref = pkg.from_colmajor(want["poses"])
bad = np.argwhere(~np.isclose(got.poses, ref, rtol=1e-5, atol=1e-12))
print("accepted equal", np.array_equal(got.accepted, want["accepted"]))
for p, i, r, c in bad[:20]:
    print(p, i, r, c, repr(got.poses[p, i, r, c]), repr(ref[p, i, r, c]), "acc", got.accepted[p, i])
# exact-equality census per placement
for p in range(len(base.placements)):
    eq = (got.poses[p] == ref[p]).all(axis=(1, 2))
    print("placement", p, "exactly equal poses:", eq.sum(), "/", len(eq))
