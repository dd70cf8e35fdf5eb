"""CPU: the oracle's margin > 0 path (tri_tri_distance, collision.cpp:136-212,312-313) is
live -- a positive margin turns near misses into collisions -- so the GPU margin parity
cases in test_gpu_parity.py compare two non-trivial masks."""
import math

import numpy as np


def test_margin_turns_near_misses_into_hits(ref, pkg):
    box = pkg.make_box(0.1, 0.1, 0.1)
    n = 64
    res = {}
    for margin in (0.0, 0.01):
        R = ref.RefWorld(n, margin)
        g = R.register_geometry(box.vertices, box.triangles)
        o = R.add_object(g)
        poses = np.stack([np.eye(4)] * n)
        R.update_transforms(o, pkg.colmajor(poses))
        R.set_enabled(o, np.arange(n, dtype=np.uint32), True)
        cand = np.stack([np.eye(4)] * n)
        # gaps 0 .. 12 mm along the effective (-x face) side, yaw 0
        cand[:, 0, 3] = -(0.1 + np.linspace(0.0, 0.012, n))
        free, contact = R.check_batch(g, pkg.colmajor(cand), np.arange(n, dtype=np.uint32))
        res[margin] = free.copy()
    # every instance free at margin 0 past contact; within 10 mm some collide with margin
    assert res[0.0][n // 2:].all()
    assert (res[0.01] == 0).sum() > (res[0.0] == 0).sum()
