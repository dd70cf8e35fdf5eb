"""Reference driver (CPU) with per-instance support frames: a surface on an earlier
placed object follows that object's accepted pose (stacking), and a support given as a
batch of frames moves per instance."""
import numpy as np

import paper_2512_16896_b200 as pkg
from tests.test_gpu_support_frames import stacking_scene


def test_stacked_boxes_rest_on_the_crate(ref):
    scene = stacking_scene(pkg, 64)
    r = ref.generate(scene, 5, threads=2)
    poses = pkg.from_colmajor(r["poses"])
    ok = (r["accepted"][0] >= 0) & (r["accepted"][1] >= 0)
    assert ok.sum() > 10
    crate, box = poses[0][ok], poses[1][ok]
    # the stacked box's origin, expressed in the crate frame, lies over the crate's top rect
    rel = np.einsum("nij,njk->nik", np.linalg.inv(crate), box)
    assert np.all(np.abs(rel[:, 0, 3]) <= 0.15 + 1e-9) and np.all(np.abs(rel[:, 1, 3]) <= 0.125 + 1e-9)
    assert np.all(rel[:, 2, 3] > 0.04)


def test_support_batch_moves_per_instance(ref):
    scene = stacking_scene(pkg, 32)
    shift = np.tile(np.eye(4), (32, 1, 1))
    shift[:, 0, 3] = np.linspace(-0.3, 0.3, 32)
    shift[:, 2, 3] = 0.75
    scene.supports[0].poses = shift  # the table surface, moved per instance
    r = ref.generate(scene, 5, threads=2)
    poses = pkg.from_colmajor(r["poses"])
    ok = r["accepted"][0] >= 0
    x = poses[0][ok][:, 0, 3] - shift[ok][:, 0, 3]
    assert np.all(np.abs(x) <= 0.6 + 1e-9)
