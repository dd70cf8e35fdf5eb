"""GPU: the CUDA path against the golden fixtures produced by the reference itself
(tests/golden/make_golden.py). Accepted attempt indices, valid masks and check_batch
masks bit-exact; poses within the north_star 1e-5 bar (bit-exact except for glibc's own
sin/cos misroundings, see DESIGN.md libm)."""
import os

import numpy as np
import pytest

from tests.test_golden import GOLD, SCENE_NAMES, _world_meshes, scene

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", SCENE_NAMES)
def test_generation_matches_golden(gpu, name):
    g = np.load(os.path.join(GOLD, f"gen_{name}.npz"))
    got = gpu.Engine(scene(name)).generate(7)
    assert np.array_equal(got.accepted, g["accepted"])
    assert np.array_equal(got.valid, g["valid"])
    want = gpu.from_colmajor(g["poses"])
    assert np.allclose(got.poses, want, rtol=1e-5, atol=1e-12)
    exact = (got.poses == want).all(axis=(2, 3)).mean()
    assert exact > 0.95, exact
    st = got.stats
    assert [st["valid_instances"], st["candidate_checks"], st["narrow_phase_tests"], st["rounds"],
            st["per_instance_placements"]] == [int(x) for x in g["stats"]]


@pytest.mark.parametrize("k", [0, 1, 2])
def test_check_batch_matches_golden(gpu, k):
    g = np.load(os.path.join(GOLD, f"world{k}.npz"))
    n = g["poses"].shape[1]
    W = gpu.CollisionWorld(n)
    gids = [W.register_geometry(m) for m in _world_meshes()]
    for o, mi in enumerate(g["obj_mesh"]):
        obj = W.add_object(f"o{o}", gids[int(mi)])
        W.update_transforms(obj, gpu.from_colmajor(g["poses"][o]))
        W.set_enabled(obj, np.nonzero(g["enabled"][o])[0], True)
    free, contact = W.check_batch(gids[int(g["cand_mesh"])], gpu.from_colmajor(g["cand"]),
                                  g["active"])
    assert np.array_equal(free, g["free"]) and np.array_equal(contact, g["contact"])
