"""BASELINE C5 at full size against reference digests (tests/golden/make_scale_digests.py):
2^20 variations x {10, 50, 100} cuboids, plus the 100-object sweep at 2^10 and 2^16.
Accepted attempt indices and valid masks must hash to the reference's sha256 (bit-exact),
the work counters must equal the reference's, and a seeded sample of accepted poses must
equal the reference's (bit-exact; the tolerance fallback is north_star's 1e-5)."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2512_16896_b200 import scenes

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
DIGESTS = json.load(open(os.path.join(GOLD, "scale_digests.json")))
FACTORY = {
    "c5_1M_x10": lambda: scenes.scale_sweep(1 << 20, 10),
    "c5_1M_x50": lambda: scenes.scale_sweep(1 << 20, 50),
    "c5_1M_x100": lambda: scenes.scale_sweep(1 << 20, 100),
    "c5_64k_x100": lambda: scenes.scale_sweep(1 << 16, 100),
    "c5_1k_x100": lambda: scenes.scale_sweep(1 << 10, 100),
}
COUNTERS = ("valid_instances", "candidates_sampled", "candidate_checks", "narrow_phase_tests",
            "rounds", "per_instance_placements")


@pytest.mark.parametrize("name", sorted(n for n in FACTORY if n in DIGESTS))
def test_scale_digest(gpu, name):
    d = DIGESTS[name]
    scene = FACTORY[name]()
    assert scene.n_instances == d["n"] and len(scene.placements) == d["placements"]
    eng = gpu.Engine(scene)
    got = eng.generate(d["run_seed"], with_poses=False)
    acc = np.ascontiguousarray(got.accepted, np.int16)
    assert hashlib.sha256(acc.tobytes()).hexdigest() == d["accepted_sha256"], \
        f"accepted indices differ (hist {np.bincount(acc.ravel() + 1)[:8]} vs {d['accepted_hist']})"
    assert hashlib.sha256(np.ascontiguousarray(got.valid, np.uint8).tobytes()).hexdigest() == \
        d["valid_sha256"]
    for k in COUNTERS:
        assert got.stats[k] == d["stats"][k], k
    # seeded pose sample, read from the engine's world (object = n_fixed + placement)
    rng = np.random.default_rng(d["pose_sample_seed"])
    S = len(np.load(os.path.join(GOLD, f"scale_{name}.npz"))["poses"])
    pi, ii = rng.integers(0, d["placements"], S), rng.integers(0, d["n"], S)
    want = np.load(os.path.join(GOLD, f"scale_{name}.npz"))["poses"]
    w = eng.world()
    nf = len(scene.fixed)
    exact = checked = 0
    for k in range(S):
        if acc[pi[k], ii[k]] < 0:
            continue
        mine = gpu.colmajor(w.object_pose(nf + int(pi[k]), int(ii[k])))
        assert np.allclose(mine, want[k], rtol=1e-5, atol=1e-12)
        exact += int(np.array_equal(mine, want[k]))
        checked += 1
    assert checked > 0
    print(f"{name}: {exact}/{checked} sampled poses bit-exact")
