"""Randomised scenes (seeded; every run the same): random mixes of boxes, cylinders, UV
spheres and sphere sets on a random table, random relations (distance bands incl. holes,
axis / vector / local-frame directions, angle thresholds), orientations (uniform, fixed,
face_to), ratio_on_support, attempt budgets and sizes -- the device engine against the
reference driver: accepted indices, valid masks, counters and accepted poses bit-exact."""
import math

import numpy as np
import pytest

from paper_2512_16896_b200 import _capi as A
from paper_2512_16896_b200 import scenes
from paper_2512_16896_b200.world import Fixed, Placement, Relation, Scene, Support, translation
from tests.test_gpu_parity import POSE_ATOL, POSE_RTOL, run_generate_pair

pytestmark = pytest.mark.gpu


def random_scene(pkg, seed, n_range=(4, 12), sizes=(1, 37, 256, 700)):
    rng = np.random.default_rng(seed)
    srng = scenes.Pcg32(1000 + seed)
    tx, ty = rng.uniform(0.8, 2.0), rng.uniform(0.6, 1.4)
    tmesh = pkg.make_box(tx, ty, 0.75)
    meshes = [tmesh]
    sup = Support(translation(0.0, 0.0, 0.75), (-tx / 2, -ty / 2, tx / 2, ty / 2))
    n_obj = int(rng.integers(*n_range))
    places = []
    for k in range(n_obj):
        kind = rng.integers(4)
        if kind == 0:
            m = pkg.make_box(*rng.uniform(0.03, 0.14, 3))
        elif kind == 1:
            m = pkg.make_cylinder(rng.uniform(0.02, 0.06), rng.uniform(0.04, 0.15),
                                  int(rng.integers(6, 20)))
        elif kind == 2:
            m = pkg.make_sphere(rng.uniform(0.02, 0.07), int(rng.integers(4, 9)),
                                int(rng.integers(5, 12)))
        else:
            m = scenes.sphere_set(srng)
        meshes.append(m)
        rel = Relation()
        ratio = 0.0
        if k > 0 and rng.random() < 0.5:
            anchor = int(rng.integers(k))
            dt = int(rng.choice([A.SB_DIST_NONE, A.SB_DIST_LESS, A.SB_DIST_GREATER, A.SB_DIST_EQUAL]))
            dr = int(rng.choice([A.SB_DIR_NONE, A.SB_DIR_LEFT, A.SB_DIR_RIGHT, A.SB_DIR_FRONT,
                                 A.SB_DIR_BACK, A.SB_DIR_VECTOR]))
            dist = float(rng.uniform(0.1, 0.5))
            theta = float(rng.choice([0.0, math.pi / 6, math.pi / 2, 2.0]))
            rel = Relation(anchor=anchor, distance_type=dt, direction=dr,
                           frame=int(rng.integers(2)) if dr != A.SB_DIR_NONE else 0,
                           direction_vector=tuple(rng.normal(size=2)), distance=dist,
                           angle_threshold=theta)
        elif rng.random() < 0.3:
            ratio = float(rng.uniform(0.1, 1.0))
        orient = int(rng.choice([A.SB_ORIENT_UNIFORM_YAW, A.SB_ORIENT_FIXED, A.SB_ORIENT_FACE_TO]))
        face = -1
        if orient == A.SB_ORIENT_FACE_TO:
            if k == 0:
                orient = A.SB_ORIENT_UNIFORM_YAW
            else:
                face = int(rng.integers(k))
        places.append(Placement(mesh=len(meshes) - 1, support=0, orientation=orient,
                                face_target=face, relation=rel, ratio_on_support=ratio))
    n = int(rng.choice(list(sizes)))
    return Scene(f"fuzz{seed}", n, int(rng.choice([8, 32, 64])), meshes,
                 [Fixed(0, translation(0.0, 0.0, 0.375))], [sup], places)


def check_against_reference(gpu, scene, got, want):
    """Bit-exact: accepted indices, valid masks, the reference's work counters and the
    accepted poses themselves (the device libm is glibc's, sb_glibcm.cuh, so even the
    local-frame chain anchor yaw -> direction -> arc points reproduces the reference)."""
    assert np.array_equal(got.valid, want["valid"]), "valid mask differs"
    diff = np.argwhere(got.accepted != want["accepted"])
    assert len(diff) == 0, f"accepted differs at (placement, inst) {diff[:10].tolist()}"
    refp = gpu.from_colmajor(want["poses"])
    placed = got.accepted >= 0
    same = (got.poses == refp).all(axis=(2, 3))
    assert same[placed].all(), f"{np.sum(~same[placed])} accepted poses differ"
    for k in ("valid_instances", "candidate_checks", "narrow_phase_tests", "rounds"):
        assert got.stats[k] == want["stats"][k], k


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("SB_FUZZ_SEEDS", "48"))))
def test_fuzz_engine_matches_reference(gpu, ref, seed):
    scene = random_scene(gpu, seed)
    eng, got, want = run_generate_pair(gpu, ref, scene, seed=seed + 1)
    check_against_reference(gpu, scene, got, want)

@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("SB_FUZZ_WIDE_SEEDS", "16"))))
def test_fuzz_wide_round0_matches_reference(gpu, ref, seed, monkeypatch):
    """The grid-wide round 0 (k_wide_*; normally from 131,072 instances) forced onto the
    random scenes: every FIFO placement without a relation takes it, the rest keep the
    persistent path -- bit-exact against the reference like the default path."""
    monkeypatch.setenv("SB_WIDE", "1")
    scene = random_scene(gpu, 1000 + seed)
    eng, got, want = run_generate_pair(gpu, ref, scene, seed=seed + 7)
    check_against_reference(gpu, scene, got, want)


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("device_exchange", [False, True])
def test_fuzz_sharded_equals_single(gpu, seed, device_exchange):
    """Randomised scenes split over 2 shards (host or device-side count exchange) equal
    the single-engine run bit for bit (scenes with >= 2 instances)."""
    import threading

    from tests.test_gpu_parity import ThreadAllgather, ThreadDevAllgather

    scene = random_scene(gpu, 100 + seed)
    if scene.n_instances < 2:
        scene.n_instances = 256
    whole = gpu.Engine(scene).generate(seed + 3)
    world = 2
    ag, agd = ThreadAllgather(world), ThreadDevAllgather(world)
    bounds = [scene.n_instances * r // world for r in range(world + 1)]
    engines = [gpu.Engine(scene, gpu.Shard(bounds[r], bounds[r + 1], r, world, ag.fn(r),
                                           agd.fn(r) if device_exchange else None))
               for r in range(world)]
    results = [None] * world

    def run(r):
        results[r] = engines[r].generate(seed + 3)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert np.array_equal(np.concatenate([r.accepted for r in results], axis=1), whole.accepted)
    assert np.array_equal(np.concatenate([r.valid for r in results]), whole.valid)
    assert np.array_equal(np.concatenate([r.poses for r in results], axis=1), whole.poses)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("SB_FUZZ_GRID_SEEDS", "6"))))
def test_fuzz_occupancy_grid_path(gpu, ref, seed):
    """Randomised scenes with 33-48 objects: the broad phase goes through the occupancy grid
    (k_place<true>); same bar as above."""
    scene = random_scene(gpu, 5000 + seed, n_range=(33, 49), sizes=(64, 300))
    eng, got, want = run_generate_pair(gpu, ref, scene, seed=seed + 1)
    check_against_reference(gpu, scene, got, want)
