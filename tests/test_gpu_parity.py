"""GPU parity: the CUDA path (through the C ABI) against the reference oracle.

Bar (BASELINE.json north_star): accepted candidate indices and collision-free masks
bit-exact; accepted poses within 1e-5 relative (tolerance written in assert_poses)."""
import math
import threading

import numpy as np
import pytest

from paper_2512_16896_b200 import _capi as A
from paper_2512_16896_b200 import scenes

pytestmark = pytest.mark.gpu

POSE_RTOL = 1e-5   # north_star: accepted poses within 1e-5 relative
POSE_ATOL = 1e-12  # entries that are exactly 0 in one build and ~1e-17 in the other


def rot_from_quat(q):
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                     [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                     [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])


def random_pose(rng, spread, upright, z=None):
    m = np.eye(4)
    if upright:
        a = rng.uniform(0, 2 * math.pi)
        c, s = math.cos(a), math.sin(a)
        m[:2, :2] = [[c, -s], [s, c]]
    else:
        m[:3, :3] = rot_from_quat(rng.normal(size=4))
    m[:3, 3] = rng.uniform(-spread, spread, size=3)
    if z is not None:
        m[2, 3] = z
    return m


def assert_poses(got, ref_colmajor, pkg, accepted=None):
    """north_star's bar (1e-5 relative) everywhere; with `accepted`, every accepted pose
    must also be bit-identical (the device libm is glibc's own, sb_glibcm.cuh)."""
    ref = pkg.from_colmajor(ref_colmajor)
    assert got.shape == ref.shape
    bad = ~np.isclose(got, ref, rtol=POSE_RTOL, atol=POSE_ATOL)
    assert not bad.any(), f"{bad.sum()} pose entries outside tolerance"
    if accepted is not None:
        same = (got == ref).all(axis=(-2, -1))
        placed = accepted >= 0
        assert same[placed].all(), f"{np.sum(~same[placed])} accepted poses not bit-identical"


def world_pair(pkg, ref, n, meshes, margin=0.0):
    W = pkg.CollisionWorld(n, margin)
    R = ref.RefWorld(n, margin)
    gids = []
    for m in meshes:
        g1 = W.register_geometry(m)
        g2 = R.register_geometry(m.vertices, m.triangles)
        assert g1 == g2
        gids.append(g1)
    return W, R, gids


def mesh_zoo(pkg):
    rng = scenes.Pcg32(99)
    return [pkg.make_box(0.1, 0.08, 0.12), pkg.make_box(0.3, 0.2, 0.05),
            pkg.make_cylinder(0.05, 0.1, 16), pkg.make_sphere(0.06, 8, 10),
            scenes.sphere_set(rng), scenes.open_container(0.3, 0.25, 0.15, 0.01)]


@pytest.mark.parametrize("upright,seed,margin", [(True, 0, 0.0), (True, 1, 0.0), (True, 2, 0.0),
                                                 (False, 0, 0.0), (False, 1, 0.0), (False, 2, 0.0),
                                                 # margin > 0: tri_tri_distance path (collision.cpp:136-212)
                                                 (True, 3, 0.004), (False, 4, 0.004),
                                                 (True, 5, 0.02), (False, 6, 0.02)])
def test_check_batch_random_worlds(gpu, ref, upright, seed, margin):
    pkg = gpu
    rng = np.random.default_rng(seed)
    n = 512
    meshes = mesh_zoo(pkg)
    W, R, gids = world_pair(pkg, ref, n, meshes, margin)
    n_obj = 8
    for k in range(n_obj):
        g = gids[rng.integers(len(gids))]
        o1, o2 = W.add_object(f"o{k}", g), R.add_object(g)
        assert o1 == o2
        poses = np.stack([random_pose(rng, 0.12, upright) for _ in range(n)])
        W.update_transforms(o1, poses)
        R.update_transforms(o2, pkg.colmajor(poses))
        en = np.nonzero(rng.random(n) < 0.7)[0].astype(np.uint32)
        W.set_enabled(o1, en, True)
        R.set_enabled(o2, en, True)
    for trial in range(3):
        act = np.sort(rng.choice(n, size=n // 2 + trial * 50, replace=False)).astype(np.uint32)
        cand = np.stack([random_pose(rng, 0.12, upright) for _ in act])
        g = gids[rng.integers(len(gids))]
        f1, c1 = W.check_batch(g, cand, act)
        f2, c2 = R.check_batch(g, pkg.colmajor(cand), act)
        assert np.array_equal(f1, f2), f"free mask differs at {np.nonzero(f1 != f2)[0][:10]}"
        assert np.array_equal(c1, c2), "contact_object differs"
        assert 0 < (f1[act] == 0).sum() < len(act)  # both outcomes exercised
    s1, s2 = W.stats(), R.stats()
    assert s1["checked_instances"] == s2["checked_instances"]
    assert s1["narrow_phase_tests"] == s2["narrow_phase_tests"]
    assert s1["triangle_pair_tests"] <= s2["triangle_pair_tests"]


def test_check_batch_resting_coplanar(gpu, ref):
    """Objects resting on one plane share bottom faces: the coplanar branch
    (collision.cpp:63-83) decides; SURVEY Appendix A scenario included."""
    pkg = gpu
    n = 256
    big, small = pkg.make_box(0.4, 0.4, 0.4), pkg.make_box(0.1, 0.1, 0.1)
    W, R, (gb, gs) = world_pair(pkg, ref, n, [big, small])
    o = W.add_object("big", gb)
    R.add_object(gb)
    poses = np.stack([pkg.translation(0, 0, 0.201)] * n)
    W.update_transforms(o, poses)
    R.update_transforms(o, pkg.colmajor(poses))
    W.set_enabled_all(o, True)
    R.set_enabled_all(o, True)
    rng = np.random.default_rng(5)
    cand = []
    for i in range(n):
        c = random_pose(rng, 0.35, True, z=0.051)
        cand.append(c)
    # Appendix A fixed cases in the first slots
    cases = [(0, 0, 0.051, 0.3), (0, 0, 0.201, 0.3), (0.2, 0, 0.051, 0.0), (0.5, 0, 0.051, 0.0)]
    for i, (x, y, z, yaw) in enumerate(cases):
        m = np.eye(4)
        m[:2, :2] = [[math.cos(yaw), -math.sin(yaw)], [math.sin(yaw), math.cos(yaw)]]
        m[:3, 3] = (x, y, z)
        cand[i] = m
    cand = np.stack(cand)
    act = np.arange(n, dtype=np.uint32)
    f1, c1 = W.check_batch(gs, cand, act)
    f2, c2 = R.check_batch(gs, pkg.colmajor(cand), act)
    assert np.array_equal(f1, f2) and np.array_equal(c1, c2)
    assert list(f1[:4]) == [0, 1, 1, 1]  # collide, contained-free, straddle-free, free


def test_world_api_semantics(gpu):
    pkg = gpu
    W = pkg.CollisionWorld(4)
    g = W.register_geometry(pkg.make_box(1, 1, 1))
    assert W.register_geometry(pkg.make_box(1, 1, 1)) == g  # fingerprint dedupe
    o = W.add_object("cube", g)
    assert not W.enabled(o, 0)
    assert np.array_equal(W.object_pose(o, 3), np.eye(4))
    cand = np.stack([pkg.translation(0.5, 0, 0)] * 4)
    act = np.arange(4, dtype=np.uint32)
    free, contact = W.check_batch(g, cand, act)
    assert free.all()  # disabled objects never collide
    W.set_enabled(o, [0, 2], True)
    free, contact = W.check_batch(g, cand, act)
    assert list(free) == [0, 1, 0, 1] and list(contact) == [0, -1, 0, -1]
    W.update_transform(o, 2, pkg.translation(2, 0, 0))
    free, _ = W.check_batch(g, cand, act)
    assert list(free) == [0, 1, 1, 1]
    free, contact = W.check_batch(g, cand[:1], [1])
    assert free.all() and (contact == -1).all()  # inactive / free untouched
    with pytest.raises(IndexError):
        W.set_enabled(o, [9], True)
    with pytest.raises(IndexError):
        W.add_object("x", 42)
    bad = np.eye(4)
    bad[3, 3] = 2.0
    with pytest.raises(ValueError):
        W.update_transform(o, 0, bad)
    assert W.stats()["check_calls"] == 4


def run_generate_pair(pkg, ref, scene, seed=1):
    eng = pkg.Engine(scene)
    got = eng.generate(seed)
    want = ref.generate(scene, seed, threads=8)
    return eng, got, want


def assert_same(pkg, got, want):
    assert np.array_equal(got.valid, want["valid"]), "valid mask differs"
    diff = np.argwhere(got.accepted != want["accepted"])
    assert len(diff) == 0, f"accepted differs at (placement, inst) {diff[:10].tolist()}"
    assert_poses(got.poses, want["poses"], pkg, got.accepted)
    for k in ("valid_instances", "candidate_checks", "narrow_phase_tests", "rounds",
              "per_instance_placements"):
        assert got.stats[k] == want["stats"][k], k


@pytest.mark.parametrize("name,factory", [
    ("c1_tabletop_1024", lambda: scenes.tabletop_boxes(1024)),
    ("c2_mixed_2048", lambda: scenes.tabletop_mixed(2048)),
    ("c3_kitchen_1024", lambda: scenes.kitchen(1024, attempts=128)),
    ("c4_clutter_512", lambda: scenes.dense_clutter(512, n_objects=60)),
    ("c5_sweep_4096x50", lambda: scenes.scale_sweep(4096, 50)),
])
def test_generate_matches_reference(gpu, ref, name, factory):
    scene = factory()
    eng, got, want = run_generate_pair(gpu, ref, scene)
    assert_same(gpu, got, want)
    assert got.stats["valid_instances"] > 0


def test_generate_is_deterministic_and_warm(gpu, ref):
    scene = scenes.tabletop_mixed(1024, n_objects=12)
    eng = gpu.Engine(scene)
    a = eng.generate(5)
    b = eng.generate(5)  # warm: same engine, same seed -> identical output
    assert np.array_equal(a.accepted, b.accepted) and np.array_equal(a.poses, b.poses)
    c = eng.generate(6)
    assert not np.array_equal(a.accepted, c.accepted)
    assert_same(gpu, c, ref.generate(scene, 6, threads=8))


def _variant_scene(pkg, local_vector):
    base = scenes.tabletop_boxes(1024, n_objects=8, table=(1.6, 1.2))
    rels = {
        2: pkg.Relation(anchor=1, distance_type=A.SB_DIST_GREATER, direction=A.SB_DIR_FRONT,
                        distance=0.2, angle_threshold=math.pi / 3),
        5: pkg.Relation(anchor=4, distance_type=A.SB_DIST_LESS, distance=0.35),
        6: pkg.Relation(anchor=2, direction=A.SB_DIR_RIGHT),
    }
    if local_vector:
        rels[3] = pkg.Relation(anchor=0, distance_type=A.SB_DIST_EQUAL, direction=A.SB_DIR_VECTOR,
                               direction_vector=(0.3, -0.4), distance=0.3,
                               frame=A.SB_FRAME_LOCAL)
    for k, r in rels.items():
        base.placements[k].relation = r
    base.placements[4].orientation = A.SB_ORIENT_FACE_TO
    base.placements[4].face_target = 0
    base.placements[7].orientation = A.SB_ORIENT_FIXED
    return base


def test_generate_relations_variants(gpu, ref):
    """greater / less / none distance bands, axis directions, face_to, fixed yaw."""
    eng, got, want = run_generate_pair(gpu, ref, _variant_scene(gpu, False), seed=3)
    assert_same(gpu, got, want)


def test_generate_relations_local_vector(gpu, ref):
    """Local-frame vector direction: the arc count ceil(2*theta/step) sits on an integer
    boundary, so it depends on the last bit of atan2 / sin / cos -- passes because the
    device libm is correctly rounded like glibc (sb_crmath.cuh)."""
    eng, got, want = run_generate_pair(gpu, ref, _variant_scene(gpu, True), seed=3)
    assert_same(gpu, got, want)


def test_generate_canonical_relation_fast_path(gpu, ref):
    """N=1: anchors cannot vary, so the relation region is canonical and the FIFO
    fast path samples from it (relationships.cpp:188-190)."""
    scene = scenes.tabletop_mixed(1, n_objects=9)
    eng, got, want = run_generate_pair(gpu, ref, scene, seed=2)
    assert got.stats["per_instance_placements"] == 0
    assert_same(gpu, got, want)


def test_generate_impossible_placement(gpu, ref):
    """A relation whose region misses its support is empty in every instance
    (placeable = 0, Appendix C.6): all instances end invalid after K attempts."""
    pkg = gpu
    scene = scenes.tabletop_boxes(256, n_objects=3, attempts=5)
    far = pkg.Support(pkg.translation(5.0, 0.0, 0.75), (-0.3, -0.3, 0.3, 0.3))
    scene.supports.append(far)
    scene.placements[2].support = 1
    scene.placements[2].relation = pkg.Relation(anchor=0, distance_type=A.SB_DIST_LESS,
                                                distance=0.1)
    eng, got, want = run_generate_pair(pkg, ref, scene)
    assert got.valid.sum() == 0 and (got.accepted[2] == -1).all()
    assert_same(pkg, got, want)


class ThreadAllgather:
    """In-process allgather among `world` engine threads (one GPU, several shards)."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world

    def fn(self, rank):
        def allgather(vals):
            self.slots[rank] = list(vals)
            self.barrier.wait()
            out = [v for r in range(self.world) for v in self.slots[r]]
            self.barrier.wait()
            return out
        return allgather


class ThreadDevAllgather:
    """In-process stand-in for NCCL all_gather on the engines' streams (shards on one GPU):
    each rank records an event behind its send word, every rank's stream waits for all the
    events and copies the words into its receive buffer (device to device)."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world

    def fn(self, rank):
        import torch

        from paper_2512_16896_b200.dist import _DevArray

        def allgather_dev(send, n, recv, stream):
            ext = torch.cuda.ExternalStream(stream)
            ev = torch.cuda.Event()
            ev.record(ext)
            self.slots[rank] = (send, ev)
            self.barrier.wait()
            dst = torch.as_tensor(_DevArray(recv, self.world * n), device="cuda")
            with torch.cuda.stream(ext):
                for r, (sp, evr) in enumerate(self.slots):
                    ext.wait_event(evr)
                    dst[r * n:(r + 1) * n].copy_(torch.as_tensor(_DevArray(sp, n), device="cuda"))
            self.barrier.wait()
        return allgather_dev


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_device_exchange_equals_single(gpu, ref, world):
    """FIFO placements with the device-side count exchange (sb_shard.allgather_dev: rounds
    chained on the device, host checks every few rounds) equal the single-shard run."""
    pkg = gpu
    scene = scenes.tabletop_mixed(1500, n_objects=10)
    whole = pkg.Engine(scene).generate(4)
    ag, agd = ThreadAllgather(world), ThreadDevAllgather(world)
    bounds = [scene.n_instances * r // world for r in range(world + 1)]
    engines = [pkg.Engine(scene, pkg.Shard(bounds[r], bounds[r + 1], r, world, ag.fn(r),
                                           agd.fn(r))) for r in range(world)]
    results = [None] * world

    def run(r):
        results[r] = engines[r].generate(4)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert all(r is not None for r in results)
    assert np.array_equal(np.concatenate([r.accepted for r in results], axis=1), whole.accepted)
    assert np.array_equal(np.concatenate([r.valid for r in results]), whole.valid)
    assert np.array_equal(np.concatenate([r.poses for r in results], axis=1), whole.poses)
    assert sum(r.stats["rounds"] for r in results) >= whole.stats["rounds"]


def _run_shards(pkg, scene, world, seed, device_exchange=True):
    ag, agd = ThreadAllgather(world), ThreadDevAllgather(world)
    bounds = [scene.n_instances * r // world for r in range(world + 1)]
    engines = [pkg.Engine(scene, pkg.Shard(bounds[r], bounds[r + 1], r, world, ag.fn(r),
                                           agd.fn(r) if device_exchange else None))
               for r in range(world)]
    results = [None] * world

    def run(r):
        results[r] = engines[r].generate(seed)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert all(r is not None for r in results)
    return results


@pytest.mark.parametrize("name,world,factory,force", [
    ("mixed_relations_forced", 2, lambda: scenes.tabletop_mixed(1500, n_objects=10), True),
    ("mixed_relations_forced", 3, lambda: scenes.tabletop_mixed(1500, n_objects=10), True),
    ("clutter40_full_size", 2, lambda: scenes.dense_clutter(262144, n_objects=40), False),
])
def test_sharded_wide_round0_equals_single(gpu, monkeypatch, name, world, factory, force):
    """Sharded runs with the device exchange take round 0 grid-wide too (k_wide_* with the
    draw base from the gathered round-0 counts, survivors left in their tiles for the
    per-round kernels): bit-identical to the single-GPU run. `force`: SB_WIDE=1 below the
    131,072-instance threshold (relation placements keep the per-round path)."""
    pkg = gpu
    scene = factory()
    whole = pkg.Engine(scene).generate(6)
    if force:
        monkeypatch.setenv("SB_WIDE", "1")
    results = _run_shards(pkg, scene, world, 6)
    assert np.array_equal(np.concatenate([r.accepted for r in results], axis=1), whole.accepted)
    assert np.array_equal(np.concatenate([r.valid for r in results]), whole.valid)
    assert np.array_equal(np.concatenate([r.poses for r in results], axis=1), whole.poses)
    assert sum(r.stats["candidate_checks"] for r in results) == whole.stats["candidate_checks"]


def _run_bounds(pkg, scene, bounds, seed, device_exchange=True):
    world = len(bounds) - 1
    ag, agd = ThreadAllgather(world), ThreadDevAllgather(world)
    engines = [pkg.Engine(scene, pkg.Shard(bounds[r], bounds[r + 1], r, world, ag.fn(r),
                                           agd.fn(r) if device_exchange else None))
               for r in range(world)]
    results = [None] * world

    def run(r):
        results[r] = engines[r].generate(seed)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert all(r is not None for r in results)
    return results


@pytest.mark.parametrize("attempts", [8, 9])
@pytest.mark.parametrize("wide", [False, True])
def test_sharded_early_finisher_and_exhausted_shard(gpu, monkeypatch, attempts, wide):
    """a tiny shard runs out of survivors at some round r0 while the
    other exhausts all K attempts; with both parities of K - r0 (K = 8, 9) the idle shard's
    tile counts must not let the final invalidation clear instances it already placed."""
    pkg = gpu
    scene = scenes.tabletop_boxes(700, n_objects=40, attempts=attempts)  # ~half end invalid
    whole = pkg.Engine(scene).generate(3)
    assert (whole.valid == 0).any(), "the scene must exhaust K for some instances"
    if wide:
        monkeypatch.setenv("SB_WIDE", "1")
        single = pkg.Engine(scene).generate(3)  # single-GPU wide round 0 + persistent rounds
        assert np.array_equal(single.valid, whole.valid)
        assert np.array_equal(single.accepted, whole.accepted)
    for bounds in ([0, 3, 700], [0, 697, 700], [0, 1, 2, 700]):
        results = _run_bounds(pkg, scene, bounds, 3)
        assert np.array_equal(np.concatenate([r.valid for r in results]), whole.valid), bounds
        assert np.array_equal(np.concatenate([r.accepted for r in results], axis=1), whole.accepted), bounds


@pytest.mark.parametrize("attempts", [3, 4, 64])
def test_dense_wide_rounds_match_reference(gpu, ref, monkeypatch, attempts):
    """Dense placements run later rounds grid-wide too once a run has seen many survivors
    (SB_WIDE_MORE: the survivor count that earns another wide round; 1 here, so every
    placement with a survivor goes up to 4 wide rounds on the repeated runs, including
    K = 3 / 4 where the wide rounds reach the last attempt). Every run equals the reference."""
    monkeypatch.setenv("SB_WIDE", "1")
    monkeypatch.setenv("SB_WIDE_MORE", "1")
    scene = scenes.tabletop_boxes(1500, n_objects=40, attempts=attempts)
    want = ref.generate(scene, 5, threads=8)
    eng = gpu.Engine(scene)
    for _ in range(4):  # run 1 records survivors, later runs use 2, 3, 4 wide rounds
        got = eng.generate(5)
        assert_same(gpu, got, want)


@pytest.mark.parametrize("lookback", ["0", "1"])
@pytest.mark.parametrize("attempts", [2, 64])
def test_fast_rounds_lookback_and_barrier_match_reference(gpu, ref, monkeypatch, lookback, attempts):
    """The persistent fast rounds with the decoupled look-back on the tile counts (default)
    and with a grid barrier per round (SB_LOOKBACK=0) both equal the reference, with and
    without the grid-wide round 0, including K = 2 where the survivors exhaust K."""
    monkeypatch.setenv("SB_LOOKBACK", lookback)
    scene = scenes.tabletop_boxes(3000, n_objects=30, attempts=attempts)
    want = ref.generate(scene, 11, threads=8)
    for wide in ("0", "1"):
        monkeypatch.setenv("SB_WIDE", wide)
        got = gpu.Engine(scene).generate(11)
        assert_same(gpu, got, want)


def test_per_instance_tile_order_from_history(gpu, ref):
    """Per-instance placements claim their tiles slowest-first from the previous run's tile
    times (several tiles per CTA: 30,000 instances here). Repeated runs -- the second and
    third with the learned order -- equal the reference."""
    scene = scenes.tabletop_mixed(30000)
    want = ref.generate(scene, 3, threads=8)
    eng = gpu.Engine(scene)
    for _ in range(3):
        got = eng.generate(3)
        assert_same(gpu, got, want)
        assert got.stats["per_instance_placements"] > 0


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_generate_equals_single(gpu, ref, world):
    """Variation-batch sharding: G shards with the per-round count exchange
    reproduce the single-shard run bit for bit (fast path and per-instance path)."""
    pkg = gpu
    scene = scenes.tabletop_mixed(1500, n_objects=10)
    whole = pkg.Engine(scene).generate(4)
    ag = ThreadAllgather(world)
    bounds = [scene.n_instances * r // world for r in range(world + 1)]
    engines = [pkg.Engine(scene, pkg.Shard(bounds[r], bounds[r + 1], r, world, ag.fn(r)))
               for r in range(world)]
    results = [None] * world

    def run(r):
        results[r] = engines[r].generate(4)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    acc = np.concatenate([r.accepted for r in results], axis=1)
    valid = np.concatenate([r.valid for r in results])
    poses = np.concatenate([r.poses for r in results], axis=1)
    assert np.array_equal(acc, whole.accepted)
    assert np.array_equal(valid, whole.valid)
    assert np.array_equal(poses, whole.poses)


def _hole_scene(pkg, n):
    """Full annuli with a hole (direction none, theta = pi, min_r > 0): 'greater' keeps
    a hole that may clip against the table edge, 'equal' a band ring; the region is
    triangulated through bridge_hole (polygon.cpp:197-258)."""
    base = scenes.tabletop_boxes(n, n_objects=7, table=(1.6, 1.2))
    base.placements[2].relation = pkg.Relation(anchor=0, distance_type=A.SB_DIST_GREATER,
                                               distance=0.25)
    base.placements[4].relation = pkg.Relation(anchor=1, distance_type=A.SB_DIST_EQUAL,
                                               distance=0.3)
    base.placements[6].relation = pkg.Relation(anchor=3, distance_type=A.SB_DIST_GREATER,
                                               distance=0.5)
    return base


def test_generate_wide_annular_sectors(gpu, ref):
    """Annular sectors wide enough (2 * 70+ arc points) to outgrow the group path's ring
    take the serial big-ring region path (sbp::big_region_table)."""
    pkg = gpu
    base = scenes.tabletop_boxes(768, n_objects=6, table=(1.6, 1.2))
    base.placements[2].relation = pkg.Relation(anchor=0, distance_type=A.SB_DIST_GREATER,
                                               direction=A.SB_DIR_LEFT, distance=0.2,
                                               angle_threshold=2.9)
    base.placements[4].relation = pkg.Relation(anchor=1, distance_type=A.SB_DIST_EQUAL,
                                               direction=A.SB_DIR_VECTOR,
                                               direction_vector=(0.6, 0.8), distance=0.3,
                                               angle_threshold=2.5, frame=A.SB_FRAME_LOCAL)
    eng, got, want = run_generate_pair(pkg, ref, base, seed=4)
    assert_same(pkg, got, want)


@pytest.mark.parametrize("n,seed", [(1024, 3), (1, 2)])
def test_generate_annulus_with_hole(gpu, ref, n, seed):
    eng, got, want = run_generate_pair(gpu, ref, _hole_scene(gpu, n), seed=seed)
    assert_same(gpu, got, want)
    if n > 1:
        assert got.stats["per_instance_placements"] == 3


@pytest.mark.parametrize("name,factory", [
    ("c2_full_16384x25", lambda: scenes.tabletop_mixed(16384)),
    ("c3_full_65536x50_k256", lambda: scenes.kitchen(65536)),
    ("c4_full_262144x100_sphere_sets", lambda: scenes.dense_clutter(262144)),
    ("c5_1M_x10", lambda: scenes.scale_sweep(1 << 20, 10)),
])
def test_generate_matches_reference_at_scale(gpu, ref, name, factory):
    """BASELINE sizes (C2, C3, C4 in full, C5's 2^20 x 10 point): the device
    engine against the reference on the box's host cores -- accepted indices and valid
    masks bit-exact, poses within 1e-5, work counters equal."""
    import os

    scene = factory()
    eng = gpu.Engine(scene)
    got = eng.generate(1)
    want = ref.generate(scene, 1, threads=os.cpu_count() or 8)
    assert_same(gpu, got, want)


@pytest.mark.parametrize("spec", [8, 64])
def test_fifo_speculative_solo_tail(gpu, ref, spec, monkeypatch):
    """SB_SOLO_SPEC > 0: the FIFO solo tail evaluates several rounds at once (draw of round
    a + s, rank e = draws + s * nt + e) and keeps only the rounds up to the first accept;
    results must equal the sequential reference (off by default: not faster on C2)."""
    monkeypatch.setenv("SB_SOLO_SPEC", str(spec))
    monkeypatch.setenv("SB_SOLO", "32")
    for scene in (scenes.tabletop_mixed(2048), scenes.kitchen(1024, attempts=128)):
        eng, got, want = run_generate_pair(gpu, ref, scene, seed=7)
        assert_same(gpu, got, want)


def test_generate_ratio_on_support(gpu, ref):
    """apply_ratio_on_support (relationships.cpp:220-230) on rect supports: the region is
    eroded by ratio * min(footprint) / 2 (Boost buffer stand-in, oracle/shim); a support
    too small for the erosion leaves the placement impossible."""
    pkg = gpu
    scene = scenes.tabletop_boxes(1024, n_objects=6)
    scene.placements[1].ratio_on_support = 1.0
    scene.placements[3].ratio_on_support = 0.5
    eng, got, want = run_generate_pair(pkg, ref, scene, seed=5)
    assert_same(pkg, got, want)
    assert got.valid.sum() > 0
    small = pkg.Support(pkg.translation(0.0, 0.0, 0.75), (-0.03, -0.03, 0.03, 0.03))
    scene.supports.append(small)
    scene.placements[5].support = len(scene.supports) - 1
    scene.placements[5].ratio_on_support = 1.0  # boxes >= 0.08 wide: eroded away
    eng, got, want = run_generate_pair(pkg, ref, scene, seed=5)
    assert_same(pkg, got, want)
    assert (got.accepted[5] == -1).all() and got.valid.sum() == 0


def test_generate_ratio_on_support_relations(gpu, ref):
    """Erosion of (convex) relation regions on the device: a disc clipped to the table and
    90-degree sectors, eroded per instance by the region kernel."""
    pkg = gpu
    scene = scenes.tabletop_boxes(1024, n_objects=8, table=(1.6, 1.2))
    scene.placements[2].relation = pkg.Relation(anchor=1, distance_type=A.SB_DIST_LESS,
                                                distance=0.35)
    scene.placements[4].relation = pkg.Relation(anchor=3, direction=A.SB_DIR_RIGHT)
    scene.placements[6].relation = pkg.Relation(anchor=5, distance_type=A.SB_DIST_LESS,
                                                direction=A.SB_DIR_FRONT, distance=0.4)
    for k, ratio in ((2, 0.6), (4, 1.0), (6, 0.4), (7, 0.8)):
        scene.placements[k].ratio_on_support = ratio
    eng, got, want = run_generate_pair(pkg, ref, scene, seed=2)
    assert_same(pkg, got, want)
    assert got.stats["per_instance_placements"] >= 3


def test_ratio_on_support_validation(gpu, ref):
    pkg = gpu
    scene = scenes.tabletop_boxes(16, n_objects=3)
    scene.placements[1].ratio_on_support = 1.5
    with pytest.raises(ValueError):
        pkg.Engine(scene)
    # an annulus whose hole survives the clip is not hole-free: the reference's erosion
    # (the Boost stand-in's buffer) throws, and the engine's region build fails with it
    scene.placements[1].ratio_on_support = 0.5
    scene.placements[1].relation = pkg.Relation(anchor=0, distance_type=A.SB_DIST_GREATER,
                                                distance=0.3)
    with pytest.raises(Exception):
        ref.generate(scene, 1)
    with pytest.raises(RuntimeError):
        pkg.Engine(scene).generate(1)


def test_graph_replay_equals_direct(gpu, ref, monkeypatch):
    """SB_GRAPH=1: the run captured once into a CUDA graph and replayed (seed read on the
    device) gives the same results as direct launches, for several seeds."""
    monkeypatch.setenv("SB_GRAPH", "1")
    scene = scenes.tabletop_mixed(1024, n_objects=9)
    eng = gpu.Engine(scene)
    for seed in (1, 2, 1):
        got = eng.generate(seed)
        assert_same(gpu, got, ref.generate(scene, seed, threads=8))
