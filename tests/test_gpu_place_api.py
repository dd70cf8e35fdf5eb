"""GPU: placement-stepped runs (sb_engine_place) -- the reference's per-placement loop
(Appendix C) driven by the caller, one or several placements per call,
with the world readable between calls. Any split equals one sb_engine_generate bit for bit
(accepted indices, valid masks, poses, work counters)."""
import ctypes as C
import threading

import numpy as np
import pytest

from paper_2512_16896_b200 import _capi as A
from paper_2512_16896_b200 import scenes

pytestmark = pytest.mark.gpu

# the reference-defined counters (triangle / node pair tests depend on which warp sees a
# lower hit first and are only bounded by the reference's, not equal to it)
STAT_KEYS = ("valid_instances", "candidate_checks", "narrow_phase_tests", "rounds",
             "per_instance_placements", "candidates_sampled", "accepted_candidates")


def assert_same(a, b):
    assert np.array_equal(a.accepted, b.accepted)
    assert np.array_equal(a.valid, b.valid)
    assert np.array_equal(a.poses, b.poses)
    for k in STAT_KEYS:
        assert a.stats[k] == b.stats[k], k


def stepped(eng, seed, splits):
    P = len(eng.scene.placements)
    bounds = [0] + list(splits) + [P]
    out = None
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        _, out = eng.place(seed, lo, hi - lo)
    return out


@pytest.mark.parametrize("name,factory,n", [
    ("c1", lambda n: scenes.tabletop_boxes(n), 1024),
    ("c2_relations", lambda n: scenes.tabletop_mixed(n), 2048),
    ("c4_grid", lambda n: scenes.dense_clutter(n, n_objects=40), 1024),
    ("c4_wide_round0", lambda n: scenes.dense_clutter(n, n_objects=12), 131072),
])
def test_place_one_by_one_equals_generate(gpu, name, factory, n):
    scene = factory(n)
    eng = gpu.Engine(scene)
    whole = eng.generate(5)
    P = len(scene.placements)
    assert_same(stepped(eng, 5, range(1, P)), whole)
    assert_same(stepped(eng, 5, [P // 3, P // 2]), whole)
    assert_same(eng.generate(5), whole)  # a full run after stepped ones


def test_world_readable_between_placements(gpu):
    """After placement p the engine's world holds p's accepted poses (sb_engine_world)."""
    scene = scenes.tabletop_boxes(256)
    eng = gpu.Engine(scene)
    whole = eng.generate(9)
    P = len(scene.placements)
    first_obj = len(scene.fixed)
    W = eng.world()
    for p in range(P):
        stats, res = eng.place(9, p, 1)
        for inst in (0, 17, 255):
            if whole.accepted[p, inst] >= 0:
                assert np.array_equal(W.object_pose(first_obj + p, inst), whole.poses[p, inst])
        assert stats["accepted_candidates"] == int((whole.accepted[:p + 1] >= 0).sum())
    assert_same(res, whole)


def test_place_protocol_errors(gpu):
    scene = scenes.tabletop_boxes(64)
    eng = gpu.Engine(scene)
    P = len(scene.placements)
    L = A.lib()
    st = A.sb_run_stats()
    assert L.sb_engine_place(eng._h, 3, 1, 1, None, C.byref(st)) == A.SB_ERR_LOGIC  # no open run
    assert L.sb_engine_place(eng._h, 3, 0, 2, None, C.byref(st)) == A.SB_OK
    assert L.sb_engine_place(eng._h, 3, 3, 1, None, C.byref(st)) == A.SB_ERR_LOGIC  # skips 2
    assert L.sb_engine_place(eng._h, 4, 2, 1, None, C.byref(st)) == A.SB_ERR_LOGIC  # other seed
    acc = np.empty((P, 64), np.int16)
    res = A.sb_result(acc.ctypes.data_as(C.POINTER(C.c_int16)), None, None)
    assert L.sb_engine_place(eng._h, 3, 2, 1, C.byref(res), C.byref(st)) == A.SB_ERR_INVALID_ARGUMENT
    assert L.sb_engine_place(eng._h, 3, 2, P, None, C.byref(st)) == A.SB_ERR_INVALID_ARGUMENT
    assert L.sb_engine_place(eng._h, 3, 2, P - 2, C.byref(res), C.byref(st)) == A.SB_OK
    assert np.array_equal(acc, eng.generate(3).accepted)


def test_place_sharded_equals_single(gpu):
    """Two shards stepped placement by placement (device-side count exchange) equal the
    single-engine run."""
    from tests.test_gpu_parity import ThreadAllgather, ThreadDevAllgather

    scene = scenes.tabletop_mixed(1024)
    whole = gpu.Engine(scene).generate(2)
    world = 2
    ag, agd = ThreadAllgather(world), ThreadDevAllgather(world)
    b = [scene.n_instances * r // world for r in range(world + 1)]
    engines = [gpu.Engine(scene, gpu.Shard(b[r], b[r + 1], r, world, ag.fn(r), agd.fn(r)))
               for r in range(world)]
    P = len(scene.placements)
    results = [None] * world

    def run(r):
        for p in range(P):
            _, results[r] = engines[r].place(2, p, 1)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert np.array_equal(np.concatenate([r.accepted for r in results], axis=1), whole.accepted)
    assert np.array_equal(np.concatenate([r.valid for r in results]), whole.valid)
    assert np.array_equal(np.concatenate([r.poses for r in results], axis=1), whole.poses)
