"""GPU parity of ReachMap4D (sb_reach_*) against the reference (oracle/_ref): the built
occupancy bitset (compared as the reference's own SBRM file bytes), per-cell sample
counts, batched queries with and without inclination, placement_filter, and files
exchanged both ways."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from tests import reach_cases as RC

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("chain,samples,res,psi", [("arm", 200000, 0.05, math.pi / 8),
                                                    ("arm", 50000, 0.02, 0.3),
                                                    ("planar", 30000, 0.05, 0.5)])
def test_build_matches_reference(gpu, ref, tmp_path, chain, samples, res, psi):
    ch = getattr(RC, chain)()
    D = gpu.ReachMap4D.build(ch, samples, res, psi, seed=5)
    R = O.RefReachMap.build(ch, samples, res, psi, seed=5, threads=8)
    pd, pr = str(tmp_path / "d.sbrm"), str(tmp_path / "r.sbrm")
    D.save(pd)
    R.save(pr)
    db, rb = open(pd, "rb").read(), open(pr, "rb").read()
    assert len(db) == len(rb) and db[:4] == b"SBRM"
    diff = np.frombuffer(db[88:], np.uint64) ^ np.frombuffer(rb[88:], np.uint64)
    assert db[:88] == rb[:88], "header differs"
    # each FK sample is bit-identical unless glibc misrounds a joint's sin/cos; a bin can
    # only flip if that ulp straddles a cell boundary
    assert int(np.unpackbits(diff.view(np.uint8)).sum()) == 0
    info = D.info()
    assert info["occupied_cells"] == R.info()["occupied_cells"] > 0
    rng = np.random.default_rng(0)
    for _ in range(20):
        c = (int(rng.integers(info["nr"])), int(rng.integers(info["nz"])), int(rng.integers(info["npsi"])))
        assert D.cell_samples(*c) == R.cell_samples(*c)


def test_queries_and_filter(gpu, ref, tmp_path):
    ch = RC.arm()
    R = O.RefReachMap.build(ch, 100000, 0.04, math.pi / 6, seed=9, threads=8)
    p = str(tmp_path / "arm.sbrm")
    R.save(p)
    D = gpu.ReachMap4D.load(p)  # the reference's file, queried on the device
    n = 20000
    B, T = RC.bases(n, 1), RC.targets(n, 1)
    want = R.query_batch(B, T)
    assert 0 < want.sum() < n
    assert np.array_equal(D.query_batch(B, T), want)
    for inc in (0.0, 0.7, math.pi, 4.0, -1.0):
        assert np.array_equal(D.query_batch(B, T, inc), R.query_batch(B, T, inc))
    frames = [np.tile(np.eye(4), (n, 1, 1)) for _ in range(3)]
    for k, f in enumerate(frames):
        f[:, :3, 3] = RC.targets(n, 10 + k, spread=0.9)
    frames[1] = None
    act = np.sort(np.random.default_rng(3).choice(n, 7000, replace=False)).astype(np.uint32)
    want = R.placement_filter(B, frames, act)
    assert 0 < want.sum() < len(act)
    assert np.array_equal(gpu.placement_filter(D, B, frames, act), want)
    assert D.cell_samples(0, 0, 0) == 0  # counts are not in the file
    q = str(tmp_path / "again.sbrm")
    D.save(q)
    assert open(q, "rb").read() == open(p, "rb").read()


def test_reach_errors(gpu, tmp_path):
    with pytest.raises(ValueError):
        gpu.ReachMap4D.build(gpu.KinematicChain(), 10, 0.1, 0.1, 1)
    with pytest.raises(ValueError):
        gpu.ReachMap4D.build(RC.arm(), 10, 0.0, 0.1, 1)
    bad = tmp_path / "bad.sbrm"
    bad.write_bytes(b"XXXX")
    with pytest.raises(RuntimeError):
        gpu.ReachMap4D.load(str(bad))


@pytest.mark.parametrize("seed", [1, 2])
def test_engine_fused_reach_filter(gpu, ref, tmp_path, seed):
    """Fused reachability filter in the placement engine (Appendix C item 8) against the
    reference driver applying placement_filter before collision: accepted indices, valid
    masks and work counters equal."""
    from tests.test_gpu_parity import assert_same
    from paper_2512_16896_b200 import scenes

    n = 2048
    scene = scenes.tabletop_mixed(n, n_objects=9)
    R = O.RefReachMap.build(RC.arm(), 200000, 0.04, math.pi / 6, seed=3, threads=8)
    p = str(tmp_path / "arm.sbrm")
    R.save(p)
    D = gpu.ReachMap4D.load(p)
    base = RC.bases(n, seed)  # arms on a 1.15 m circle round the table: part of it is
    ang = np.random.default_rng(seed).uniform(0, 2 * math.pi, n)  # out of reach
    base[:, 0, 3], base[:, 1, 3], base[:, 2, 3] = 1.15 * np.cos(ang), 1.15 * np.sin(ang), 0.5
    eng = gpu.Engine(scene)
    try:
        for pl in (1, 3, 4, 7):
            eng.set_reach_filter(pl, D, base)
            O.set_reach_filter(pl, R, base)
        got = eng.generate(seed)
        want = O.generate(scene, seed, threads=8)
    finally:
        O.clear_reach_filters()
    assert_same(gpu, got, want)
    assert got.stats["candidates_sampled"] == want["stats"]["candidates_sampled"]
    # the filter bites: many sampled candidates are never collision-checked
    assert got.stats["candidates_sampled"] > 2 * got.stats["candidate_checks"]
    eng.set_reach_filter(1, None)  # cleared: back to plain collision placement for 1


def test_sharded_engine_with_reach_filter(gpu, tmp_path):
    """The fused filter in the sharded kernels (k_fast_round / k_place_instances kReach
    variants): 2 shards with the per-round count exchange equal the single engine."""
    import threading

    from paper_2512_16896_b200 import scenes
    from tests.test_gpu_parity import ThreadAllgather

    n, world = 1500, 2
    scene = scenes.tabletop_mixed(n, n_objects=8)
    R = O.RefReachMap.build(RC.arm(), 100000, 0.04, math.pi / 6, seed=3, threads=8)
    p = str(tmp_path / "arm.sbrm")
    R.save(p)
    D = gpu.ReachMap4D.load(p)
    base = RC.bases(n, 5)
    ang = np.random.default_rng(5).uniform(0, 2 * math.pi, n)
    base[:, 0, 3], base[:, 1, 3], base[:, 2, 3] = 1.15 * np.cos(ang), 1.15 * np.sin(ang), 0.5
    whole_eng = gpu.Engine(scene)
    for pl in (1, 2, 5):
        whole_eng.set_reach_filter(pl, D, base)
    whole = whole_eng.generate(4)
    ag = ThreadAllgather(world)
    bounds = [n * r // world for r in range(world + 1)]
    engines = [gpu.Engine(scene, gpu.Shard(bounds[r], bounds[r + 1], r, world, ag.fn(r)))
               for r in range(world)]
    for r, e in enumerate(engines):
        for pl in (1, 2, 5):
            e.set_reach_filter(pl, D, base[bounds[r]:bounds[r + 1]])
    results = [None] * world

    def run(r):
        results[r] = engines[r].generate(4)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert np.array_equal(np.concatenate([r.accepted for r in results], axis=1), whole.accepted)
    assert np.array_equal(np.concatenate([r.valid for r in results]), whole.valid)
    assert whole.stats["candidates_sampled"] > 2 * whole.stats["candidate_checks"]
