"""GPU parity of the standalone PositionSampler / sample_orientations (sb_sampler_*,
sb_sample_orientations) against the reference compiled from /root/reference
(oracle/_ref). Positions and placeable masks are bit-exact: the device replays the
reference's FIFO cache as draw indices with PCG jump-ahead and computes every point with
the reference's operation order (-fmad=false)."""
import numpy as np
import pytest

from paper_2512_16896_b200 import _capi as A
from tests import sampler_cases as S

pytestmark = pytest.mark.gpu

YAW_ULPS = 1  # face_to: device atan2 is correctly rounded, glibc's is within 1 ulp


@pytest.mark.parametrize("n,seed,upright", [(64, 0, True), (1000, 1, False), (4096, 2, True)])
def test_fifo_cache_history(gpu, ref, n, seed, upright):
    sup = S.supports(n, seed + 10, upright)
    a = S.run_fifo(S.RefAdapter(ref, 3 + seed), n, seed, sup)
    b = S.run_fifo(S.DeviceAdapter(gpu, 3 + seed), n, seed, sup)
    assert len(a) == len(b)
    for k, ((pa, la, ra), (pb, lb, rb)) in enumerate(zip(a, b)):
        assert np.array_equal(la, lb), f"op {k}: placeable"
        assert np.array_equal(pa, pb), f"op {k}: {np.sum(pa != pb)} position entries differ"
        assert ra == rb, f"op {k}: refill count {rb} vs {ra}"


@pytest.mark.parametrize("n,seed", [(97, 0), (3000, 1)])
def test_per_instance_regions(gpu, ref, n, seed):
    sup = S.supports(n, seed, upright=seed % 2 == 0)
    regions = S.per_instance_regions(n, seed + 5)
    A_, B = S.RefAdapter(ref, 12), S.DeviceAdapter(gpu, 12)
    for ad in (A_, B):
        ad.prepare(regions, n, 99 + seed, True)
    rng = np.random.default_rng(seed)
    act = np.arange(n, dtype=np.uint32)
    for attempt in range(4):
        pa, la = A_.sample(sup, act, attempt)
        pb, lb = B.sample(sup, act, attempt)
        assert np.array_equal(la, lb)
        assert np.array_equal(pa, pb)
        act = np.sort(rng.choice(act, size=len(act) // 2, replace=False)).astype(np.uint32)
    assert B.refills() == 0  # per-instance regions never touch the cache


def test_orientations(gpu, ref):
    rng = np.random.default_rng(1)
    n = 5000
    act = np.sort(rng.choice(n, 3000, replace=False)).astype(np.uint32)
    pos = rng.uniform(-3, 3, size=(len(act), 3))
    face = rng.uniform(-3, 3, size=(n, 2))
    face[act[::97]] = pos[::97, :2]  # coincident targets -> yaw 0
    face[act[5]] = pos[5, :2] + [0.0, 1e-13]  # below face_to_yaw's 1e-12 threshold
    for kind in (gpu.sampler.FIXED, gpu.sampler.UNIFORM_YAW, gpu.sampler.FACE_TO):
        f = face if kind == gpu.sampler.FACE_TO else None
        want = ref.sample_orientations(kind, act, pos, f, 1234, 77, 3)
        got = gpu.sample_orientations(kind, act, pos, f, 1234, 77, 3)
        if kind == gpu.sampler.FACE_TO:
            ulp = np.spacing(np.abs(want))
            assert np.all(np.abs(got - want) <= YAW_ULPS * ulp)
            assert np.mean(got == want) > 0.99
        else:
            assert np.array_equal(got, want)


def test_sampler_errors(gpu):
    s = gpu.PositionSampler(1)
    sup = S.supports(4, 0)
    with pytest.raises(A.SbError):  # logic_error: prepare() not called
        s.sample(sup, [0], 0)
    s.prepare([S.SLIVER], 4, 1)
    with pytest.raises(ValueError):  # zero-area canonical region
        s.sample(sup, [0, 1], 0)
    s.prepare([S.RECT], 4, 1)
    with pytest.raises(IndexError):
        s.sample(sup, [0, 4], 0)
    pos, pl = s.sample(sup, [], 0)
    assert pos.shape == (0, 3) and len(pl) == 0
    with pytest.raises(ValueError):
        gpu.sample_orientations(gpu.sampler.FACE_TO, [0], np.zeros((1, 3)), None, 1, 1, 0)
    with pytest.raises(IndexError):
        gpu.sample_orientations(gpu.sampler.FACE_TO, [3], np.zeros((1, 3)), np.zeros((2, 2)), 1, 1, 0)
