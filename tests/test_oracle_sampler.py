"""CPU: the pure-Python PositionSampler / sample_orientations restatement
(oracle/restate.py) against the reference compiled from /root/reference (oracle/_ref):
FIFO cache history, per-instance regions and orientations, bit-exact."""
import numpy as np

from oracle import restate as R
from tests import sampler_cases as S


def test_fifo_cache_history_matches_reference(ref):
    n, sup = 48, S.supports(48, 3)
    a = S.run_fifo(S.RefAdapter(ref, 5), n, 1, sup)
    b = S.run_fifo(S.RestateAdapter(R, 5), n, 1, sup)
    assert len(a) == len(b)
    for (pa, la, ra), (pb, lb, rb) in zip(a, b):
        assert np.array_equal(pa, pb) and np.array_equal(la, lb) and ra == rb


def test_per_instance_regions_match_reference(ref):
    n, sup = 60, S.supports(60, 4, upright=False)
    regions = S.per_instance_regions(n, 2)
    A, B = S.RefAdapter(ref, 9), S.RestateAdapter(R, 9)
    for ad in (A, B):
        ad.prepare(regions, n, 21, True)
    act = np.arange(n, dtype=np.uint32)
    for attempt in range(3):
        pa, la = A.sample(sup, act, attempt)
        pb, lb = B.sample(sup, act, attempt)
        assert np.array_equal(np.asarray(pa), np.asarray(pb).reshape(-1, 3))
        assert np.array_equal(np.asarray(la), np.asarray(lb, np.uint8))
        act = act[::2]


def test_orientations_match_reference(ref):
    rng = np.random.default_rng(0)
    n = 40
    act = np.sort(rng.choice(n, 25, replace=False)).astype(np.uint32)
    pos = rng.uniform(-1, 1, size=(len(act), 3))
    face = rng.uniform(-1, 1, size=(n, 2))
    face[act[3]] = pos[3, :2]  # coincident target -> yaw 0
    for kind in (0, 1, 2):
        a = ref.sample_orientations(kind, act, pos, face if kind == 2 else None, 17, 4, 2)
        b = R.sample_orientations(kind, [int(x) for x in act], pos, face, 17, 4, 2)
        assert np.array_equal(a, np.asarray(b))
