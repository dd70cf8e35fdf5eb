"""Device-resident variants of the standalone APIs (sb_sampler_sample_device,
sb_graph_world_poses_device, sb_reach_query_batch_device) equal their host-buffer forms
bit for bit; buffers are torch CUDA tensors passed by pointer on a side stream."""
import math

import numpy as np
import pytest

from tests import graph_cases as G
from tests import reach_cases as RC
from tests import sampler_cases as S

pytestmark = pytest.mark.gpu


def _colmajor(p):
    return np.ascontiguousarray(np.swapaxes(p, -1, -2)).reshape(p.shape[:-2] + (16,))


def test_sampler_device_equals_host(gpu):
    import torch

    n = 4096
    sup = S.supports(n, 2)
    act = np.sort(np.random.default_rng(0).choice(n, 3000, replace=False)).astype(np.uint32)
    for per_instance, region in ((False, [S.RECT]), (True, S.per_instance_regions(n, 1))):
        H, D = gpu.PositionSampler(5), gpu.PositionSampler(5)
        H.prepare(region, n, 9, per_instance)
        D.prepare(region, n, 9, per_instance)
        st = torch.cuda.Stream()
        dsup = torch.tensor(_colmajor(sup), device="cuda")
        dact = torch.tensor(act.astype(np.int32), device="cuda")
        for attempt in range(3):  # several calls: the FIFO cache history must match
            hp, hl = H.sample(sup, act, attempt)
            dpos = torch.empty((len(act), 3), dtype=torch.float64, device="cuda")
            dpl = torch.empty(len(act), dtype=torch.uint8, device="cuda")
            D.sample_device(dsup.data_ptr(), dact.data_ptr(), len(act), attempt, dpos.data_ptr(),
                            dpl.data_ptr(), st.cuda_stream)
            st.synchronize()
            assert np.array_equal(dpos.cpu().numpy(), hp) and np.array_equal(dpl.cpu().numpy(), hl)
        assert H.cache_info() == D.cache_info()


def test_graph_and_reach_device_equal_host(gpu, tmp_path):
    import torch

    n = 2048
    g = gpu.BatchedSceneGraph(n)
    ids, _ = G.build(g, n, 3)
    st = torch.cuda.Stream()
    for nid in ids:
        out = torch.empty((n, 16), dtype=torch.float64, device="cuda")
        g.world_poses_device(nid, out.data_ptr(), st.cuda_stream)
        st.synchronize()
        want = _colmajor(g.world_poses(nid))
        assert np.array_equal(out.cpu().numpy(), want)
    m = gpu.ReachMap4D.build(RC.arm(), 100000, 0.05, math.pi / 6, seed=2)
    B, T = RC.bases(n, 4), RC.targets(n, 4)
    db = torch.tensor(_colmajor(B), device="cuda")
    dt = torch.tensor(T, device="cuda")
    for inc in (None, 0.5):
        out = torch.empty(n, dtype=torch.uint8, device="cuda")
        m.query_batch_device(db.data_ptr(), dt.data_ptr(), n, out.data_ptr(), inc, st.cuda_stream)
        st.synchronize()
        assert np.array_equal(out.cpu().numpy(), m.query_batch(B, T, inc))


def test_orientations_device_equals_host(gpu):
    import torch

    from paper_2512_16896_b200.sampler import FACE_TO, UNIFORM_YAW, sample_orientations_device

    rng = np.random.default_rng(3)
    n = 3000
    act = np.sort(rng.choice(n, 2000, replace=False)).astype(np.uint32)
    pos = rng.uniform(-2, 2, (len(act), 3))
    face = rng.uniform(-2, 2, (n, 2))
    da = torch.tensor(act.astype(np.int32), device="cuda")
    dp, df = torch.tensor(pos, device="cuda"), torch.tensor(face, device="cuda")
    st = torch.cuda.Stream()
    for kind in (UNIFORM_YAW, FACE_TO):
        dy = torch.empty(len(act), dtype=torch.float64, device="cuda")
        sample_orientations_device(kind, da.data_ptr(), len(act), dp.data_ptr(), df.data_ptr(),
                                   77, 5, 2, dy.data_ptr(), st.cuda_stream)
        st.synchronize()
        want = gpu.sample_orientations(kind, act, pos, face, 77, 5, 2)
        assert np.array_equal(dy.cpu().numpy(), want)
