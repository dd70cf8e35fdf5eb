"""Golden fixtures of the widened components (tests/golden/make_golden_components.py,
generated from the reference): the oracle must reproduce them (CPU, pins the oracle
build) and so must the device path (GPU, no oracle needed at run time)."""
import os

import numpy as np
import pytest

from tests import graph_cases as G
from tests import sampler_cases as S

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _sampler(adapter):
    f = np.load(os.path.join(GOLD, "sampler_fifo_n48.npz"))
    res = S.run_fifo(adapter, 48, 1, S.supports(48, 3))
    assert [len(r[0]) for r in res] == f["sizes"].tolist()
    assert np.array_equal(np.concatenate([r[0] for r in res]), f["positions"])
    assert np.array_equal(np.concatenate([r[1] for r in res]), f["placeable"])
    assert [r[2] for r in res] == f["refills"].tolist()


def _graph(g):
    f = np.load(os.path.join(GOLD, "graph_fk_n16.npz"))
    ids, specs = G.build(g, 16, 0)
    assert ids == f["ids"].tolist()
    for k, nid in enumerate(ids):
        np.testing.assert_allclose(g.world_poses(nid), f["poses"][k], rtol=0, atol=1e-12)


def test_oracle_reproduces_component_fixtures(ref, tmp_path):
    _sampler(S.RefAdapter(ref, 5))
    _graph(ref.RefGraph(16))
    from tests import reach_cases as RC

    m = ref.RefReachMap.build(RC.planar(), 20000, 0.05, 0.5, seed=3)
    p = str(tmp_path / "r.sbrm")
    m.save(p)
    assert open(p, "rb").read() == open(os.path.join(GOLD, "reach_planar.sbrm"), "rb").read()


@pytest.mark.gpu
def test_device_reproduces_component_fixtures(gpu, tmp_path):
    _sampler(S.DeviceAdapter(gpu, 5))
    _graph(gpu.BatchedSceneGraph(16))
    from tests import reach_cases as RC

    m = gpu.ReachMap4D.build(RC.planar(), 20000, 0.05, 0.5, seed=3)
    p = str(tmp_path / "d.sbrm")
    m.save(p)
    assert open(p, "rb").read() == open(os.path.join(GOLD, "reach_planar.sbrm"), "rb").read()
