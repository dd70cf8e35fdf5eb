"""CPU: the reference ReachMap4D (oracle/_ref) against SPEC's analytic workspace (1-joint
planar arm -> a ring of radius 1) and its own save / load round trip."""
import numpy as np

from oracle import oracle as O
from tests import reach_cases as RC


def test_planar_arm_ring(ref, tmp_path):
    m = O.RefReachMap.build(RC.planar(), 20000, 0.05, 0.5, seed=3)
    pts = np.array([[np.cos(t), np.sin(t), 0.0] for t in np.linspace(0, 6.2, 40)])
    eye = np.tile(np.eye(4), (len(pts), 1, 1))
    assert m.query_batch(eye, pts).all()
    assert not m.query_batch(eye, pts * 0.5).any()
    p = str(tmp_path / "planar.sbrm")
    m.save(p)
    m2 = O.RefReachMap.load(p)
    assert (m2.query_batch(eye, pts) == 1).all()
    assert m2.info()["occupied_cells"] == m.info()["occupied_cells"]
    assert m2.cell_samples(0, 0, 0) == 0
