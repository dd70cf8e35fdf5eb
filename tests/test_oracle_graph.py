"""CPU: the reference BatchedSceneGraph (oracle/_ref) against SPEC's scene_graph
properties -- identity edges, lower-limit joint init, batched FK equal to the sequential
per-instance composition within 1e-9, tree integrity."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_16896_b200.graph import PRISMATIC, REVOLUTE, JointSpec
from tests import graph_cases as G


def test_identity_and_lower_limit_init(ref):
    g = O.RefGraph(8)
    a = g.add_node(0, "table")
    assert np.array_equal(g.world_poses(a), np.tile(np.eye(4), (8, 1, 1)))
    d = g.add_node(a, "drawer", -1, JointSpec(PRISMATIC, (1, 0, 0), 0.1, 0.4))
    assert np.array_equal(g.joint_states(d), np.full(8, 0.1))
    assert np.allclose(g.world_poses(d)[:, 0, 3], 0.1)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_batched_fk_equals_sequential(ref, seed):
    n = 16
    g = O.RefGraph(n)
    ids, specs = G.build(g, n, seed)
    assert g.is_tree()
    for nid in ids:
        wp = g.world_poses(nid)
        for i in range(0, n, 5):
            chain, cur = [], nid
            while cur != 0:
                chain.append(g.edge_batch(cur)[i])
                cur = specs[cur][0]
            acc = np.eye(4)
            for e in reversed(chain):
                acc = acc @ e
            assert np.allclose(wp[i], acc, atol=1e-9)
            assert np.allclose(g.world_pose(nid, i), wp[i], atol=1e-12)


def test_errors(ref):
    g = O.RefGraph(4)
    a = g.add_node(0, "a")
    with pytest.raises(ValueError):
        g.add_node(0, "a")
    with pytest.raises(IndexError):
        g.add_node(9, "b")
    with pytest.raises(ValueError):
        g.set_joint_states(a, [0, 0, 0, 0])
    bad = np.tile(np.eye(4), (4, 1, 1))
    bad[1, 3, 3] = 2.0
    with pytest.raises(ValueError):
        g.set_edge_batch(0, a, bad)
    j = g.add_node(a, "j", -1, JointSpec(REVOLUTE, (0, 0, 1), 0.0, 1.0))
    with pytest.raises(ValueError):
        g.set_joint_states(j, [0, 0.5, 1.5, 0])
