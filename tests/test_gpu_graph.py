"""GPU parity of the device BatchedSceneGraph (sb_graph_*) against the reference
(oracle/_ref): random trees with rigid edges, revolute / prismatic joints and
single-instance updates; batched FK, world_pose, edges, joint states, validity, errors,
and the engine's accepted-pose write-back."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_16896_b200 import scenes
from paper_2512_16896_b200.graph import PRISMATIC, REVOLUTE, JointSpec
from tests import graph_cases as G

pytestmark = pytest.mark.gpu


def _close(got, want, specs, nid):
    """Bit-exact unless a revolute joint sits on the chain: its sin/cos is correctly
    rounded on the device and glibc's can be 1 ulp off."""
    cur, rev = nid, False
    while cur != 0:
        j = specs[cur][1]
        rev = rev or (j is not None and j.kind == REVOLUTE)
        cur = specs[cur][0]
    if not rev:
        assert np.array_equal(got, want)
    else:
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)
        assert np.mean(got == want) > 0.99


@pytest.mark.parametrize("n,seed", [(64, 0), (1000, 1), (4096, 2)])
def test_graph_matches_reference(gpu, ref, n, seed):
    D, R = gpu.BatchedSceneGraph(n), O.RefGraph(n)
    ids, specs = G.build(D, n, seed)
    ids_r, _ = G.build(R, n, seed)
    assert ids == ids_r and D.is_tree() and D.node_count() == len(ids)
    for nid in ids[1:]:
        _close(D.edge_batch(nid), R.edge_batch(nid), specs, nid)
        _close(D.world_poses(nid), R.world_poses(nid), specs, nid)
        for i in (0, n // 2, n - 1):
            _close(D.world_pose(nid, i), R.world_pose(nid, i), specs, nid)
        j = specs[nid][1]
        if j is not None:
            assert np.array_equal(D.joint_states(nid), R.joint_states(nid))
            assert D.articulated(nid) and D.joint(nid).kind == j.kind
        assert D.parent(nid) == specs[nid][0] and D.name(nid) == f"n{ids.index(nid) - 1}"
    assert D.find("n3") == ids[4] and D.find("nope") is None
    assert D.children(0) == [k for k in ids[1:] if specs[k][0] == 0]


def test_graph_validity_and_errors(gpu):
    g = gpu.BatchedSceneGraph(8)
    a = g.add_node(0, "a", 2)
    assert g.valid_count() == 8
    g.mark_invalid(3)
    g.mark_invalid(5)
    assert g.valid_count() == 6 and not g.valid(3) and list(g.valid_mask()) == [1, 1, 1, 0, 1, 0, 1, 1]
    g.reset_validity()
    assert g.valid_count() == 8
    with pytest.raises(ValueError):
        g.add_node(0, "a")
    with pytest.raises(IndexError):
        g.add_node(7, "b")
    with pytest.raises(ValueError):
        g.set_joint_states(a, np.zeros(8))
    with pytest.raises(ValueError):
        g.set_edge(0, 0, np.eye(4))
    with pytest.raises(IndexError):
        g.set_edge(a, 8, np.eye(4))
    b = g.add_node(a, "b")
    with pytest.raises(ValueError):  # not an edge
        g.set_edge_batch(0, b, np.tile(np.eye(4), (8, 1, 1)))
    bad = np.tile(np.eye(4), (8, 1, 1))
    bad[2, 3, 0] = 1e-3
    with pytest.raises(ValueError):
        g.set_edge_batch(0, a, bad)
    j = g.add_node(a, "j", -1, JointSpec(PRISMATIC, (0, 0, 2), 0.0, 0.5))
    assert np.allclose(g.joint(j).axis, (0, 0, 1))  # normalised
    with pytest.raises(ValueError):
        g.set_joint_states(j, np.full(8, 0.6))
    with pytest.raises(ValueError):
        g.add_node(0, "z", -1, JointSpec(REVOLUTE, (0, 0, 0), 0, 1))
    with pytest.raises(ValueError):
        g.add_node(0, "z", -1, JointSpec(REVOLUTE, (0, 0, 1), 1, 0))


def test_engine_write_back(gpu, ref):
    """Accepted poses of a placement land in the graph (device to device) and the run's
    invalid instances are marked invalid; an articulated node takes them as its base."""
    scene = scenes.tabletop_boxes(512, n_objects=6, attempts=8)
    eng = gpu.Engine(scene)
    res = eng.generate(3)
    g = gpu.BatchedSceneGraph(512)
    nodes = [g.add_node(0, f"obj{p}") for p in range(len(scene.placements))]
    for p, node in enumerate(nodes):
        eng.write_back(p, g, node)
        assert np.array_equal(g.world_poses(node), res.poses[p])
    assert np.array_equal(g.valid_mask(), res.valid)
    lid = g.add_node(nodes[0], "lid", -1, JointSpec(PRISMATIC, (0, 0, 1), 0.0, 0.1))
    g.set_joint_states(lid, np.full(512, 0.05))
    want = res.poses[0].copy()
    want[:, :3, 3] += want[:, :3, 2] * 0.05
    np.testing.assert_allclose(g.world_poses(lid), want, atol=1e-12)
    with pytest.raises(ValueError):
        eng.write_back(0, g, lid)  # not a child of the root
