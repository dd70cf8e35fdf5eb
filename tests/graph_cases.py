"""Random BatchedSceneGraph scenarios (SPEC scene_graph properties: random trees of depth
<= 5, random rigid edges, revolute / prismatic joints) applied to any implementation with
the package's graph API, so the device graph and the reference see the same history."""
import math

import numpy as np

from paper_2512_16896_b200.graph import PRISMATIC, REVOLUTE, JointSpec


def rigid(rng, n, spread=1.0):
    out = np.tile(np.eye(4), (n, 1, 1))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    out[:, 0, 0] = 1 - 2 * (y * y + z * z)
    out[:, 0, 1] = 2 * (x * y - z * w)
    out[:, 0, 2] = 2 * (x * z + y * w)
    out[:, 1, 0] = 2 * (x * y + z * w)
    out[:, 1, 1] = 1 - 2 * (x * x + z * z)
    out[:, 1, 2] = 2 * (y * z - x * w)
    out[:, 2, 0] = 2 * (x * z - y * w)
    out[:, 2, 1] = 2 * (y * z + x * w)
    out[:, 2, 2] = 1 - 2 * (x * x + y * y)
    out[:, :3, 3] = rng.uniform(-spread, spread, size=(n, 3))
    return out


def build(g, n, seed, n_nodes=12, joints=True):
    """Random tree of depth <= 5; returns the node ids, their depths and joint specs."""
    rng = np.random.default_rng(seed)
    ids, depth, specs = [0], {0: 0}, {}
    for k in range(n_nodes):
        parent = int(rng.choice([i for i in ids if depth[i] < 5]))
        joint = None
        if joints and rng.random() < 0.4:
            kind = REVOLUTE if rng.random() < 0.5 else PRISMATIC
            axis = tuple(rng.normal(size=3) * (1.0 if rng.random() < 0.5 else 2.5))
            lo = float(rng.uniform(-1.0, 0.0))
            joint = JointSpec(kind, axis, lo, lo + float(rng.uniform(0.1, 1.5)))
        nid = g.add_node(parent, f"n{k}", int(rng.integers(-1, 5)), joint)
        ids.append(nid)
        depth[nid] = depth[parent] + 1
        specs[nid] = (parent, joint)
    for nid, (parent, joint) in specs.items():
        if rng.random() < 0.8:
            g.set_edge_batch(parent, nid, rigid(rng, n))
        if joint is not None and rng.random() < 0.8:
            g.set_joint_states(nid, rng.uniform(joint.lo, joint.hi, size=n))
    for _ in range(3):  # single-instance edge updates
        nid = int(rng.choice(ids[1:]))
        g.set_edge(nid, int(rng.integers(n)), rigid(rng, 1)[0])
    return ids, specs
