"""Kinematic chains and query batches shared by the reachability oracle (CPU) and device
parity (GPU) tests. The arm: yaw about z, shoulder and elbow about y, a prismatic wrist."""
import math

import numpy as np

from paper_2512_16896_b200.graph import PRISMATIC, REVOLUTE, JointSpec
from paper_2512_16896_b200.reach import ChainLink, KinematicChain


def translation(x, y, z):
    m = np.eye(4)
    m[:3, 3] = (x, y, z)
    return m


def arm():
    return KinematicChain(
        links=[ChainLink(translation(0, 0, 0.3), JointSpec(REVOLUTE, (0, 0, 1), -math.pi, math.pi)),
               ChainLink(translation(0, 0, 0.1), JointSpec(REVOLUTE, (0, 1, 0), -1.5, 1.5)),
               ChainLink(translation(0.4, 0, 0), JointSpec(REVOLUTE, (0, 2, 0), -2.0, 2.0)),
               ChainLink(translation(0.3, 0, 0), JointSpec(PRISMATIC, (1, 0, 0), 0.0, 0.1))],
        ee_offset=translation(0.05, 0, 0))


def planar():  # 1-joint planar arm, link 1 m (SPEC: occupied cells form a circle r = 1)
    return KinematicChain(links=[ChainLink(np.eye(4), JointSpec(REVOLUTE, (0, 0, 1), -math.pi, math.pi))],
                          ee_offset=translation(1.0, 0, 0))


def bases(n, seed):
    rng = np.random.default_rng(seed)
    out = np.tile(np.eye(4), (n, 1, 1))
    a = rng.uniform(-math.pi, math.pi, n)
    out[:, 0, 0], out[:, 0, 1], out[:, 1, 0], out[:, 1, 1] = np.cos(a), -np.sin(a), np.sin(a), np.cos(a)
    out[:, :3, 3] = rng.uniform(-0.5, 0.5, (n, 3))
    return out


def targets(n, seed, spread=1.3):
    return np.random.default_rng(seed + 100).uniform(-spread, spread, (n, 3))
