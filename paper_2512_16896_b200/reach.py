"""``ReachMap4D`` / ``KinematicChain`` / ``placement_filter`` (reachability.hpp:14-94) over
the C ABI: the FK-sampled occupancy map is built and queried on the GPU; ``save`` / ``load``
read and write the reference's "SBRM" v1 files byte for byte."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi as A
from .graph import JointSpec
from .world import _dp, _up, colmajor


@dataclass
class ChainLink:
    origin: np.ndarray = field(default_factory=lambda: np.eye(4))
    joint: JointSpec = field(default_factory=JointSpec)


@dataclass
class KinematicChain:
    links: List[ChainLink] = field(default_factory=list)
    ee_offset: np.ndarray = field(default_factory=lambda: np.eye(4))


class ReachMap4D:
    def __init__(self, _handle):
        self._h = _handle

    @classmethod
    def build(cls, chain: KinematicChain, samples: int, resolution: float,
              psi_resolution: float, seed: int, device: int = 0) -> "ReachMap4D":
        links = (A.sb_chain_link * max(1, len(chain.links)))()
        for i, l in enumerate(chain.links):
            links[i].origin[:] = list(colmajor(np.asarray(l.origin, np.float64)))
            links[i].joint = l.joint.to_c()
        ee = colmajor(np.asarray(chain.ee_offset, np.float64))
        h = C.c_void_p()
        A.check(A.lib().sb_reach_build(links, len(chain.links), _dp(ee), samples, resolution,
                                       psi_resolution, seed, device, C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path: str, device: int = 0) -> "ReachMap4D":
        h = C.c_void_p()
        A.check(A.lib().sb_reach_load(path.encode(), device, C.byref(h)))
        return cls(h)

    def save(self, path: str) -> None:
        A.check(A.lib().sb_reach_save(self._h, path.encode()))

    def close(self):
        if getattr(self, "_h", None):
            A.lib().sb_reach_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        o = A.sb_reach_info()
        A.check(A.lib().sb_reach_get_info(self._h, C.byref(o)))
        return {k: getattr(o, k) for k, _ in A.sb_reach_info._fields_}

    def built(self) -> bool:
        return self.info()["nr"] > 0

    def cell_samples(self, ir: int, iz: int, ipsi: int) -> int:
        c = C.c_uint32()
        A.check(A.lib().sb_reach_cell_samples(self._h, ir, iz, ipsi, C.byref(c)))
        return c.value

    def query_batch(self, base_poses: np.ndarray, targets: np.ndarray,
                    inclination: Optional[float] = None) -> np.ndarray:
        b = colmajor(np.asarray(base_poses, np.float64)).reshape(-1, 16)
        t = np.ascontiguousarray(targets, np.float64).reshape(-1, 3)
        if len(b) != len(t):
            raise ValueError("query_batch: size mismatch")
        out = np.zeros(len(t), np.uint8)
        A.check(A.lib().sb_reach_query_batch(self._h, _dp(b), _dp(t), len(t),
                                             0 if inclination is None else 1,
                                             0.0 if inclination is None else inclination,
                                             out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out

    def query_batch_device(self, d_base16: int, d_targets: int, n: int, d_out: int,
                           inclination: Optional[float] = None, stream: int = 0) -> None:
        """query_batch on device pointers (N column-major Mat4, N x 3 f64, N u8)."""
        A.check(A.lib().sb_reach_query_batch_device(
            self._h, d_base16, d_targets, n, 0 if inclination is None else 1,
            0.0 if inclination is None else inclination, d_out, stream or None))

    def query(self, target_in_base, inclination: Optional[float] = None) -> bool:
        return bool(self.query_batch(np.eye(4)[None], np.asarray(target_in_base)[None],
                                     inclination)[0])


def placement_filter(m: ReachMap4D, robot_base: np.ndarray,
                     frames: Sequence[Optional[np.ndarray]], active) -> np.ndarray:
    """reachability.cpp:164-190: instance passes when every frame origin is reachable."""
    b = colmajor(np.asarray(robot_base, np.float64)).reshape(-1, 16)
    n = len(b)
    keep = [None if f is None else colmajor(np.asarray(f, np.float64)).reshape(-1, 16)
            for f in frames]
    ptrs = (C.POINTER(C.c_double) * max(1, len(keep)))()
    for i, f in enumerate(keep):
        if f is not None:
            if len(f) != n:
                raise ValueError("placement_filter: frame batch size mismatch")
            ptrs[i] = _dp(f)
    act = np.ascontiguousarray(active, np.uint32)
    out = np.zeros(len(act), np.uint8)
    A.check(A.lib().sb_reach_placement_filter(m._h, _dp(b), n, ptrs, len(keep), _up(act),
                                              len(act), out.ctypes.data_as(C.POINTER(C.c_uint8))))
    return out
