"""``BatchedSceneGraph`` / ``JointSpec`` (scene_graph.hpp:19-94) over the C ABI.

Every edge batch lives on the GPU; ``world_poses`` is the batched forward kinematics kernel
(sb_graph.cu). Poses are numpy (N, 4, 4) float64 arrays (row, col), crossing the ABI
column-major like a reference ``TransformBatch``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _capi as A
from .world import _dp, colmajor, from_colmajor

REVOLUTE, PRISMATIC = 0, 1


@dataclass
class JointSpec:
    kind: int = REVOLUTE
    axis: tuple = (0.0, 0.0, 1.0)
    lo: float = 0.0
    hi: float = 0.0

    def to_c(self) -> "A.sb_joint":
        return A.sb_joint(self.kind, (C.c_double * 3)(*map(float, self.axis)), self.lo, self.hi)


class BatchedSceneGraph:
    def __init__(self, batch_size: int, device: int = 0):
        h = C.c_void_p()
        A.check(A.lib().sb_graph_create(batch_size, device, C.byref(h)))
        self._h, self.n = h, batch_size

    def close(self):
        if getattr(self, "_h", None):
            A.lib().sb_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def batch_size(self) -> int:
        return self.n

    def root(self) -> int:
        return 0

    def add_node(self, parent: int, name: str, geometry_id: int = -1,
                 joint: Optional[JointSpec] = None) -> int:
        out = C.c_uint32()
        j = joint.to_c() if joint is not None else None
        A.check(A.lib().sb_graph_add_node(self._h, parent, name.encode(), geometry_id,
                                          C.byref(j) if j is not None else None, C.byref(out)))
        return out.value

    def set_edge_batch(self, parent: int, child: int, transforms: np.ndarray) -> None:
        t = colmajor(np.asarray(transforms, np.float64)).reshape(-1, 16)
        if len(t) != self.n:
            raise ValueError("transform batch size mismatch")
        A.check(A.lib().sb_graph_set_edge_batch(self._h, parent, child, _dp(t)))

    def set_edge(self, child: int, instance: int, transform: np.ndarray) -> None:
        t = colmajor(np.asarray(transform, np.float64)).reshape(16)
        A.check(A.lib().sb_graph_set_edge(self._h, child, instance, _dp(t)))

    def _batch(self, fn, node: int) -> np.ndarray:
        out = np.empty((self.n, 16))
        A.check(fn(self._h, node, _dp(out)))
        return from_colmajor(out)

    def edge_batch(self, child: int) -> np.ndarray:
        return self._batch(A.lib().sb_graph_edge_batch, child)

    def world_poses(self, node: int) -> np.ndarray:
        return self._batch(A.lib().sb_graph_world_poses, node)

    def world_poses_device(self, node: int, d_out16: int, stream: int = 0) -> None:
        """Batched FK into device memory (N column-major Mat4 at d_out16), on `stream`."""
        A.check(A.lib().sb_graph_world_poses_device(self._h, node, d_out16, stream or None))

    def world_pose(self, node: int, instance: int) -> np.ndarray:
        out = np.empty(16)
        A.check(A.lib().sb_graph_world_pose(self._h, node, instance, _dp(out)))
        return from_colmajor(out)

    def set_joint_states(self, node: int, values: Sequence[float]) -> None:
        v = np.ascontiguousarray(values, np.float64)
        if len(v) != self.n:
            raise ValueError("joint value batch size mismatch")
        A.check(A.lib().sb_graph_set_joint_states(self._h, node, _dp(v)))

    def joint_states(self, node: int) -> np.ndarray:
        out = np.empty(self.n)
        A.check(A.lib().sb_graph_joint_states(self._h, node, _dp(out)))
        return out

    def find(self, name: str) -> Optional[int]:
        out = C.c_int64()
        A.check(A.lib().sb_graph_find(self._h, name.encode(), C.byref(out)))
        return None if out.value < 0 else out.value

    def _info(self, node: int):
        name, parent, geom, art = C.c_char_p(), C.c_uint32(), C.c_int64(), C.c_int()
        j = A.sb_joint()
        A.check(A.lib().sb_graph_node_info(self._h, node, C.byref(name), C.byref(parent),
                                           C.byref(geom), C.byref(art), C.byref(j)))
        return name.value.decode(), parent.value, geom.value, bool(art.value), j

    def name(self, node: int) -> str:
        return self._info(node)[0]

    def parent(self, node: int) -> int:
        return self._info(node)[1]

    def geometry(self, node: int) -> int:
        return self._info(node)[2]

    def articulated(self, node: int) -> bool:
        return self._info(node)[3]

    def joint(self, node: int) -> Optional[JointSpec]:
        _, _, _, art, j = self._info(node)
        return JointSpec(j.kind, tuple(j.axis), j.lo, j.hi) if art else None

    def node_count(self) -> int:
        return A.lib().sb_graph_node_count(self._h)

    def children(self, node: int) -> List[int]:
        cnt = C.c_uint32()
        A.check(A.lib().sb_graph_children(self._h, node, None, 0, C.byref(cnt)))
        out = (C.c_uint32 * max(1, cnt.value))()
        A.check(A.lib().sb_graph_children(self._h, node, out, cnt.value, C.byref(cnt)))
        return list(out)[:cnt.value]

    def is_tree(self) -> bool:
        t = C.c_int()
        A.check(A.lib().sb_graph_is_tree(self._h, C.byref(t)))
        return bool(t.value)

    def valid_mask(self) -> np.ndarray:
        m = np.empty(self.n, np.uint8)
        A.check(A.lib().sb_graph_valid_mask(self._h, m.ctypes.data_as(C.POINTER(C.c_uint8))))
        return m

    def valid(self, instance: int) -> bool:
        if not 0 <= instance < self.n:
            raise IndexError("instance out of range")
        return bool(self.valid_mask()[instance])

    def mark_invalid(self, instance: int) -> None:
        A.check(A.lib().sb_graph_mark_invalid(self._h, instance))

    def reset_validity(self) -> None:
        A.check(A.lib().sb_graph_reset_validity(self._h))

    def valid_count(self) -> int:
        c = C.c_uint64()
        A.check(A.lib().sb_graph_valid_count(self._h, C.byref(c)))
        return c.value
