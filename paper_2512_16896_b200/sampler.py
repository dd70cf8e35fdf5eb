"""``PositionSampler`` and ``sample_orientations`` (sampler.hpp:66-104) over the C ABI.

Mirrors the reference class: ``PositionSampler(placement_salt)``, ``prepare(region,
batch_size, run_seed)``, ``sample(support_world, active, attempt) -> (positions,
placeable)``, plus ``cache_info()`` for the SampleCache state (sampler.hpp:18-36). A region
is a list of hole-free rings ((k, 2) arrays) -- the canonical ``ConstraintRegion::region``
-- or, with ``per_instance=True``, one such list per instance
(``ConstraintRegion::regions_by_instance``). Points are drawn on the GPU; the FIFO cache is
host bookkeeping of draw indices (see sb_runtime.cpp "PositionSampler").
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _capi as A
from .world import _dp, _up, colmajor

FIXED, UNIFORM_YAW, FACE_TO = 0, 1, 2  # OrientationRule::Kind (sampler.hpp:53-57)


def _flatten(rings: Sequence[np.ndarray]):
    xy = [np.asarray(r, np.float64).reshape(-1, 2) for r in rings]
    off = np.zeros(len(xy) + 1, np.uint32)
    for i, r in enumerate(xy):
        off[i + 1] = off[i] + len(r)
    flat = np.ascontiguousarray(np.concatenate(xy) if xy else np.zeros((0, 2)), np.float64)
    return flat, off


class PositionSampler:
    def __init__(self, placement_salt: int, device: int = 0):
        h = C.c_void_p()
        A.check(A.lib().sb_sampler_create(placement_salt, device, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            A.lib().sb_sampler_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prepare(self, region, batch_size: int, run_seed: int, per_instance: bool = False):
        if per_instance:
            if len(region) != batch_size:
                raise ValueError("prepare: one region per instance expected")
            rings, inst = [], np.zeros(batch_size + 1, np.uint32)
            for i, reg in enumerate(region):
                rings.extend(reg)
                inst[i + 1] = len(rings)
        else:
            rings, inst = list(region), None
        self._xy, self._off = _flatten(rings)
        self._inst = inst
        A.check(A.lib().sb_sampler_prepare(self._h, _dp(self._xy), _up(self._off), len(rings),
                                           None if inst is None else _up(inst), batch_size,
                                           run_seed))

    def prepare_relation(self, relation, support_rect, anchor_states, run_seed: int):
        """build_constraint_region + prepare on the device. relation: world.Relation
        (anchor >= 0 = anchored); anchor_states: (N, 3) x, y, yaw in the support frame."""
        st = np.ascontiguousarray(anchor_states, np.float64).reshape(-1, 3)
        rect = np.ascontiguousarray(support_rect, np.float64)
        r = relation.to_c()
        A.check(A.lib().sb_sampler_prepare_relation(self._h, C.byref(r), _dp(rect), _dp(st),
                                                    len(st), run_seed))

    def sample(self, support_world: np.ndarray, active: Sequence[int], attempt: int):
        """support_world: (N, 4, 4) poses. Returns (positions (m, 3), placeable uint8 (m,))."""
        sw = colmajor(np.asarray(support_world, np.float64)).reshape(-1, 16)
        act = np.ascontiguousarray(active, np.uint32)
        pos = np.zeros((len(act), 3))
        pl = np.zeros(len(act), np.uint8)
        A.check(A.lib().sb_sampler_sample(self._h, _dp(sw), _up(act), len(act), attempt, _dp(pos),
                                          pl.ctypes.data_as(C.POINTER(C.c_uint8))))
        return pos, pl

    def sample_device(self, d_support16: int, d_active: int, m: int, attempt: int,
                      d_positions: int, d_placeable: int, stream: int = 0) -> None:
        """Device-resident sample (raw device pointers, e.g. torch .data_ptr()): supports
        (N column-major Mat4), active (u32), positions (m x 3 f64), placeable (u8); enqueued
        on `stream` (a cudaStream_t as int)."""
        A.check(A.lib().sb_sampler_sample_device(self._h, d_support16, d_active, m, attempt,
                                                 d_positions, d_placeable, stream or None))

    def cache_info(self):
        q, r = C.c_uint64(), C.c_uint64()
        A.check(A.lib().sb_sampler_cache_info(self._h, C.byref(q), C.byref(r)))
        return q.value, r.value


def sample_orientations(kind: int, active: Sequence[int], positions: Optional[np.ndarray],
                        face_targets: Optional[np.ndarray], run_seed: int, placement_salt: int,
                        attempt: int, device: int = 0) -> np.ndarray:
    """sampler.cpp:129-156; face_targets: (N, 2) target xy per instance (FACE_TO only)."""
    act = np.ascontiguousarray(active, np.uint32)
    pos = None if positions is None else np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
    ft = None if face_targets is None else np.ascontiguousarray(face_targets, np.float64).reshape(-1, 2)
    y = np.zeros(len(act))
    A.check(A.lib().sb_sample_orientations(kind, _up(act), len(act),
                                           None if pos is None else _dp(pos),
                                           None if ft is None else _dp(ft),
                                           0 if ft is None else len(ft), run_seed, placement_salt,
                                           attempt, _dp(y), device))
    return y


def sample_orientations_device(kind: int, d_active: int, m: int, d_positions: int,
                               d_face_targets: int, run_seed: int, placement_salt: int,
                               attempt: int, d_yaws: int, stream: int = 0) -> None:
    """sample_orientations on device pointers (e.g. torch .data_ptr()), on `stream`."""
    A.check(A.lib().sb_sample_orientations_device(kind, d_active, m, d_positions or None,
                                                  d_face_targets or None, run_seed,
                                                  placement_salt, attempt, d_yaws,
                                                  stream or None))
