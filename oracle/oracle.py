"""TEST INFRASTRUCTURE ONLY: ctypes face of the oracle (oracle/_ref/libsbref.so).

libsbref.so is the UNMODIFIED reference (/root/reference/proj/src/*.cpp, compiled in place
by oracle/Makefile against oracle/shim) plus the builder-written rejection-loop driver
(oracle/ref_driver.cpp). Only tests/, __graft_entry__.smoke() and bench.py's reference /
cpu_baseline legs may import this module -- and only as the checker or the timed CPU
baseline, never as part of the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libsbref.so")
REF_SRC = "/root/reference/proj"

_lib = None


def build() -> str:
    """Compile the oracle (needs /root/reference; on the GPU box the prebuilt .so is used)."""
    if os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)
    if not os.path.exists(REF_LIB):
        raise FileNotFoundError(f"{REF_LIB} missing and /root/reference unavailable to build it")
    return REF_LIB


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(REF_LIB):
            build()
        L = C.CDLL(REF_LIB)
        u64, d = C.c_uint64, C.POINTER(C.c_double)
        L.ref_last_error.restype = C.c_char_p
        L.ref_mix64.restype = u64
        L.ref_mix64.argtypes = [u64]
        L.ref_stream_key2.restype = u64
        L.ref_stream_key2.argtypes = [u64, u64]
        L.ref_stream_key3.restype = u64
        L.ref_stream_key3.argtypes = [u64, u64, u64]
        L.ref_pcg_next_u64.restype = u64
        L.ref_pcg_next_u64.argtypes = [u64]
        L.ref_pcg_u32s.argtypes = [u64, C.c_void_p, C.c_uint32]
        L.ref_stream_doubles.argtypes = [u64, C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32]
        L.ref_mesh_fingerprint.restype = u64
        L.ref_mesh_fingerprint.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32]
        L.ref_region_fingerprint_rect.restype = u64
        L.ref_region_fingerprint_rect.argtypes = [C.c_double] * 4
        for name in ("ref_make_box",):
            getattr(L, name).argtypes = [C.c_double] * 3 + [C.c_void_p] * 4
        L.ref_make_cylinder.argtypes = [C.c_double, C.c_double, C.c_int] + [C.c_void_p] * 4
        L.ref_make_sphere.argtypes = [C.c_double, C.c_int, C.c_int] + [C.c_void_p] * 4
        L.ref_tri_tri.argtypes = [C.c_void_p]
        L.ref_tri_tri_batch.argtypes = [C.c_void_p, u64, C.c_void_p]
        L.ref_polygon_draws.argtypes = [C.c_void_p, C.c_uint32, u64, C.c_void_p, C.c_uint32,
                                        C.c_void_p, C.c_uint32]
        L.ref_triangulate.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p]
        L.ref_region_draws.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                       C.c_double, u64, C.c_void_p, C.c_uint32, C.c_void_p,
                                       C.c_uint32, C.c_void_p]
        L.ref_extract_support_surfaces.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32,
                                                   C.c_int32, C.c_void_p, C.c_uint32, C.c_void_p]
        L.ref_middle_polygon.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.c_void_p]
        L.ref_relation_region.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                                          C.c_double, C.c_void_p, C.c_uint32, C.c_void_p,
                                          C.c_void_p]
        L.ref_world_create.restype = C.c_void_p
        L.ref_world_create.argtypes = [u64, C.c_double, C.c_int]
        L.ref_world_destroy.argtypes = [C.c_void_p]
        L.ref_register_geometry.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p,
                                            C.c_uint32, C.c_void_p]
        L.ref_add_object.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
        L.ref_set_enabled.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, u64, C.c_int]
        L.ref_set_enabled_all.argtypes = [C.c_void_p, C.c_int32, C.c_int]
        L.ref_update_transforms.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
        L.ref_update_transform.argtypes = [C.c_void_p, C.c_int32, u64, C.c_void_p]
        L.ref_check_batch.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, u64,
                                      C.c_void_p, C.c_void_p]
        L.ref_get_stats.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_generate.argtypes = [C.c_void_p, C.c_void_p, u64, C.c_int, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p]
        L.ref_engine_create.restype = C.c_void_p
        L.ref_engine_create.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
        L.ref_engine_destroy.argtypes = [C.c_void_p]
        L.ref_engine_generate.argtypes = [C.c_void_p, u64, C.c_void_p, C.c_void_p]
        L.ref_sampler_create.restype = C.c_void_p
        L.ref_sampler_create.argtypes = [u64]
        L.ref_sampler_destroy.argtypes = [C.c_void_p]
        L.ref_sampler_prepare.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32,
                                          C.c_void_p, u64, u64]
        L.ref_sampler_sample.argtypes = [C.c_void_p, C.c_void_p, u64, C.c_void_p, u64, u64,
                                         C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_sampler_prepare_relation.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                   u64, u64]
        L.ref_sample_orientations.argtypes = [C.c_int, C.c_void_p, u64, C.c_void_p, C.c_void_p,
                                              u64, u64, u64, u64, C.c_void_p]
        L.ref_graph_create.restype = C.c_void_p
        L.ref_graph_create.argtypes = [u64]
        L.ref_graph_destroy.argtypes = [C.c_void_p]
        L.ref_graph_add_node.argtypes = [C.c_void_p, C.c_uint32, C.c_char_p, C.c_int64, C.c_int,
                                         C.c_int, C.c_void_p, C.c_double, C.c_double, C.c_void_p]
        L.ref_graph_set_edge_batch.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p]
        L.ref_graph_set_edge.argtypes = [C.c_void_p, C.c_uint32, u64, C.c_void_p]
        L.ref_graph_edge_batch.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]
        L.ref_graph_set_joint_states.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, u64]
        L.ref_graph_joint_states.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]
        L.ref_graph_world_poses.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]
        L.ref_graph_world_pose.argtypes = [C.c_void_p, C.c_uint32, u64, C.c_void_p]
        L.ref_graph_is_tree.argtypes = [C.c_void_p]
        L.ref_graph_mark_invalid.argtypes = [C.c_void_p, u64]
        L.ref_graph_valid_count.restype = u64
        L.ref_graph_valid_count.argtypes = [C.c_void_p]
        L.ref_reach_build.restype = C.c_void_p
        L.ref_reach_build.argtypes = [C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, u64,
                                      C.c_double, C.c_double, u64, C.c_int]
        L.ref_reach_destroy.argtypes = [C.c_void_p]
        L.ref_reach_save.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_reach_load.restype = C.c_void_p
        L.ref_reach_load.argtypes = [C.c_char_p]
        L.ref_reach_info.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_reach_cell_samples.restype = C.c_uint32
        L.ref_reach_cell_samples.argtypes = [C.c_void_p, u64, u64, u64]
        L.ref_reach_query_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, u64, C.c_int,
                                            C.c_double, C.c_void_p]
        L.ref_reach_placement_filter.argtypes = [C.c_void_p, C.c_void_p, u64, C.c_void_p,
                                                 C.c_void_p, C.c_uint32, C.c_void_p, u64,
                                                 C.c_void_p]
        L.ref_set_reach_filter.argtypes = [C.c_uint32, C.c_void_p, C.c_void_p, u64]
        L.ref_clear_reach_filters.argtypes = []
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def check(rc: int):
    if rc != 0:
        msg = lib().ref_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(msg)
        if rc == 2:
            raise IndexError(msg)
        raise RuntimeError(msg)


# ------------------------------------------------------------------ meshes / KATs
def make_box(sx, sy, sz):
    return _mesh(lib().ref_make_box, C.c_double(sx), C.c_double(sy), C.c_double(sz))


def make_cylinder(r, h, seg=32):
    return _mesh(lib().ref_make_cylinder, C.c_double(r), C.c_double(h), C.c_int(seg))


def make_sphere(r, stacks=12, slices=16):
    return _mesh(lib().ref_make_sphere, C.c_double(r), C.c_int(stacks), C.c_int(slices))


def _mesh(fn, *args):
    nv, nt = C.c_uint32(), C.c_uint32()
    check(fn(*args, None, C.byref(nv), None, C.byref(nt)))
    v = np.zeros((nv.value, 3))
    t = np.zeros((nt.value, 3), np.uint32)
    check(fn(*args, _p(v), C.byref(nv), _p(t), C.byref(nt)))
    return v, t


def tri_tri(p: np.ndarray) -> np.ndarray:
    """tri_tri_intersect over (n, 18) sextuples -> uint8 (n,)."""
    p = np.ascontiguousarray(p, dtype=np.float64).reshape(-1, 18)
    out = np.zeros(len(p), np.uint8)
    lib().ref_tri_tri_batch(_p(p), len(p), _p(out))
    return out


def stream_doubles(seed: int, counters, n: int) -> np.ndarray:
    c = np.ascontiguousarray(counters, dtype=np.uint64)
    out = np.zeros(n)
    lib().ref_stream_doubles(C.c_uint64(seed), _p(c), len(c), _p(out), n)
    return out


def polygon_draws(ring, seed: int, counters, n: int) -> np.ndarray:
    r = np.ascontiguousarray(ring, dtype=np.float64).reshape(-1, 2)
    c = np.ascontiguousarray(counters, dtype=np.uint64)
    out = np.zeros((n, 2))
    check(lib().ref_polygon_draws(_p(r), len(r), C.c_uint64(seed), _p(c), len(c), _p(out), n))
    return out


def triangulate(ring) -> np.ndarray:
    r = np.ascontiguousarray(ring, dtype=np.float64).reshape(-1, 2)
    out = np.zeros((512, 6))
    nt = C.c_uint32()
    check(lib().ref_triangulate(_p(r), len(r), _p(out), 512, C.byref(nt)))
    return out[: nt.value].reshape(-1, 3, 2)


def region_draws(rel_c, sup_c, states, ratio, fx, fy, seed, c, n):
    """region_for(0) of build_constraint_region (+ apply_ratio_on_support) for one instance's
    anchor states ((na, 3): x, y, yaw) -> (n draws (n, 2), sampler triangle count)."""
    st = np.ascontiguousarray(np.asarray(states, np.float64).reshape(-1))
    cc = np.ascontiguousarray(np.asarray(c, np.uint64))
    out = np.zeros((max(n, 1), 2))
    nt = C.c_int32()
    check(lib().ref_region_draws(C.byref(rel_c), C.byref(sup_c), _p(st) if st.size else None,
                                 ratio, fx, fy, seed, _p(cc), len(cc), _p(out), n, C.byref(nt)))
    return out[:n].copy(), nt.value


def extract_support_surfaces(vertices, triangles, mode=0):
    """extract_support_surfaces (mode 0 on / 1 inside) or extract_all_support_surfaces
    (mode -1) of the reference -> list of (polygon (k, 2), frame colmajor 16, roofed, area)."""
    class sb_surface(C.Structure):  # include/scenebatch_b200.h
        _fields_ = [("frame", C.c_double * 16), ("area", C.c_double), ("roofed", C.c_int32),
                    ("n_polygon", C.c_uint32), ("polygon_xy", C.c_double * 192)]

    v = np.ascontiguousarray(vertices, np.float64)
    t = np.ascontiguousarray(triangles, np.uint32)
    cap = 256
    arr = (sb_surface * cap)()
    n = C.c_uint32()
    check(lib().ref_extract_support_surfaces(_p(v), len(v), _p(t), len(t), mode, arr, cap,
                                             C.byref(n)))
    out = []
    for k in range(min(n.value, cap)):
        s = arr[k]
        out.append((np.array(s.polygon_xy[: 2 * s.n_polygon]).reshape(-1, 2), np.array(s.frame),
                    bool(s.roofed), s.area))
    return out


def middle_polygon(points):
    """middle_polygon (relationships.cpp:124-157) -> exterior ring (k, 2)."""
    xy = np.ascontiguousarray(np.asarray(points, np.float64).reshape(-1, 2))
    out = np.zeros((256, 2))
    k = C.c_uint32()
    check(lib().ref_middle_polygon(_p(xy), len(xy), _p(out), 256, C.byref(k)))
    return out[: k.value].copy()


def relation_region(rel_c, rect, ax, ay, ayaw):
    """build_constraint_region for one anchor state -> (exterior ring of part 0, n_parts)."""
    rc = np.ascontiguousarray(rect, dtype=np.float64)
    out = np.zeros((512, 2))
    npts, nparts = C.c_uint32(), C.c_uint32()
    check(lib().ref_relation_region(C.byref(rel_c), _p(rc), ax, ay, ayaw, _p(out), 512,
                                    C.byref(npts), C.byref(nparts)))
    return out[: npts.value].copy(), nparts.value


# ------------------------------------------------------------------ CollisionWorld
class RefWorld:
    def __init__(self, n: int, margin: float = 0.0, threads: int = 1):
        self.n = n
        self.h = lib().ref_world_create(n, margin, threads)
        if not self.h:
            raise ValueError(lib().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_world_destroy(self.h)
            self.h = None

    def register_geometry(self, v, t) -> int:
        v = np.ascontiguousarray(v, np.float64)
        t = np.ascontiguousarray(t, np.uint32)
        out = C.c_int32()
        check(lib().ref_register_geometry(self.h, _p(v), len(v), _p(t), len(t), C.byref(out)))
        return out.value

    def add_object(self, geom: int) -> int:
        out = C.c_int32()
        check(lib().ref_add_object(self.h, geom, C.byref(out)))
        return out.value

    def set_enabled(self, obj, inst, flag):
        i = np.ascontiguousarray(inst, np.uint32)
        check(lib().ref_set_enabled(self.h, obj, _p(i), len(i), int(flag)))

    def set_enabled_all(self, obj, flag):
        check(lib().ref_set_enabled_all(self.h, obj, int(flag)))

    def update_transforms(self, obj, poses_colmajor):
        p = np.ascontiguousarray(poses_colmajor, np.float64)
        check(lib().ref_update_transforms(self.h, obj, _p(p)))

    def update_transform(self, obj, inst, pose_colmajor):
        p = np.ascontiguousarray(pose_colmajor, np.float64)
        check(lib().ref_update_transform(self.h, obj, inst, _p(p)))

    def check_batch(self, geom, poses_colmajor, active):
        p = np.ascontiguousarray(poses_colmajor, np.float64).reshape(-1, 16)
        a = np.ascontiguousarray(active, np.uint32)
        free = np.ones(self.n, np.uint8)
        contact = np.full(self.n, -1, np.int32)
        check(lib().ref_check_batch(self.h, geom, _p(p), _p(a), len(a), _p(free), _p(contact)))
        return free, contact

    def stats(self):
        out = np.zeros(6, np.uint64)
        lib().ref_get_stats(self.h, _p(out))
        keys = ("geometry_registrations", "bvh_builds", "check_calls", "checked_instances",
                "narrow_phase_tests", "triangle_pair_tests")
        return dict(zip(keys, map(int, out)))


# ------------------------------------------------------------------ generation
TRACE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.c_int32, C.c_uint64,
                       C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.POINTER(C.c_uint8),
                       C.POINTER(C.c_uint8))


def generate(scene, run_seed: int, threads: int = 1, shard=None, with_poses: bool = True,
             trace=None):
    """Run the reference rejection loop on `scene` (a paper_2512_16896_b200.world.Scene).

    Returns dict(accepted (P, n) int16, valid (n,) uint8, poses (P, n, 16) colmajor | None,
    stats dict). `shard` is a paper_2512_16896_b200.world.Shard (or None)."""
    from paper_2512_16896_b200 import _capi as A  # data layout only

    sc, keep = scene.to_c()
    n = scene.n_instances if shard is None else shard.end - shard.begin
    P = len(scene.placements)
    acc = np.empty((P, n), np.int16)
    valid = np.empty(n, np.uint8)
    poses = np.empty((P, n, 16)) if with_poses else None
    res = A.sb_result(acc.ctypes.data_as(C.POINTER(C.c_int16)),
                      poses.ctypes.data_as(C.POINTER(C.c_double)) if with_poses else None,
                      valid.ctypes.data_as(C.POINTER(C.c_uint8)))
    st = A.sb_run_stats()
    sh = shard.to_c() if shard is not None else None
    cb = None
    if trace is not None:
        def _t(ctx, p, a, m, act, poses16, placeable, free):
            trace(p, a, np.ctypeslib.as_array(act, (m,)).copy(),
                  np.ctypeslib.as_array(poses16, (m, 16)).copy(),
                  np.ctypeslib.as_array(placeable, (m,)).copy(),
                  np.ctypeslib.as_array(free, (m,)).copy())
        cb = TRACE_FN(_t)
    rc = lib().ref_generate(C.byref(sc), C.byref(sh) if sh is not None else None,
                            C.c_uint64(run_seed), threads, C.byref(res), C.byref(st),
                            cb, None)
    check(rc)
    stats = {k: getattr(st, k) for k, _ in A.sb_run_stats._fields_}
    return {"accepted": acc, "valid": valid, "poses": poses, "stats": stats}


class RefEngine:
    """The rejection loop split into its cold part (constructor: RefWorld + ThreadPool,
    geometry registration / BVH builds, objects) and warm runs (generate), so a timer can
    bracket only the generation loop (warm time)."""

    def __init__(self, scene, threads: int = 1):
        self.scene = scene
        self._sc, self._keep = scene.to_c()
        self.h = lib().ref_engine_create(C.byref(self._sc), None, threads)
        if not self.h:
            raise ValueError(lib().ref_last_error().decode())
        self.n = scene.n_instances

    def close(self):
        if getattr(self, "h", None):
            lib().ref_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass

    def generate(self, run_seed: int, with_poses: bool = False):
        from paper_2512_16896_b200 import _capi as A  # data layout only

        P = len(self.scene.placements)
        acc = np.empty((P, self.n), np.int16)
        valid = np.empty(self.n, np.uint8)
        poses = np.empty((P, self.n, 16)) if with_poses else None
        res = A.sb_result(acc.ctypes.data_as(C.POINTER(C.c_int16)),
                          poses.ctypes.data_as(C.POINTER(C.c_double)) if with_poses else None,
                          valid.ctypes.data_as(C.POINTER(C.c_uint8)))
        st = A.sb_run_stats()
        check(lib().ref_engine_generate(self.h, C.c_uint64(run_seed), C.byref(res), C.byref(st)))
        stats = {k: getattr(st, k) for k, _ in A.sb_run_stats._fields_}
        return {"accepted": acc, "valid": valid, "poses": poses, "stats": stats}


def transformed_vertices(v, pose):
    """trimesh.cpp:112-118 (transform_point per vertex, transform.hpp:71-73) in the Eigen
    shim's order: ((r0 x + r1 y) + r2 z) + t, rounded once per operation."""
    v = np.asarray(v, np.float64)
    m = np.asarray(pose, np.float64)
    out = np.empty_like(v)
    for r in range(3):
        out[:, r] = ((m[r, 0] * v[:, 0] + m[r, 1] * v[:, 1]) + m[r, 2] * v[:, 2]) + m[r, 3]
    return out


def _rings(rings):
    """List of rings ((k, 2) xy arrays) -> flat xy (float64) and offsets (uint32)."""
    xy = np.ascontiguousarray(np.concatenate([np.asarray(r, np.float64).reshape(-1, 2) for r in rings])
                              if rings else np.zeros((0, 2)), dtype=np.float64)
    off = np.zeros(len(rings) + 1, np.uint32)
    for i, r in enumerate(rings):
        off[i + 1] = off[i] + len(r)
    return xy, off


class RefSampler:
    """The reference's PositionSampler (sampler.hpp:71-96) over a region given as rings."""

    def __init__(self, salt: int):
        self.h = lib().ref_sampler_create(salt)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ref_sampler_destroy(self.h)
                self.h = None
        except Exception:  # interpreter shutdown
            pass

    def prepare(self, rings, n: int, run_seed: int, instance_rings=None):
        self._xy, self._off = _rings(rings)
        self._inst = None if instance_rings is None else np.ascontiguousarray(instance_rings, np.uint32)
        check(lib().ref_sampler_prepare(self.h, _p(self._xy), _p(self._off), len(rings),
                                        None if self._inst is None else _p(self._inst), n, run_seed))

    def prepare_relation(self, rel_c, rect, states, n: int, run_seed: int):
        rc = np.ascontiguousarray(rect, np.float64)
        self._st = np.ascontiguousarray(states, np.float64).reshape(-1, 3)
        check(lib().ref_sampler_prepare_relation(self.h, C.byref(rel_c), _p(rc), _p(self._st), n,
                                                 run_seed))

    def sample(self, support16: np.ndarray, active, attempt: int):
        sw = np.ascontiguousarray(support16, np.float64)
        act = np.ascontiguousarray(active, np.uint32)
        pos = np.zeros((len(act), 3))
        pl = np.zeros(len(act), np.uint8)
        rc = C.c_uint64()
        check(lib().ref_sampler_sample(self.h, _p(sw), sw.shape[0], _p(act), len(act), attempt,
                                       _p(pos), _p(pl), C.byref(rc)))
        return pos, pl, rc.value


def sample_orientations(kind: int, active, positions, face_xy, run_seed: int, salt: int,
                        attempt: int) -> np.ndarray:
    act = np.ascontiguousarray(active, np.uint32)
    pos = np.ascontiguousarray(positions, np.float64)
    fx = None if face_xy is None else np.ascontiguousarray(face_xy, np.float64)
    y = np.zeros(len(act))
    check(lib().ref_sample_orientations(kind, _p(act), len(act), _p(pos),
                                        None if fx is None else _p(fx),
                                        0 if fx is None else fx.shape[0], run_seed, salt, attempt,
                                        _p(y)))
    return y


def _cm(poses):  # (..., 4, 4) -> column-major (..., 16)
    p = np.asarray(poses, np.float64)
    return np.ascontiguousarray(np.swapaxes(p, -1, -2)).reshape(p.shape[:-2] + (16,))


def _uncm(flat):
    f = np.asarray(flat, np.float64)
    return np.swapaxes(f.reshape(f.shape[:-1] + (4, 4)), -1, -2).copy()


class RefGraph:
    """The reference's BatchedSceneGraph (scene_graph.cpp) with the package's Python API."""

    def __init__(self, n: int):
        self.h = lib().ref_graph_create(n)
        if not self.h:
            raise ValueError(lib().ref_last_error().decode())
        self.n = n

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ref_graph_destroy(self.h)
                self.h = None
        except Exception:  # interpreter shutdown
            pass

    def add_node(self, parent, name, geometry_id=-1, joint=None):
        out = C.c_uint32()
        ax = np.ascontiguousarray(joint.axis if joint is not None else (0, 0, 1), np.float64)
        check(lib().ref_graph_add_node(self.h, parent, name.encode(), geometry_id,
                                       1 if joint is not None else 0,
                                       joint.kind if joint is not None else 0, _p(ax),
                                       joint.lo if joint is not None else 0.0,
                                       joint.hi if joint is not None else 0.0, C.byref(out)))
        return out.value

    def set_edge_batch(self, parent, child, transforms):
        t = _cm(transforms).reshape(-1, 16)
        check(lib().ref_graph_set_edge_batch(self.h, parent, child, _p(t)))

    def set_edge(self, child, instance, transform):
        t = _cm(transform).reshape(16)
        check(lib().ref_graph_set_edge(self.h, child, instance, _p(t)))

    def _batch(self, fn, node):
        out = np.empty((self.n, 16))
        check(fn(self.h, node, _p(out)))
        return _uncm(out)

    def edge_batch(self, child):
        return self._batch(lib().ref_graph_edge_batch, child)

    def world_poses(self, node):
        return self._batch(lib().ref_graph_world_poses, node)

    def world_pose(self, node, instance):
        out = np.empty(16)
        check(lib().ref_graph_world_pose(self.h, node, instance, _p(out)))
        return _uncm(out)

    def set_joint_states(self, node, values):
        v = np.ascontiguousarray(values, np.float64)
        check(lib().ref_graph_set_joint_states(self.h, node, _p(v), len(v)))

    def joint_states(self, node):
        out = np.empty(self.n)
        check(lib().ref_graph_joint_states(self.h, node, _p(out)))
        return out

    def is_tree(self):
        return bool(lib().ref_graph_is_tree(self.h))

    def mark_invalid(self, i):
        lib().ref_graph_mark_invalid(self.h, i)

    def valid_count(self):
        return lib().ref_graph_valid_count(self.h)


class RefReachMap:
    """The reference's ReachMap4D (reachability.cpp) built / loaded through oracle/_ref."""

    def __init__(self, h):
        if not h:
            raise RuntimeError(lib().ref_last_error().decode())
        self.h = h

    @classmethod
    def build(cls, chain, samples, resolution, psi_resolution, seed, threads=1):
        n = len(chain.links)
        org = np.ascontiguousarray(np.concatenate([_cm(l.origin).reshape(1, 16) for l in chain.links]))
        jt = np.ascontiguousarray([[float(l.joint.kind), *map(float, l.joint.axis), l.joint.lo,
                                    l.joint.hi] for l in chain.links], np.float64)
        ee = _cm(chain.ee_offset).reshape(16)
        return cls(lib().ref_reach_build(n, _p(org), _p(jt), _p(ee), samples, resolution,
                                         psi_resolution, seed, threads))

    @classmethod
    def load(cls, path):
        return cls(lib().ref_reach_load(path.encode()))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().ref_reach_destroy(self.h)
                self.h = None
        except Exception:  # interpreter shutdown
            pass

    def save(self, path):
        check(lib().ref_reach_save(self.h, path.encode()))

    def info(self):
        o = np.zeros(6)
        lib().ref_reach_info(self.h, _p(o))
        return dict(zip(("samples", "resolution", "psi_resolution", "max_radius", "cell_count",
                         "occupied_cells"), o.tolist()))

    def cell_samples(self, ir, iz, ip):
        return lib().ref_reach_cell_samples(self.h, ir, iz, ip)

    def query_batch(self, base_poses, targets, inclination=None):
        b = _cm(base_poses).reshape(-1, 16)
        t = np.ascontiguousarray(targets, np.float64).reshape(-1, 3)
        out = np.zeros(len(t), np.uint8)
        check(lib().ref_reach_query_batch(self.h, _p(b), _p(t), len(t),
                                          0 if inclination is None else 1,
                                          0.0 if inclination is None else inclination, _p(out)))
        return out

    def placement_filter(self, robot_base, frames, active):
        b = _cm(robot_base).reshape(-1, 16)
        n = len(b)
        pres = np.array([f is not None for f in frames], np.uint8)
        fr = np.ascontiguousarray(np.concatenate(
            [(_cm(f).reshape(-1, 16) if f is not None else np.zeros((n, 16))) for f in frames])
            if frames else np.zeros((0, 16)))
        act = np.ascontiguousarray(active, np.uint32)
        out = np.zeros(len(act), np.uint8)
        check(lib().ref_reach_placement_filter(self.h, _p(b), n, _p(fr), _p(pres), len(frames),
                                               _p(act), len(act), _p(out)))
        return out


def set_reach_filter(placement: int, refmap, robot_base):
    """Appendix C item 8 for ref generate: refmap = RefReachMap (kept alive by the caller),
    robot_base = (N_total, 4, 4); None clears it."""
    if refmap is None:
        check(lib().ref_set_reach_filter(placement, None, None, 0))
        return
    b = _cm(robot_base).reshape(-1, 16)
    check(lib().ref_set_reach_filter(placement, refmap.h, _p(b), len(b)))


def clear_reach_filters():
    lib().ref_clear_reach_filters()
