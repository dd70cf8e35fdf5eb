"""Python face of the C-ABI drop-in, mirroring the reference's scenebatch class API.

Names and argument meaning follow /root/reference/proj/include/scenebatch:
``TriMesh`` / ``make_box`` / ``make_cylinder`` / ``make_sphere`` (trimesh.hpp:12-38),
``CollisionWorld`` (collision.hpp:76-127) and the generation engine the reference leaves
unimplemented. Errors map onto the reference's exception types:
std::invalid_argument -> ValueError, std::out_of_range -> IndexError.
Poses are numpy (4, 4) float64 arrays (row, col) -- i.e. Eigen::Matrix4d semantics; they
cross the C ABI column-major, exactly the reference's memory layout.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi as A


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _up(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def colmajor(poses: np.ndarray) -> np.ndarray:
    """(..., 4, 4) row/col matrices -> contiguous column-major doubles (..., 16)."""
    p = np.asarray(poses, dtype=np.float64)
    return np.ascontiguousarray(np.swapaxes(p, -1, -2)).reshape(p.shape[:-2] + (16,))


def from_colmajor(flat: np.ndarray) -> np.ndarray:
    f = np.asarray(flat, dtype=np.float64)
    return np.swapaxes(f.reshape(f.shape[:-1] + (4, 4)), -1, -2).copy()


def translation(x: float, y: float, z: float) -> np.ndarray:
    m = np.eye(4)
    m[:3, 3] = (x, y, z)
    return m


# ---------------------------------------------------------------------------- meshes
@dataclass
class TriMesh:
    vertices: np.ndarray   # (n, 3) float64
    triangles: np.ndarray  # (m, 3) uint32

    def __post_init__(self):
        self.vertices = np.ascontiguousarray(self.vertices, dtype=np.float64).reshape(-1, 3)
        self.triangles = np.ascontiguousarray(self.triangles, dtype=np.uint32).reshape(-1, 3)

    def aabb(self):
        return self.vertices.min(axis=0), self.vertices.max(axis=0)

    def fingerprint(self) -> int:
        out = C.c_uint64()
        A.check(A.lib().sb_mesh_fingerprint(_dp(self.vertices), len(self.vertices),
                                            _up(self.triangles), len(self.triangles),
                                            C.byref(out)))
        return out.value

    def bvh_info(self) -> dict:
        info = (C.c_int32 * 4)()
        A.check(A.lib().sb_bvh_info(_dp(self.vertices), len(self.vertices), _up(self.triangles),
                                    len(self.triangles), info))
        return dict(nodes=info[0], depth=info[1], effective_nodes=info[2], reachable_tris=info[3])

    def rest_z_offset(self) -> float:
        out = C.c_double()
        A.check(A.lib().sb_rest_z_offset(_dp(self.vertices), len(self.vertices), C.byref(out)))
        return out.value


def _make(fn, *args) -> TriMesh:
    nv, nt = C.c_uint32(), C.c_uint32()
    A.check(fn(*args, None, C.byref(nv), None, C.byref(nt)))
    v = np.zeros((nv.value, 3), np.float64)
    t = np.zeros((nt.value, 3), np.uint32)
    A.check(fn(*args, _dp(v), C.byref(nv), _up(t), C.byref(nt)))
    return TriMesh(v, t)


def make_box(sx: float, sy: float, sz: float) -> TriMesh:
    """trimesh.hpp:27 -- axis-aligned box centred at the origin (12 triangles)."""
    return _make(A.lib().sb_make_box, C.c_double(sx), C.c_double(sy), C.c_double(sz))


def load_obj(path: str) -> TriMesh:
    """config.hpp:88-90 -- Wavefront OBJ subset (v / f, polygon faces fan-triangulated);
    parse errors raise with "path:line:" in the message."""
    return _make(A.lib().sb_load_obj, str(path).encode())


def make_cylinder(radius: float, height: float, segments: int = 32) -> TriMesh:
    """trimesh.hpp:30 -- capped cylinder along z (4 * segments triangles)."""
    return _make(A.lib().sb_make_cylinder, C.c_double(radius), C.c_double(height),
                 C.c_int(segments))


def make_sphere(radius: float, stacks: int = 12, slices: int = 16) -> TriMesh:
    """trimesh.hpp:32 -- UV sphere centred at the origin."""
    return _make(A.lib().sb_make_sphere, C.c_double(radius), C.c_int(stacks), C.c_int(slices))


def transformed(mesh: TriMesh, pose: np.ndarray) -> TriMesh:
    """trimesh.hpp:35 -- rigidly transformed copy (transform_point per vertex)."""
    v = mesh.vertices.copy()
    A.check(A.lib().sb_transform_vertices(_dp(colmajor(pose)), _dp(v), len(v)))
    return TriMesh(v, mesh.triangles.copy())


def merge(meshes: Sequence[TriMesh]) -> TriMesh:
    """Concatenate meshes into one TriMesh (how a sphere-set asset is built)."""
    vs, ts, off = [], [], 0
    for m in meshes:
        vs.append(m.vertices)
        ts.append(m.triangles.astype(np.uint64) + off)
        off += len(m.vertices)
    return TriMesh(np.concatenate(vs), np.concatenate(ts).astype(np.uint32))


# --------------------------------------------------------------------- collision world
class CollisionWorld:
    """collision.hpp:76-127 on the GPU. All per-instance state lives in HBM."""

    def __init__(self, batch_size: int, margin: float = 0.0, device: int = 0, _handle=None):
        self._owned = _handle is None
        if _handle is None:
            h = C.c_void_p()
            A.check(A.lib().sb_world_create(batch_size, margin, device, C.byref(h)))
            _handle = h
        self._h = _handle
        self.n = batch_size

    def close(self):
        if self._owned and self._h:
            A.lib().sb_world_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def batch_size(self) -> int:
        return self.n

    def register_geometry(self, mesh: TriMesh) -> int:
        out = C.c_int32()
        A.check(A.lib().sb_register_geometry(self._h, _dp(mesh.vertices), len(mesh.vertices),
                                             _up(mesh.triangles), len(mesh.triangles),
                                             C.byref(out)))
        return out.value

    def add_object(self, name: str, geom_id: int) -> int:
        out = C.c_int32()
        A.check(A.lib().sb_add_object(self._h, name.encode(), geom_id, C.byref(out)))
        return out.value

    def set_enabled(self, obj: int, instances: Sequence[int], enabled: bool) -> None:
        idx = np.ascontiguousarray(instances, dtype=np.uint32)
        A.check(A.lib().sb_set_enabled(self._h, obj, _up(idx), len(idx), int(bool(enabled))))

    def set_enabled_all(self, obj: int, enabled: bool) -> None:
        A.check(A.lib().sb_set_enabled_all(self._h, obj, int(bool(enabled))))

    def update_transforms(self, obj: int, poses: np.ndarray) -> None:
        p = colmajor(poses)
        if p.shape != (self.n, 16):
            raise ValueError("update_transforms: batch size mismatch")
        A.check(A.lib().sb_update_transforms(self._h, obj, _dp(p)))

    def update_transform(self, obj: int, instance: int, pose: np.ndarray) -> None:
        A.check(A.lib().sb_update_transform(self._h, obj, instance, _dp(colmajor(pose))))

    def object_pose(self, obj: int, instance: int) -> np.ndarray:
        out = np.zeros(16)
        A.check(A.lib().sb_object_pose(self._h, obj, instance, _dp(out)))
        return from_colmajor(out)

    def enabled(self, obj: int, instance: int) -> bool:
        out = C.c_int()
        A.check(A.lib().sb_enabled(self._h, obj, instance, C.byref(out)))
        return bool(out.value)

    def check_batch(self, geom_id: int, poses: np.ndarray, active: Sequence[int]):
        """Returns (free uint8[N], contact_object int32[N]) like CollisionMask."""
        act = np.ascontiguousarray(active, dtype=np.uint32)
        p = colmajor(poses).reshape(-1, 16)
        if len(p) != len(act):
            raise ValueError("check_batch: poses/active size mismatch")
        free = np.ones(self.n, np.uint8)
        contact = np.full(self.n, -1, np.int32)
        A.check(A.lib().sb_check_batch(self._h, geom_id, _dp(p), _up(act), len(act),
                                       free.ctypes.data_as(C.POINTER(C.c_uint8)),
                                       contact.ctypes.data_as(C.POINTER(C.c_int32))))
        return free, contact

    def stats(self) -> dict:
        s = A.sb_stats()
        A.check(A.lib().sb_get_stats(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in A.sb_stats._fields_}

    def reset_stats(self) -> None:
        A.check(A.lib().sb_reset_stats(self._h))


# ------------------------------------------------------------------------ scene spec
@dataclass
class Relation:
    """RelationshipSpec (relationships.hpp:18-38): anchors = [anchor] + extra_anchors
    (placement indices); `middle` takes two or more, the other distance types and a
    direction exactly one."""
    anchor: int = -1
    distance_type: int = A.SB_DIST_NONE
    direction: int = A.SB_DIR_NONE
    frame: int = A.SB_FRAME_GLOBAL
    direction_vector: tuple = (0.0, 0.0)
    distance: float = 0.0
    angle_threshold: float = 0.0   # <= 0: default
    extra_anchors: tuple = ()

    def to_c(self) -> "A.sb_relation":
        if len(self.extra_anchors) > A.SB_MAX_ANCHORS - 1:
            raise ValueError(f"at most {A.SB_MAX_ANCHORS} anchors per relation")
        extra = list(self.extra_anchors) + [-1] * (A.SB_MAX_ANCHORS - 1 - len(self.extra_anchors))
        return A.sb_relation(self.anchor, self.distance_type, self.direction, self.frame,
                             (C.c_double * 2)(*self.direction_vector), self.distance,
                             self.angle_threshold, len(self.extra_anchors),
                             (C.c_int32 * (A.SB_MAX_ANCHORS - 1))(*extra))


@dataclass
class Placement:
    mesh: int
    support: int
    orientation: int = A.SB_ORIENT_UNIFORM_YAW
    face_target: int = -1
    relation: Relation = field(default_factory=Relation)
    ratio_on_support: float = 0.0  # apply_ratio_on_support (relationships.cpp:220-230)


@dataclass
class Support:
    """A support surface (sb_support) in the z = 0 plane of its frame: `rect`, or the
    convex `polygon` ((k, 2), k <= 16; SupportSurface::polygon) when given. The frame is
    `pose`, or per instance `poses` ((N, 4, 4), e.g. FK world poses of a drawer times the
    surface frame), or -- with on_placement >= 0 -- the accepted pose of that earlier
    placement times `pose` (a surface on a placed object)."""
    pose: np.ndarray
    rect: tuple = (0.0, 0.0, 0.0, 0.0)  # x0, y0, x1, y1 in the support frame
    poses: Optional[np.ndarray] = None
    on_placement: int = -1
    polygon: Optional[np.ndarray] = None


@dataclass
class SupportSurface:
    """SupportSurface (surface.hpp:15-20): polygon in the z = 0 plane of `frame` (the
    mesh frame translated to the cluster's top), roof flag and area."""
    polygon: np.ndarray  # (k, 2)
    frame: np.ndarray    # (4, 4)
    roofed: bool
    area: float

    def support(self, object_pose=None) -> "Support":
        """A Support on this surface of a mesh placed at object_pose (default identity)."""
        pose = self.frame if object_pose is None else np.asarray(object_pose) @ self.frame
        return Support(pose, polygon=self.polygon.copy())


def _surfaces_from(arr, n) -> List["SupportSurface"]:
    out = []
    for k in range(n):
        s = arr[k]
        poly = np.array(s.polygon_xy[: 2 * s.n_polygon]).reshape(-1, 2)
        out.append(SupportSurface(poly, from_colmajor(np.array(s.frame)), bool(s.roofed), s.area))
    return out


def extract_support_surfaces(mesh: "TriMesh", mode: int = A.SB_SURFACE_ON) -> List["SupportSurface"]:
    """extract_support_surfaces / extract_all_support_surfaces (surface.cpp:53-153); mode
    SB_SURFACE_ON, SB_SURFACE_INSIDE or SB_SURFACE_ALL."""
    cap = 64
    while True:
        arr = (A.sb_surface * cap)()
        n = C.c_uint32()
        A.check(A.lib().sb_extract_support_surfaces(_dp(mesh.vertices), len(mesh.vertices),
                                                    _up(mesh.triangles), len(mesh.triangles),
                                                    mode, arr, cap, C.byref(n)))
        if n.value <= cap:
            return _surfaces_from(arr, n.value)
        cap = n.value


def support_to_c(s: "Support", keep: list) -> "A.sb_support":
    """sb_support of a Support (keep: keepalive list for the arrays it points to)."""
    out = A.sb_support()
    out.pose[:] = list(colmajor(s.pose))
    out.rect[:] = list(map(float, s.rect))
    out.on_placement = s.on_placement
    if s.polygon is not None:
        poly = np.ascontiguousarray(np.asarray(s.polygon, np.float64).reshape(-1, 2))
        keep.append(poly)
        out.n_polygon = len(poly)
        out.polygon_xy = _dp(poly)
    return out


def region_draws_host(relation: "Relation", support: "Support", states, erode_r: float,
                      seed: int, c, n: int):
    """sb_region_draws_host: region_for(0) restated on the host (the serial region path's
    code) + n sampler draws; returns ((n, 2) points, triangle count). states: (na, 3)."""
    keep = []
    sup = support_to_c(support, keep)
    rel = relation.to_c()
    st = np.ascontiguousarray(np.asarray(states, np.float64).reshape(-1))
    cc = np.ascontiguousarray(np.asarray(c, np.uint64))
    out = np.zeros((max(n, 1), 2))
    nt = C.c_int32()
    A.check(A.lib().sb_region_draws_host(C.byref(rel), C.byref(sup), _dp(st) if st.size else None,
                                         erode_r, seed,
                                         cc.ctypes.data_as(C.POINTER(C.c_uint64)), len(cc),
                                         _dp(out), n, C.byref(nt)))
    return out[:n].copy(), nt.value


@dataclass
class Fixed:
    """A fixed object: one pose, or per-instance `poses` ((N, 4, 4), a TransformBatch)."""
    mesh: int
    pose: np.ndarray
    poses: Optional[np.ndarray] = None


@dataclass
class Scene:
    name: str
    n_instances: int
    attempts: int
    meshes: List[TriMesh]
    fixed: List[Fixed]
    supports: List[Support]
    placements: List[Placement]

    def to_c(self):
        """Build the sb_scene struct; returns (struct, keepalive list)."""
        keep = []
        meshes = (A.sb_mesh * max(1, len(self.meshes)))()
        for i, m in enumerate(self.meshes):
            meshes[i] = A.sb_mesh(_dp(m.vertices), len(m.vertices), _up(m.triangles),
                                  len(m.triangles))
            keep.append(m)
        def batch(poses):
            if poses is None:
                return None
            b = colmajor(poses).reshape(-1, 16)
            if len(b) != self.n_instances:
                raise ValueError("per-instance poses must have n_instances entries")
            keep.append(b)
            return _dp(b)

        fixed = (A.sb_fixed_object * max(1, len(self.fixed)))()
        for i, f in enumerate(self.fixed):
            fixed[i].mesh = f.mesh
            fixed[i].pose[:] = list(colmajor(f.pose))
            fixed[i].poses16 = batch(f.poses)
        sups = (A.sb_support * max(1, len(self.supports)))()
        for i, s in enumerate(self.supports):
            sups[i] = support_to_c(s, keep)
            sups[i].poses16 = batch(s.poses)
        pls = (A.sb_placement * max(1, len(self.placements)))()
        for i, p in enumerate(self.placements):
            r = p.relation
            pls[i] = A.sb_placement(p.mesh, p.support, p.orientation, p.face_target, r.to_c(),
                                    p.ratio_on_support)
        sc = A.sb_scene(self.n_instances, self.attempts, 0,
                        len(self.meshes), meshes, len(self.fixed), fixed,
                        len(self.supports), sups, len(self.placements), pls)
        keep += [meshes, fixed, sups, pls]
        return sc, keep


@dataclass
class GenerationResult:
    accepted: np.ndarray   # (placements, n) int16, -1 = none
    valid: np.ndarray      # (n,) uint8
    poses: Optional[np.ndarray]  # (placements, n, 4, 4) or None
    stats: dict


class Shard:
    """Instance range [begin, end) of one rank plus the allgather used by the fast path.
    `allgather(vals) -> list` exchanges host u64 values; the optional
    `allgather_dev(send_ptr, n, recv_ptr, stream_ptr)` enqueues a device-side all-gather of
    n u64 (device pointers) on the engine's CUDA stream (e.g. NCCL), which lets FIFO
    placements chain their rounds on the device."""

    def __init__(self, begin: int, end: int, rank: int, world_size: int, allgather=None,
                 allgather_dev=None):
        self.begin, self.end, self.rank, self.world_size = begin, end, rank, world_size
        self._py = allgather
        self._pydev = allgather_dev

        def _cb(ctx, send, n, recv):
            try:
                vals = [send[i] for i in range(n)]
                out = self._py(vals)  # list of world_size * n ints
                for i, v in enumerate(out):
                    recv[i] = int(v)
                return 0
            except Exception:  # pragma: no cover - surfaced as an engine error
                import traceback
                traceback.print_exc()
                return 1

        def _cbdev(ctx, send, n, recv, stream):
            try:
                self._pydev(send, n, recv, stream)
                return 0
            except Exception:  # pragma: no cover - surfaced as an engine error
                import traceback
                traceback.print_exc()
                return 1

        self._cb = A.ALLGATHER_FN(_cb) if allgather is not None else A.ALLGATHER_FN()
        self._cbdev = A.ALLGATHER_DEV_FN(_cbdev) if allgather_dev is not None else A.ALLGATHER_DEV_FN()

    def to_c(self):
        return A.sb_shard(self.begin, self.end, self.rank, self.world_size, self._cb, None,
                          self._cbdev, None)


class Engine:
    """initialize / generate on one GPU (one shard)."""

    def __init__(self, scene: Scene, shard: Optional[Shard] = None, device: int = 0):
        self.scene = scene
        sc, self._keep = scene.to_c()
        self._shard = shard
        sh = C.byref(shard.to_c()) if shard is not None else None
        h = C.c_void_p()
        A.check(A.lib().sb_engine_create(C.byref(sc), sh, device, C.byref(h)))
        self._h = h
        self.n = A.lib().sb_engine_local_instances(h)

    def close(self):
        if self._h:
            A.lib().sb_engine_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def world(self) -> CollisionWorld:
        return CollisionWorld(self.n, _handle=A.lib().sb_engine_world(self._h))

    def generate(self, run_seed: int, with_poses: bool = True,
                 download: bool = True) -> GenerationResult:
        P = len(self.scene.placements)
        st = A.sb_run_stats()
        acc = np.empty((P, self.n), np.int16)
        valid = np.empty(self.n, np.uint8)
        poses = np.empty((P, self.n, 16), np.float64) if with_poses else None
        res = A.sb_result(acc.ctypes.data_as(C.POINTER(C.c_int16)),
                          poses.ctypes.data_as(C.POINTER(C.c_double)) if with_poses else None,
                          valid.ctypes.data_as(C.POINTER(C.c_uint8)))
        A.check(A.lib().sb_engine_generate(self._h, run_seed, C.byref(res) if download else None,
                                           C.byref(st)))
        stats = {k: getattr(st, k) for k, _ in A.sb_run_stats._fields_}
        return GenerationResult(acc, valid, from_colmajor(poses) if with_poses else None, stats)

    def place(self, run_seed: int, first: int, count: int = 1, with_poses: bool = True):
        """Placements [first, first + count) of a run (sb_engine_place): first == 0 starts
        the run, later calls continue it in order with the same seed. Returns the run's
        cumulative stats, plus the GenerationResult when the call completes the run."""
        P = len(self.scene.placements)
        st = A.sb_run_stats()
        done = first + count == P
        res, out = None, None
        if done:
            acc = np.empty((P, self.n), np.int16)
            valid = np.empty(self.n, np.uint8)
            poses = np.empty((P, self.n, 16), np.float64) if with_poses else None
            res = A.sb_result(acc.ctypes.data_as(C.POINTER(C.c_int16)),
                              poses.ctypes.data_as(C.POINTER(C.c_double)) if with_poses else None,
                              valid.ctypes.data_as(C.POINTER(C.c_uint8)))
        A.check(A.lib().sb_engine_place(self._h, run_seed, first, count,
                                        C.byref(res) if done else None, C.byref(st)))
        stats = {k: getattr(st, k) for k, _ in A.sb_run_stats._fields_}
        if done:
            out = GenerationResult(acc, valid, from_colmajor(poses) if with_poses else None, stats)
        return stats, out

    def generate_into(self, run_seed: int, res: "A.sb_result") -> dict:
        """generate + D2H into caller-owned (pinned) buffers already wrapped in sb_result."""
        st = A.sb_run_stats()
        A.check(A.lib().sb_engine_generate(self._h, run_seed, C.byref(res), C.byref(st)))
        return {k: getattr(st, k) for k, _ in A.sb_run_stats._fields_}

    def set_reach_filter(self, placement: int, reach_map, robot_base=None) -> None:
        """Fused reachability filter for `placement` (Appendix C item 8): candidates whose
        frame origin is unreachable from the instance's robot base ((N, 4, 4)) fail."""
        if reach_map is None:
            A.check(A.lib().sb_engine_set_reach_filter(self._h, placement, None, None))
            return
        b = colmajor(np.asarray(robot_base, np.float64)).reshape(-1, 16)
        self._reach_keep = getattr(self, "_reach_keep", {})
        self._reach_keep[placement] = reach_map  # the map must outlive the engine's use
        A.check(A.lib().sb_engine_set_reach_filter(self._h, placement, reach_map._h, _dp(b)))

    def write_back(self, placement: int, graph, node: int) -> None:
        """Accepted poses of `placement` from the last run into graph node `node` (a child
        of the root); instances the run left invalid are marked invalid in the graph."""
        A.check(A.lib().sb_engine_write_back(self._h, placement, graph._h, node))

    def last_timing(self):
        t, c, n = C.c_double(), C.c_double(), C.c_uint64()
        A.check(A.lib().sb_engine_last_timing(self._h, C.byref(t), C.byref(c), C.byref(n)))
        return t.value, c.value, n.value

    def phase_profile(self) -> dict:
        out = (C.c_double * 16)()
        A.check(A.lib().sb_engine_phase_profile(self._h, out))
        # block 0's device clock inside the placement kernels (see the C header)
        keys = ("init_ms", "prefix_ms", "sample_ms", "broad_narrow_ms", "accept_ms",
                "grid_sync_ms", "per_instance_ms", "fast_rounds", "regions_ms", "total_ms",
                "ev_per_instance_ms", "ev_fast_ms", "dbg_round_max_ms", "dbg_a1_max_ms",
                "dbg_a2b_max_ms")
        return dict(zip(keys, list(out)))

    def last_launches(self) -> int:
        return A.lib().sb_engine_last_launches(self._h)
