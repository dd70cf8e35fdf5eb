"""ctypes declarations for include/scenebatch_b200.h (the C-ABI drop-in).

The shared library is built in-tree by ``__graft_entry__.build()`` (paper_2512_16896_b200/
csrc/Makefile). Loading fails loudly when it is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SB_LIB_PATH", os.path.join(_HERE, "libscenebatch_b200.so"))

SB_OK = 0
SB_ERR_INVALID_ARGUMENT = 1
SB_ERR_OUT_OF_RANGE = 2
SB_ERR_LOGIC = 3
SB_ERR_RUNTIME = 4
SB_ERR_CUDA = 5

SB_DIST_NONE, SB_DIST_GREATER, SB_DIST_LESS, SB_DIST_EQUAL, SB_DIST_MIDDLE = 0, 1, 2, 3, 4
SB_MAX_ANCHORS = 8
SB_MAX_SUPPORT_VERTS = 16
SB_DIR_NONE, SB_DIR_LEFT, SB_DIR_RIGHT, SB_DIR_FRONT, SB_DIR_BACK, SB_DIR_VECTOR = range(6)
SB_FRAME_GLOBAL, SB_FRAME_LOCAL = 0, 1
SB_ORIENT_FIXED, SB_ORIENT_UNIFORM_YAW, SB_ORIENT_FACE_TO = 0, 1, 2


class sb_stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "geometry_registrations", "bvh_builds", "check_calls", "checked_instances",
        "narrow_phase_tests", "triangle_pair_tests")]


class sb_mesh(C.Structure):
    _fields_ = [("vertices", C.POINTER(C.c_double)), ("n_vertices", C.c_uint32),
                ("triangles", C.POINTER(C.c_uint32)), ("n_triangles", C.c_uint32)]


class sb_fixed_object(C.Structure):
    _fields_ = [("mesh", C.c_int32), ("pose", C.c_double * 16), ("poses16", C.POINTER(C.c_double))]


class sb_support(C.Structure):
    _fields_ = [("pose", C.c_double * 16), ("rect", C.c_double * 4),
                ("poses16", C.POINTER(C.c_double)), ("on_placement", C.c_int32),
                ("n_polygon", C.c_uint32), ("polygon_xy", C.POINTER(C.c_double))]


SB_SURFACE_ON, SB_SURFACE_INSIDE, SB_SURFACE_ALL = 0, 1, -1
SB_MAX_SURFACE_VERTS = 96


class sb_surface(C.Structure):
    _fields_ = [("frame", C.c_double * 16), ("area", C.c_double), ("roofed", C.c_int32),
                ("n_polygon", C.c_uint32), ("polygon_xy", C.c_double * (2 * SB_MAX_SURFACE_VERTS))]


class sb_joint(C.Structure):
    _fields_ = [("kind", C.c_int32), ("axis", C.c_double * 3), ("lo", C.c_double),
                ("hi", C.c_double)]


class sb_chain_link(C.Structure):
    _fields_ = [("origin", C.c_double * 16), ("joint", sb_joint)]


class sb_reach_info(C.Structure):
    _fields_ = [("samples", C.c_uint64), ("resolution", C.c_double),
                ("psi_resolution", C.c_double), ("max_radius", C.c_double),
                ("z_min", C.c_double), ("z_max", C.c_double), ("nr", C.c_uint64),
                ("nz", C.c_uint64), ("npsi", C.c_uint64), ("cell_count", C.c_uint64),
                ("occupied_cells", C.c_uint64)]


class sb_relation(C.Structure):
    _fields_ = [("anchor", C.c_int32), ("distance_type", C.c_int32), ("direction", C.c_int32),
                ("frame", C.c_int32), ("direction_vector", C.c_double * 2),
                ("distance", C.c_double), ("angle_threshold", C.c_double),
                ("n_extra_anchors", C.c_int32), ("extra_anchors", C.c_int32 * (SB_MAX_ANCHORS - 1))]


class sb_placement(C.Structure):
    _fields_ = [("mesh", C.c_int32), ("support", C.c_int32), ("orientation", C.c_int32),
                ("face_target", C.c_int32), ("relation", sb_relation),
                ("ratio_on_support", C.c_double)]


class sb_scene(C.Structure):
    _fields_ = [("n_instances", C.c_uint64), ("attempts", C.c_int32), ("reserved", C.c_int32),
                ("n_meshes", C.c_uint32), ("meshes", C.POINTER(sb_mesh)),
                ("n_fixed", C.c_uint32), ("fixed", C.POINTER(sb_fixed_object)),
                ("n_supports", C.c_uint32), ("supports", C.POINTER(sb_support)),
                ("n_placements", C.c_uint32), ("placements", C.POINTER(sb_placement))]


class sb_result(C.Structure):
    _fields_ = [("accepted", C.POINTER(C.c_int16)), ("poses", C.POINTER(C.c_double)),
                ("valid", C.POINTER(C.c_uint8))]


class sb_run_stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "valid_instances", "candidates_sampled", "candidate_checks", "narrow_phase_tests",
        "triangle_pair_tests", "rounds", "per_instance_placements", "broad_phase_tests",
        "node_pair_tests", "accepted_candidates")]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_uint32,
                           C.POINTER(C.c_uint64))


# (ctx, d_send, n, d_recv, cuda_stream) -> status: device-side all-gather
ALLGATHER_DEV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p,
                               C.c_void_p)


class sb_shard(C.Structure):
    _fields_ = [("begin", C.c_uint64), ("end", C.c_uint64), ("rank", C.c_int32),
                ("world_size", C.c_int32), ("allgather", ALLGATHER_FN), ("ctx", C.c_void_p),
                ("allgather_dev", ALLGATHER_DEV_FN), ("ctx_dev", C.c_void_p)]


# Every symbol the header declares, with (restype, argtypes).
_P = C.c_void_p
_D = C.POINTER(C.c_double)
_U32 = C.POINTER(C.c_uint32)
SIGNATURES = {
    "sb_last_error": (C.c_char_p, []),
    "sb_abi_version": (C.c_int, []),
    "sb_device_available": (C.c_int, []),
    "sb_make_box": (C.c_int, [C.c_double, C.c_double, C.c_double, _D, _U32, _U32, _U32]),
    "sb_load_obj": (C.c_int, [C.c_char_p, _D, _U32, _U32, _U32]),
    "sb_make_cylinder": (C.c_int, [C.c_double, C.c_double, C.c_int, _D, _U32, _U32, _U32]),
    "sb_make_sphere": (C.c_int, [C.c_double, C.c_int, C.c_int, _D, _U32, _U32, _U32]),
    "sb_transform_vertices": (C.c_int, [_D, _D, C.c_uint32]),
    "sb_mesh_fingerprint": (C.c_int, [_D, C.c_uint32, _U32, C.c_uint32, C.POINTER(C.c_uint64)]),
    "sb_rest_z_offset": (C.c_int, [_D, C.c_uint32, _D]),
    "sb_bvh_info": (C.c_int, [_D, C.c_uint32, _U32, C.c_uint32, C.POINTER(C.c_int32)]),
    "sb_triangulate_ring": (C.c_int, [_D, C.c_uint32, _D, C.c_uint32, _U32]),
    "sb_mix64": (C.c_uint64, [C.c_uint64]),
    "sb_stream_key": (C.c_uint64, [C.POINTER(C.c_uint64), C.c_uint32]),
    "sb_stream_doubles": (C.c_int, [C.c_uint64, C.POINTER(C.c_uint64), C.c_uint32, _D, C.c_uint32]),
    "sb_world_create": (C.c_int, [C.c_uint64, C.c_double, C.c_int, C.POINTER(_P)]),
    "sb_world_destroy": (None, [_P]),
    "sb_register_geometry": (C.c_int, [_P, _D, C.c_uint32, _U32, C.c_uint32, C.POINTER(C.c_int32)]),
    "sb_add_object": (C.c_int, [_P, C.c_char_p, C.c_int32, C.POINTER(C.c_int32)]),
    "sb_set_enabled": (C.c_int, [_P, C.c_int32, _U32, C.c_uint64, C.c_int]),
    "sb_set_enabled_all": (C.c_int, [_P, C.c_int32, C.c_int]),
    "sb_update_transforms": (C.c_int, [_P, C.c_int32, _D]),
    "sb_update_transform": (C.c_int, [_P, C.c_int32, C.c_uint64, _D]),
    "sb_object_pose": (C.c_int, [_P, C.c_int32, C.c_uint64, _D]),
    "sb_enabled": (C.c_int, [_P, C.c_int32, C.c_uint64, C.POINTER(C.c_int)]),
    "sb_check_batch": (C.c_int, [_P, C.c_int32, _D, _U32, C.c_uint64, C.POINTER(C.c_uint8),
                                 C.POINTER(C.c_int32)]),
    "sb_get_stats": (C.c_int, [_P, C.POINTER(sb_stats)]),
    "sb_reset_stats": (C.c_int, [_P]),
    "sb_extract_support_surfaces": (C.c_int, [_D, C.c_uint32, _U32, C.c_uint32, C.c_int32,
                                              C.POINTER(sb_surface), C.c_uint32, _U32]),
    "sb_region_draws_host": (C.c_int, [C.POINTER(sb_relation), C.POINTER(sb_support), _D, C.c_double,
                                       C.c_uint64, C.POINTER(C.c_uint64), C.c_uint32, _D, C.c_uint32,
                                       C.POINTER(C.c_int32)]),
    "sb_comm_create": (C.c_int, [C.c_int32, C.c_int32, C.c_int, C.c_char_p, C.c_int32, C.c_double,
                                 C.POINTER(_P)]),
    "sb_comm_destroy": (None, [_P]),
    "sb_comm_shard": (C.c_int, [_P, C.c_uint64, C.POINTER(sb_shard)]),
    "sb_comm_allgather": (C.c_int, [_P, C.POINTER(C.c_uint64), C.c_uint32, C.POINTER(C.c_uint64)]),
    "sb_comm_allgather_dev": (C.c_int, [_P, _P, C.c_uint32, _P, _P]),
    "sb_comm_barrier": (C.c_int, [_P]),
    "sb_comm_uses_stream_waits": (C.c_int32, [_P]),
    "sb_engine_create": (C.c_int, [C.POINTER(sb_scene), C.POINTER(sb_shard), C.c_int, C.POINTER(_P)]),
    "sb_engine_destroy": (None, [_P]),
    "sb_engine_generate": (C.c_int, [_P, C.c_uint64, C.POINTER(sb_result), C.POINTER(sb_run_stats)]),
    "sb_engine_download": (C.c_int, [_P, C.POINTER(sb_result)]),
    "sb_engine_place": (C.c_int, [_P, C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(sb_result),
                                  C.POINTER(sb_run_stats)]),
    "sb_engine_world": (_P, [_P]),
    "sb_engine_local_instances": (C.c_uint64, [_P]),
    "sb_engine_last_launches": (C.c_uint64, [_P]),
    "sb_engine_last_timing": (C.c_int, [_P, _D, _D, C.POINTER(C.c_uint64)]),
    "sb_engine_phase_profile": (C.c_int, [_P, _D]),
    "sb_debug_region_profile": (C.c_int, [C.POINTER(C.c_uint64)]),
    "sb_device_math": (C.c_int, [C.c_int, _D, C.c_uint64, _D]),
    "sb_host_math": (C.c_int, [C.c_int, _D, C.c_uint64, _D]),
    "sb_debug_narrow_profile": (C.c_int, [C.POINTER(C.c_uint64)]),
    "sb_sampler_create": (C.c_int, [C.c_uint64, C.c_int, C.POINTER(_P)]),
    "sb_sampler_destroy": (None, [_P]),
    "sb_sampler_prepare": (C.c_int, [_P, _D, _U32, C.c_uint32, _U32, C.c_uint64, C.c_uint64]),
    "sb_sampler_sample": (C.c_int, [_P, _D, _U32, C.c_uint64, C.c_uint64, _D,
                                    C.POINTER(C.c_uint8)]),
    "sb_sampler_prepare_relation": (C.c_int, [_P, C.POINTER(sb_relation), _D, _D, C.c_uint64,
                                              C.c_uint64]),
    "sb_graph_create": (C.c_int, [C.c_uint64, C.c_int, C.POINTER(_P)]),
    "sb_graph_destroy": (None, [_P]),
    "sb_graph_add_node": (C.c_int, [_P, C.c_uint32, C.c_char_p, C.c_int64, C.POINTER(sb_joint),
                                    C.POINTER(C.c_uint32)]),
    "sb_graph_set_edge_batch": (C.c_int, [_P, C.c_uint32, C.c_uint32, _D]),
    "sb_graph_set_edge": (C.c_int, [_P, C.c_uint32, C.c_uint64, _D]),
    "sb_graph_edge_batch": (C.c_int, [_P, C.c_uint32, _D]),
    "sb_graph_set_joint_states": (C.c_int, [_P, C.c_uint32, _D]),
    "sb_graph_joint_states": (C.c_int, [_P, C.c_uint32, _D]),
    "sb_graph_world_poses": (C.c_int, [_P, C.c_uint32, _D]),
    "sb_graph_world_pose": (C.c_int, [_P, C.c_uint32, C.c_uint64, _D]),
    "sb_graph_find": (C.c_int, [_P, C.c_char_p, C.POINTER(C.c_int64)]),
    "sb_graph_node_info": (C.c_int, [_P, C.c_uint32, C.POINTER(C.c_char_p), C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_int64), C.POINTER(C.c_int), C.POINTER(sb_joint)]),
    "sb_graph_node_count": (C.c_uint64, [_P]),
    "sb_graph_children": (C.c_int, [_P, C.c_uint32, _U32, C.c_uint32, C.POINTER(C.c_uint32)]),
    "sb_graph_is_tree": (C.c_int, [_P, C.POINTER(C.c_int)]),
    "sb_graph_valid_mask": (C.c_int, [_P, C.POINTER(C.c_uint8)]),
    "sb_graph_mark_invalid": (C.c_int, [_P, C.c_uint64]),
    "sb_graph_reset_validity": (C.c_int, [_P]),
    "sb_graph_valid_count": (C.c_int, [_P, C.POINTER(C.c_uint64)]),
    "sb_engine_write_back": (C.c_int, [_P, C.c_uint32, _P, C.c_uint32]),
    "sb_reach_build": (C.c_int, [C.POINTER(sb_chain_link), C.c_uint32, _D, C.c_uint64, C.c_double,
                                 C.c_double, C.c_uint64, C.c_int, C.POINTER(_P)]),
    "sb_reach_load": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(_P)]),
    "sb_reach_save": (C.c_int, [_P, C.c_char_p]),
    "sb_reach_destroy": (None, [_P]),
    "sb_reach_get_info": (C.c_int, [_P, C.POINTER(sb_reach_info)]),
    "sb_reach_cell_samples": (C.c_int, [_P, C.c_uint64, C.c_uint64, C.c_uint64,
                                        C.POINTER(C.c_uint32)]),
    "sb_reach_query_batch": (C.c_int, [_P, _D, _D, C.c_uint64, C.c_int, C.c_double,
                                       C.POINTER(C.c_uint8)]),
    "sb_reach_placement_filter": (C.c_int, [_P, _D, C.c_uint64, C.POINTER(_D), C.c_uint32, _U32,
                                            C.c_uint64, C.POINTER(C.c_uint8)]),
    "sb_engine_set_reach_filter": (C.c_int, [_P, C.c_uint32, _P, _D]),
    "sb_sampler_sample_device": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_uint64, _P, _P, _P]),
    "sb_graph_world_poses_device": (C.c_int, [_P, C.c_uint32, _P, _P]),
    "sb_reach_query_batch_device": (C.c_int, [_P, _P, _P, C.c_uint64, C.c_int, C.c_double, _P,
                                              _P]),
    "sb_sample_orientations_device": (C.c_int, [C.c_int, _P, C.c_uint64, _P, _P, C.c_uint64,
                                                C.c_uint64, C.c_uint64, _P, _P]),
    "sb_sampler_cache_info": (C.c_int, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "sb_sample_orientations": (C.c_int, [C.c_int, _U32, C.c_uint64, _D, _D, C.c_uint64,
                                         C.c_uint64, C.c_uint64, C.c_uint64, _D, C.c_int]),
}

_lib = None


def lib() -> C.CDLL:
    """Load the in-tree C-ABI library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class SbError(RuntimeError):
    """Base class; subclasses mirror the reference's exception types."""


class SbCudaError(SbError):
    pass


def check(status: int) -> None:
    if status == SB_OK:
        return
    msg = lib().sb_last_error().decode(errors="replace")
    if status == SB_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if status == SB_ERR_OUT_OF_RANGE:
        raise IndexError(msg)  # std::out_of_range
    if status == SB_ERR_CUDA:
        raise SbCudaError(msg)
    raise SbError(msg)  # std::logic_error / std::runtime_error
