"""B200-native Sceniris hot path: batched candidate-pose sampling, collision checking
against placed geometry and first-valid acceptance, behind a C-ABI drop-in
(include/scenebatch_b200.h). The Python layer is a thin ctypes face used by tests and
bench.py; the product is libscenebatch_b200.so (sm_100a CUDA + C++ host runtime).
"""
from ._capi import LIB_PATH, SbCudaError, SbError, lib  # noqa: F401
from .comm import Comm, CommShard  # noqa: F401
from .graph import BatchedSceneGraph, JointSpec  # noqa: F401
from .reach import ChainLink, KinematicChain, ReachMap4D, placement_filter  # noqa: F401
from .sampler import PositionSampler, sample_orientations  # noqa: F401
from .world import (CollisionWorld, Engine, Fixed, GenerationResult, Placement, Relation,  # noqa: F401
                    Scene, Shard, Support, SupportSurface, TriMesh, colmajor,
                    extract_support_surfaces, from_colmajor, load_obj, make_box, make_cylinder,
                    make_sphere, merge, transformed, translation)


def device_available() -> bool:
    return bool(lib().sb_device_available())
