"""Synthetic scenes of the shapes BASELINE.json names (configs C1..C5).

There is no network and the reference ships no assets, so every scene is generated from
a fixed seed: object sizes come from the reference's own PCG32 (rng.hpp:24-60) seeded
with ``config_seed`` and are identical across variations. Meshes are built through the
C ABI's primitives (bit-identical to trimesh.cpp), so the reference oracle and the GPU
engine consume byte-identical inputs. ``mesh_source`` swaps the primitive constructors
(bench.py's reference arm builds the same scenes with the reference's own make_box /
make_cylinder / make_sphere, so that process never maps this package's library).
"""
from __future__ import annotations

import contextlib
import math
from typing import List

import numpy as np

from . import _capi as A
from . import world as _world
from .world import Fixed, Placement, Relation, Scene, Support, TriMesh, merge, translation

def _extract(mesh: TriMesh, mode: int):
    """(polygon (k, 2), frame (4, 4)) of each support surface (sb_extract_support_surfaces)."""
    return [(s.polygon, s.frame) for s in _world.extract_support_surfaces(mesh, mode)]


_PRIMS = {"make_box": _world.make_box, "make_cylinder": _world.make_cylinder,
          "make_sphere": _world.make_sphere, "transformed": _world.transformed,
          "extract_support_surfaces": _extract}


@contextlib.contextmanager
def mesh_source(**prims):
    """Temporarily build scenes with other primitive constructors (same signatures as
    world.make_box / make_cylinder / make_sphere / transformed, and
    extract_support_surfaces(mesh, mode) -> [(polygon, frame)])."""
    old = dict(_PRIMS)
    _PRIMS.update(prims)
    try:
        yield
    finally:
        _PRIMS.update(old)


def make_box(sx, sy, sz) -> TriMesh:
    return _PRIMS["make_box"](sx, sy, sz)


def make_cylinder(radius, height, segments=32) -> TriMesh:
    return _PRIMS["make_cylinder"](radius, height, segments)


def make_sphere(radius, stacks=12, slices=16) -> TriMesh:
    return _PRIMS["make_sphere"](radius, stacks, slices)


def transformed(mesh: TriMesh, pose) -> TriMesh:
    return _PRIMS["transformed"](mesh, pose)

M64 = (1 << 64) - 1


class Pcg32:
    """rng.hpp:24-60, used host-side for scene parameters only."""

    def __init__(self, seed: int, seq: int = 0xDA3E39CB94B95BDB):
        self.state = 0
        self.inc = ((seq << 1) | 1) & M64
        self.next_u32()
        self.state = (self.state + seed) & M64
        self.next_u32()

    def next_u32(self) -> int:
        old = self.state
        self.state = (old * 6364136223846793005 + self.inc) & M64
        xs = (((old >> 18) ^ old) >> 27) & 0xFFFFFFFF
        rot = old >> 59
        return ((xs >> rot) | (xs << ((32 - rot) & 31))) & 0xFFFFFFFF

    def next_double(self) -> float:
        hi = self.next_u32()
        lo = self.next_u32()
        return float(((hi << 32) | lo) >> 11) * 2.0 ** -53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_double()


def sphere_set(rng: Pcg32, n_spheres: int = 32, radius: float = 0.012) -> TriMesh:
    """32 x make_sphere(0.012, 4, 6) at U[+-0.03]^2 x U[0, 0.05], merged."""
    base = make_sphere(radius, 4, 6)
    parts = []
    for _ in range(n_spheres):
        off = (rng.uniform(-0.03, 0.03), rng.uniform(-0.03, 0.03), rng.uniform(0.0, 0.05))
        parts.append(transformed(base, translation(*off)))
    return merge(parts)


def _box(rng: Pcg32, lo=0.04, hi=0.12) -> TriMesh:
    return make_box(rng.uniform(lo, hi), rng.uniform(lo, hi), rng.uniform(lo, hi))


def _table(sx: float, sy: float, h: float = 0.75, at=(0.0, 0.0)):
    mesh = make_box(sx, sy, h)
    pose = translation(at[0], at[1], h / 2)
    sup = Support(translation(at[0], at[1], h), (-sx / 2, -sy / 2, sx / 2, sy / 2))
    return mesh, pose, sup


_DIRS = [A.SB_DIR_LEFT, A.SB_DIR_RIGHT, A.SB_DIR_FRONT, A.SB_DIR_BACK]


def next_to(anchor: int, k: int) -> Relation:
    return Relation(anchor=anchor, distance_type=A.SB_DIST_LESS, direction=_DIRS[k % 4],
                    distance=0.25, angle_threshold=math.pi / 4)


def tabletop_boxes(n_instances=1024, n_objects=10, attempts=64, config_seed=7,
                   table=(1.2, 0.8)) -> Scene:
    """C1: 1 table support, `n_objects` cuboids U[.04,.12]^3, uniform yaw."""
    rng = Pcg32(config_seed)
    tmesh, tpose, sup = _table(*table)
    meshes = [tmesh]
    places = []
    for _ in range(n_objects):
        meshes.append(_box(rng))
        places.append(Placement(mesh=len(meshes) - 1, support=0))
    return Scene(f"tabletop{n_objects}x{n_instances}", n_instances, attempts, meshes,
                 [Fixed(0, tpose)], [sup], places)


def tabletop_mixed(n_instances=16384, n_objects=25, attempts=64, config_seed=11,
                   table=(1.6, 1.0)) -> Scene:
    """C2: cuboids and 32-sphere sets; every third object is next-to the previous one
    (1 anchor, direction cycling left/right/front/back, less, d=0.25, theta=pi/4)."""
    rng = Pcg32(config_seed)
    tmesh, tpose, sup = _table(*table)
    meshes = [tmesh]
    places = []
    for k in range(n_objects):
        meshes.append(_box(rng) if k % 2 == 0 else sphere_set(rng))
        rel = next_to(k - 1, k // 3) if k % 3 == 2 else Relation()
        places.append(Placement(mesh=len(meshes) - 1, support=0, relation=rel))
    return Scene(f"mixed{n_objects}x{n_instances}", n_instances, attempts, meshes,
                 [Fixed(0, tpose)], [sup], places)


def open_container(sx=0.6, sy=0.5, sz=0.3, wall=0.02) -> TriMesh:
    """Open-top bin: floor slab + 4 walls merged into one mesh (frame origin at its base)."""
    parts = [transformed(make_box(sx, sy, wall), translation(0, 0, wall / 2))]
    for s in (-1, 1):
        parts.append(transformed(make_box(wall, sy, sz), translation(s * (sx - wall) / 2, 0, sz / 2)))
        parts.append(transformed(make_box(sx - 2 * wall, wall, sz),
                                 translation(0, s * (sy - wall) / 2, sz / 2)))
    return merge(parts)


def surface_support(mesh: TriMesh, pose, mode: int = A.SB_SURFACE_ON, k: int = 0) -> Support:
    """The k-th largest support surface of `mesh` placed at `pose`
    (extract_support_surfaces, surface.cpp:145-153) as a polygon Support."""
    polygon, frame = _PRIMS["extract_support_surfaces"](mesh, mode)[k]
    return Support(np.asarray(pose) @ np.asarray(frame), polygon=np.asarray(polygon))


def kitchen(n_instances=65536, n_objects=50, attempts=256, config_seed=23) -> Scene:
    """C3: counter + table + the floor of an open container, all three supports extracted
    from the fixed meshes (extract_support_surfaces, mode `on`: the bin is open to the sky,
    so its floor is not roofed); boxes, cylinders and sphere sets; every 7th object is
    next-to the previous object on its support."""
    rng = Pcg32(config_seed)
    counter, cpose, _ = _table(2.0, 0.7, 0.9, at=(0.0, 0.0))
    table, tpose, _ = _table(1.2, 1.2, 0.75, at=(0.0, 1.6))
    bin_mesh = open_container()
    bin_pose = translation(-1.8, 0.0, 0.0)
    csup = surface_support(counter, cpose)
    tsup = surface_support(table, tpose)
    bsup = surface_support(bin_mesh, bin_pose)  # the floor slab's top (largest area)
    meshes = [counter, table, bin_mesh]
    fixed = [Fixed(0, cpose), Fixed(1, tpose), Fixed(2, bin_pose)]
    supports = [csup, tsup, bsup]
    places: List[Placement] = []
    last_on = {}
    for k in range(n_objects):
        s = (0, 0, 1, 1, 2)[k % 5]
        kind = k % 3
        if s == 2:
            m = _box(rng, 0.03, 0.08) if kind != 1 else make_cylinder(
                rng.uniform(0.015, 0.04), rng.uniform(0.03, 0.1), 16)
        elif kind == 0:
            m = _box(rng)
        elif kind == 1:
            m = make_cylinder(rng.uniform(0.02, 0.05), rng.uniform(0.04, 0.15), 16)
        else:
            m = sphere_set(rng)
        meshes.append(m)
        rel = Relation()
        if k % 7 == 6 and s in last_on:
            rel = next_to(last_on[s], k // 7)
        places.append(Placement(mesh=len(meshes) - 1, support=s, relation=rel))
        last_on[s] = k
    return Scene(f"kitchen{n_objects}x{n_instances}", n_instances, attempts, meshes, fixed,
                 supports, places)


def dense_clutter(n_instances=262144, n_objects=100, attempts=64, config_seed=31) -> Scene:
    """C4: 100 sphere-set objects on one table sized 0.03 m^2 per object."""
    rng = Pcg32(config_seed)
    area = 0.03 * n_objects
    sx = math.sqrt(area * 4.0 / 3.0)
    sy = area / sx
    tmesh, tpose, sup = _table(sx, sy)
    meshes = [tmesh]
    places = []
    for _ in range(n_objects):
        meshes.append(sphere_set(rng))
        places.append(Placement(mesh=len(meshes) - 1, support=0))
    return Scene(f"clutter{n_objects}x{n_instances}", n_instances, attempts, meshes,
                 [Fixed(0, tpose)], [sup], places)


def scale_sweep(n_instances: int, n_objects: int, attempts=64, config_seed=43) -> Scene:
    """C5: cuboids on a table sized 0.04 m^2 per object."""
    area = 0.04 * n_objects
    sx = math.sqrt(area * 4.0 / 3.0)
    return tabletop_boxes(n_instances, n_objects, attempts, config_seed, table=(sx, area / sx))


CONFIGS = {
    "c1_tabletop": lambda n=1024: tabletop_boxes(n),
    "c2_mixed": lambda n=16384: tabletop_mixed(n),
    "c3_kitchen": lambda n=65536: kitchen(n),
    "c4_clutter": lambda n=262144: dense_clutter(n),
    "c5_sweep": lambda n=1 << 20, objects=100: scale_sweep(n, objects),
}
