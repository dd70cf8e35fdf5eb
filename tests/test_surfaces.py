"""Support-surface extraction (surface.cpp:53-153) on CPU: the
product's host restatement (sb_extract_support_surfaces) against the reference's own
extract_support_surfaces (oracle/_ref, union_of through the Boost stand-in of
oracle/shim) -- polygons, frames, roof flags and areas bit for bit -- on primitives, an
open container, a roofed cabinet, merged scenes and sphere sets."""
import numpy as np
import pytest

from paper_2512_16896_b200 import _capi as A
from paper_2512_16896_b200 import scenes
from paper_2512_16896_b200.world import (colmajor, extract_support_surfaces, make_box,
                                         make_cylinder, make_sphere, merge, transformed,
                                         translation)


def cabinet(sx=0.8, sy=0.5, sz=0.9, wall=0.03):
    """Bottom, top and two side slabs: the floor between them is roofed."""
    parts = [transformed(make_box(sx, sy, wall), translation(0, 0, wall / 2)),
             transformed(make_box(sx, sy, wall), translation(0, 0, sz - wall / 2)),
             transformed(make_box(wall, sy, sz), translation(-sx / 2 + wall / 2, 0, sz / 2)),
             transformed(make_box(wall, sy, sz), translation(sx / 2 - wall / 2, 0, sz / 2))]
    return merge(parts)


MESHES = {
    "box": lambda: make_box(0.6, 0.4, 0.3),
    "cylinder": lambda: make_cylinder(0.2, 0.3, 24),
    "sphere": lambda: make_sphere(0.15, 12, 16),
    "container": lambda: scenes.open_container(),
    "cabinet": cabinet,
    "table_and_container": lambda: merge([make_box(1.2, 0.8, 0.75),
                                          transformed(scenes.open_container(0.3, 0.25, 0.15, 0.01),
                                                      translation(0.2, 0.1, 0.45))]),
    "sphere_set": lambda: scenes.sphere_set(scenes.Pcg32(5)),
    "tilted_box": lambda: transformed(make_box(0.5, 0.3, 0.2),
                                      np.array([[1, 0, 0, 0], [0, np.cos(0.05), -np.sin(0.05), 0],
                                                [0, np.sin(0.05), np.cos(0.05), 0], [0, 0, 0, 1.0]])),
}


@pytest.mark.parametrize("name", sorted(MESHES))
@pytest.mark.parametrize("mode", [A.SB_SURFACE_ON, A.SB_SURFACE_INSIDE, A.SB_SURFACE_ALL])
def test_surfaces_match_reference(ref, name, mode):
    m = MESHES[name]()
    got = extract_support_surfaces(m, mode)
    want = ref.extract_support_surfaces(m.vertices, m.triangles, mode)
    assert len(got) == len(want)
    for g, (poly, frame, roofed, area) in zip(got, want):
        assert np.array_equal(g.polygon, poly), name
        assert np.array_equal(colmajor(g.frame), frame), name
        assert g.roofed == roofed and g.area == area, name


def test_surface_flags():
    ins = extract_support_surfaces(cabinet(), A.SB_SURFACE_INSIDE)
    assert len(ins) == 1 and ins[0].roofed  # the floor under the top slab
    top = extract_support_surfaces(make_box(0.6, 0.4, 0.3), A.SB_SURFACE_ON)
    assert len(top) == 1 and abs(top[0].area - 0.24) < 1e-12 and top[0].frame[2, 3] == 0.15
    assert len(top[0].polygon) == 4
