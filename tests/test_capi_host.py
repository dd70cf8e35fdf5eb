"""CPU: the C-ABI library loads, exports every symbol include/*.h declares, and its
host-side preparation (meshes, fingerprints, RNG, BVH export) matches the reference.
No compute entry point is called here (there is no GPU in this container)."""
import os
import re

import numpy as np
import pytest

import paper_2512_16896_b200 as pkg
from paper_2512_16896_b200 import _capi as A
from paper_2512_16896_b200 import scenes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            text = open(os.path.join(ROOT, "include", fn)).read()
            text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
            names |= set(re.findall(r"\b(sb_[a-z0-9_]+)\s*\(", text))
    return names - {"sb_allgather_fn"}


def test_library_exports_every_declared_symbol():
    L = pkg.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(L, s), s
    assert set(A.SIGNATURES) >= syms  # every symbol is bound with a signature
    assert L.sb_abi_version() == 2


def test_no_device_fails_loudly():
    if pkg.device_available():
        pytest.skip("a device is present")
    with pytest.raises(A.SbCudaError):
        pkg.CollisionWorld(4)


def test_meshes_match_reference(ref):
    for args in [(1, 1, 1), (0.31, 0.2, 0.07)]:
        m = pkg.make_box(*args)
        v, t = ref.make_box(*args)
        assert np.array_equal(m.vertices, v) and np.array_equal(m.triangles, t)
    for args in [(0.012, 4, 6), (1.0, 12, 16), (0.3, 5, 7)]:
        m = pkg.make_sphere(*args)
        v, t = ref.make_sphere(*args)
        assert np.array_equal(m.vertices, v) and np.array_equal(m.triangles, t)
    m = pkg.make_cylinder(0.05, 0.1, 32)
    v, t = ref.make_cylinder(0.05, 0.1, 32)
    assert np.array_equal(m.vertices, v) and np.array_equal(m.triangles, t)
    ss = scenes.sphere_set(scenes.Pcg32(3))
    assert ss.fingerprint() == ref.lib().ref_mesh_fingerprint(
        ss.vertices.ctypes.data, len(ss.vertices), ss.triangles.ctypes.data, len(ss.triangles))


def test_rng_matches_reference(ref):
    import ctypes as C

    for seed, counters in [(7, [1, 2, 3]), (31, [9, 0x79617721, 1, 7]), (1, [3, 0x63616368])]:
        c = np.array(counters, np.uint64)
        out = np.zeros(64)
        A.check(pkg.lib().sb_stream_doubles(seed, c.ctypes.data_as(C.POINTER(C.c_uint64)),
                                            len(c), out.ctypes.data_as(C.POINTER(C.c_double)),
                                            64))
        assert np.array_equal(out, ref.stream_doubles(seed, counters, 64))
    assert pkg.lib().sb_mix64(0) == ref.lib().ref_mix64(0)
    p = (C.c_uint64 * 2)(1, 2)
    assert pkg.lib().sb_stream_key(p, 2) == 0xE39317DCDF18B70D


def test_scene_pcg_matches_reference(ref):
    r = scenes.Pcg32(12345)
    hi, lo = r.next_u32(), r.next_u32()
    assert (hi << 32) | lo == 0x8630B53A16AC2A2C


def test_effective_bvh_reachable_sets():
    """reachable triangles under the reference's child indexing."""
    assert pkg.make_box(1, 1, 1).bvh_info() == dict(nodes=7, depth=3, effective_nodes=4,
                                                    reachable_tris=6)
    assert pkg.make_cylinder(0.05, 0.1, 32).bvh_info()["reachable_tris"] == 8
    assert pkg.make_sphere(1.0, 12, 16).bvh_info()["reachable_tris"] == 5
    assert pkg.make_sphere(0.012, 4, 6).bvh_info()["reachable_tris"] == 9
    info = scenes.sphere_set(scenes.Pcg32(1)).bvh_info()
    assert info["reachable_tris"] == 9 and info["effective_nodes"] <= 32


def test_rest_offset():
    m = pkg.make_box(0.2, 0.2, 0.3)
    assert m.rest_z_offset() == 0.15 + 1e-3


def _product_triangulate(ring):
    import ctypes as C

    r = np.ascontiguousarray(ring, np.float64).reshape(-1, 2)
    out = np.zeros((256, 6))
    nt = C.c_uint32()
    A.check(pkg.lib().sb_triangulate_ring(r.ctypes.data_as(C.POINTER(C.c_double)), len(r),
                                          out.ctypes.data_as(C.POINTER(C.c_double)), 256,
                                          C.byref(nt)))
    return out[: nt.value].reshape(-1, 3, 2)


def _area2(t):
    return (t[:, 1, 0] - t[:, 0, 0]) * (t[:, 2, 1] - t[:, 0, 1]) - \
        (t[:, 1, 1] - t[:, 0, 1]) * (t[:, 2, 0] - t[:, 0, 0])


@pytest.mark.parametrize("seed", range(6))
def test_triangulation_matches_reference(ref, seed):
    """Ear clipping (polygon.cpp:260-340): the exact fan fast path for convex rings and the
    general path for star-shaped (reflex) rings reproduce the reference triangle by
    triangle, in order."""
    rng = np.random.default_rng(seed)
    rings = []
    for _ in range(40):
        n = int(rng.integers(3, 40))
        ang = np.sort(rng.uniform(0, 2 * np.pi, n))
        convex = rng.random() < 0.5
        rad = np.ones(n) if convex else rng.uniform(0.3, 1.0, n)
        ring = np.stack([rad * np.cos(ang), rad * np.sin(ang)], 1) * rng.uniform(0.05, 2.0)
        ring += rng.uniform(-1, 1, 2)
        if rng.random() < 0.3:
            ring = ring[::-1]  # clockwise input: triangulate reverses it
        rings.append(ring)
    rings.append(np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float))
    for ring in rings:
        want = ref.triangulate(ring)
        want = want[np.abs(_area2(want)) > 0]
        got = _product_triangulate(ring)
        assert np.array_equal(got, want)
