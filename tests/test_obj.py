"""CPU: load_obj (config.hpp:88-90, declared by the reference and defined here): the
Wavefront OBJ subset -- v / f records, polygon faces fan-triangulated, errors with the
line number (SPEC io_cli load_asset: "malformed mesh file -> parse error with line
number"). Host code only: no GPU needed."""
import numpy as np
import pytest


def write(tmp_path, text, name="m.obj"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def obj_text(mesh, quads=False):
    lines = ["# exported", "o box"] + [f"v {float(x)!r} {float(y)!r} {float(z)!r}" for x, y, z in mesh.vertices]
    lines += [f"vn 0 0 1", "s off"]
    lines += [f"f {a + 1}/1/1 {b + 1}//1 {c + 1}" for a, b, c in mesh.triangles]
    return "\n".join(lines) + "\n"


def test_round_trip_reference_meshes(pkg, tmp_path):
    """make_box / make_cylinder / make_sphere written as OBJ load back bit-identically
    (SPEC: box 1x1x1 -> 12 triangles; cylinder 32 segments -> 128)."""
    for mesh, nt in ((pkg.make_box(1, 1, 1), 12), (pkg.make_cylinder(0.05, 0.1, 32), 128),
                     (pkg.make_sphere(0.3, 12, 16), None)):
        got = pkg.load_obj(write(tmp_path, obj_text(mesh)))
        assert np.array_equal(got.vertices, mesh.vertices)
        assert np.array_equal(got.triangles, mesh.triangles)
        if nt is not None:
            assert len(got.triangles) == nt


def test_polygon_fan_negative_indices_and_crlf(pkg, tmp_path):
    text = ("v 0 0 0\r\nv 1 0 0\r\nv 1 1 0\r\nv 0 1 0\r\nv 0.5 1.5 0 1.0\r\n"
            "f 1 2 3 4 5\r\n"  # pentagon -> 3 fan triangles
            "f -5 -4 -3\r\n"   # relative indices = 1 2 3
            "g group\r\nusemtl m\r\nvt 0 0\r\nl 1 2\r\n")
    m = pkg.load_obj(write(tmp_path, text))
    assert m.vertices.shape == (5, 3)
    assert m.triangles.tolist() == [[0, 1, 2], [0, 2, 3], [0, 3, 4], [0, 1, 2]]


@pytest.mark.parametrize("text,line,what", [
    ("v 0 0 0\nv 1 0\n", 2, "3 coordinates"),
    ("v 0 0 0\nv 1 0 0\nv 0 1 x\n", 3, "bad coordinate"),
    ("v 0 0 0\nv 1 0 0\nv 0 1 0\n\n# c\nf 1 2 4\n", 6, "out of range"),
    ("v 0 0 0\nv 1 0 0\nf 1 2\n", 3, "at least 3"),
    ("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 0 2\n", 4, "bad face index"),
])
def test_parse_errors_carry_the_line(pkg, tmp_path, text, line, what):
    path = write(tmp_path, text)
    with pytest.raises(RuntimeError) as e:
        pkg.load_obj(path)
    assert f"{path}:{line}:" in str(e.value) and what in str(e.value)


def test_missing_file_and_no_faces(pkg, tmp_path):
    with pytest.raises(RuntimeError, match="cannot open"):
        pkg.load_obj(str(tmp_path / "absent.obj"))
    with pytest.raises(RuntimeError, match="no faces"):
        pkg.load_obj(write(tmp_path, "v 0 0 0\n"))


def test_loaded_mesh_matches_bvh_of_primitive(pkg, tmp_path):
    """A loaded mesh is the same geometry for the engine: identical fingerprint and
    effective BVH as the primitive it was written from."""
    box = pkg.make_box(0.2, 0.3, 0.4)
    got = pkg.load_obj(write(tmp_path, obj_text(box)))
    assert got.fingerprint() == box.fingerprint()
    assert got.bvh_info() == box.bvh_info()
