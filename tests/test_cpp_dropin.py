"""The C++ face (include/scenebatch_b200.hpp) compiles against the C ABI and runs the
reference's CollisionWorld call sequence (SPEC.md:394-395 unit cubes)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2512_16896_b200")


def build(tmp_path):
    exe = str(tmp_path / "cpp_dropin")
    subprocess.run(["g++", "-std=c++20", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "cpp_dropin.cpp"), "-L", LIBDIR,
                    "-lscenebatch_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cpp_header_builds_and_fails_loudly_without_gpu(tmp_path, pkg):
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert "fingerprint ed59e5f2fc2480f9" in r.stdout
    if not pkg.device_available():
        assert r.returncode == 2 and "no CUDA device" in r.stdout


@pytest.mark.gpu
def test_cpp_header_unit_cubes_on_gpu(tmp_path, gpu, ref):
    r = subprocess.run([build(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "free: 0 0 1 0" in r.stdout
    assert "sampled: inside 1 refills 1" in r.stdout
    assert "apple x: 0.00 0.10 0.20 0.30" in r.stdout
    assert "reach ring: 1 0" in r.stdout
    yaw0 = ref.sample_orientations(1, [0, 1, 2, 3], None, None, 7, 1, 0)[0]
    assert f"yaw0 {yaw0!r}" in r.stdout or f"yaw0 {yaw0:.17g}" in r.stdout
