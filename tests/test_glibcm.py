"""sb_glibcm.cuh (CPU): the restatement of glibc 2.39's sincos / sin / cos / atan2 (the
functions the reference's std::sin / std::cos / std::atan2 calls run; GCC merges its
adjacent sin / cos pairs into sincos) is bit-identical to the host's libm on the domain the
hot path uses. The device build of the same header is checked in tests/test_gpu_libm.py."""
import ctypes as C
import ctypes.util
import math

import numpy as np
import pytest

from paper_2512_16896_b200 import _capi as A

LIBM = C.CDLL(ctypes.util.find_library("m"))
LIBM.sincos.argtypes = [C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)]
LIBM.sin.restype = LIBM.cos.restype = LIBM.atan2.restype = C.c_double
LIBM.sin.argtypes = LIBM.cos.argtypes = [C.c_double]
LIBM.atan2.argtypes = [C.c_double, C.c_double]


def host(fn, x):
    x = np.ascontiguousarray(x, np.float64)
    n = len(x) // 2 if fn == 2 else len(x)
    out = np.zeros(n)
    A.check(A.lib().sb_host_math(fn, x.ctypes.data_as(C.POINTER(C.c_double)), n,
                                 out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def glibc_sincos(x):
    s, c = C.c_double(), C.c_double()
    out = np.empty((len(x), 2))
    for i, v in enumerate(x):
        LIBM.sincos(float(v), C.byref(s), C.byref(c))
        out[i] = s.value, c.value
    return out


def angles(rng, n):
    """Yaws, arc angles, branch boundaries (0.126, 0.855469, 2.426265, k pi/2) +- ulps."""
    parts = [rng.uniform(0, 2 * math.pi, n), rng.uniform(-7, 10, n // 2),
             rng.uniform(-1, 1, n // 4) * 2.0 ** rng.uniform(-30, 3, n // 4),
             rng.uniform(-1e5, 1e5, n // 8),
             np.array([0.0, -0.0, 1e-300, 5e-324, math.pi, 2 * math.pi, 1.0, -1.0])]
    for c in (0.126, 0.855469, 2.426265, math.pi / 2, math.pi, 3 * math.pi / 2, 2 ** -26, 2 ** -27):
        steps = np.arange(-100, 100)
        parts.append(c + steps * math.ulp(c))
        parts.append(-(c + steps * math.ulp(c)))
    return np.concatenate(parts)


def test_sincos_bit_exact():
    x = angles(np.random.default_rng(0), 100000)
    want = glibc_sincos(x)
    assert np.array_equal(host(0, x).view(np.uint64), want[:, 0].view(np.uint64))
    assert np.array_equal(host(1, x).view(np.uint64), want[:, 1].view(np.uint64))


def test_sin_cos_bit_exact():
    x = angles(np.random.default_rng(1), 50000)
    assert np.array_equal(host(3, x).view(np.uint64),
                          np.array([LIBM.sin(float(v)) for v in x]).view(np.uint64))
    assert np.array_equal(host(4, x).view(np.uint64),
                          np.array([LIBM.cos(float(v)) for v in x]).view(np.uint64))


@pytest.mark.parametrize("scale", [1.0, 1e-3, 1e3])
def test_atan2_bit_exact(scale):
    rng = np.random.default_rng(int(scale * 10) + 3)
    yx = rng.uniform(-1, 1, (60000, 2)) * scale
    t = rng.uniform(-4, 4, 20000)
    unit = np.stack([np.sin(t), np.cos(t)], 1)          # yaw_of of rotation_z poses
    wide = rng.uniform(-1, 1, (20000, 2)) * 2.0 ** rng.uniform(-70, 70, (20000, 2))
    special = np.array([[0, 1], [1, 0], [0, -1], [-1, 0], [-0.0, -1], [-0.0, 1], [0, 0],
                        [-0.0, -0.0], [1, 1], [-1, -1], [0.3, -0.4], [1e-300, 1.0],
                        [1.0, 1e-300], [5e-324, -1.0], [np.inf, 1.0], [1.0, -np.inf],
                        [np.inf, -np.inf], [-np.inf, np.inf]])
    yx = np.concatenate([yx, unit, wide, special])
    got = host(2, yx.reshape(-1))
    want = np.array([LIBM.atan2(float(y), float(x)) for y, x in yx])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_reference_objects_call_sincos_not_sin(ref):
    """The premise: the reference build (oracle/_ref) calls sincos / atan2, never sin / cos."""
    import subprocess

    from oracle import oracle as O

    dis = subprocess.run(["objdump", "-d", O.REF_LIB], capture_output=True, text=True).stdout
    calls = {name for name in ("sincos", "sin", "cos", "atan2") if f"<{name}@plt>" in dis}
    assert "sincos" in calls and "atan2" in calls
    assert "sin" not in calls and "cos" not in calls
