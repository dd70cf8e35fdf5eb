"""Device libm (sb_glibcm.cuh): glibc 2.39's sincos / sin / cos / atan2 restated on the
device, bit-identical to the host's libm -- so rotation_z, annulus arcs, anchor yaws,
local-frame directions and face_to yaws reproduce the reference's bits."""
import ctypes as C

import numpy as np
import pytest

from paper_2512_16896_b200 import _capi as A
from tests.test_glibcm import LIBM, angles, glibc_sincos

pytestmark = pytest.mark.gpu


def device(fn, x):
    x = np.ascontiguousarray(x, np.float64)
    n = len(x) // 2 if fn == 2 else len(x)
    out = np.zeros(n)
    A.check(A.lib().sb_device_math(fn, x.ctypes.data_as(C.POINTER(C.c_double)), n,
                                   out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def test_device_sincos_is_glibc(gpu):
    x = angles(np.random.default_rng(10), 200000)
    want = glibc_sincos(x)
    assert np.array_equal(device(0, x).view(np.uint64), want[:, 0].view(np.uint64))
    assert np.array_equal(device(1, x).view(np.uint64), want[:, 1].view(np.uint64))
    assert np.array_equal(device(3, x).view(np.uint64),
                          np.array([LIBM.sin(float(v)) for v in x]).view(np.uint64))
    assert np.array_equal(device(4, x).view(np.uint64),
                          np.array([LIBM.cos(float(v)) for v in x]).view(np.uint64))


def test_device_atan2_is_glibc(gpu):
    rng = np.random.default_rng(11)
    t = rng.uniform(-4, 4, 50000)
    yx = np.concatenate([rng.uniform(-1, 1, (100000, 2)),
                         np.stack([np.sin(t), np.cos(t)], 1),
                         rng.uniform(-1, 1, (20000, 2)) * 2.0 ** rng.uniform(-70, 70, (20000, 2)),
                         np.array([[0, 1], [1, 0], [0, -1], [-1, 0], [-0.0, -1], [0, 0],
                                   [1e-300, 1.0], [1.0, 1e-300], [0.3, -0.4]])])
    got = device(2, yx.reshape(-1))
    want = np.array([LIBM.atan2(float(y), float(x)) for y, x in yx])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
