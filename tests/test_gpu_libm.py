"""Device libm (sb_crmath.cuh): correctly rounded sin / cos / atan2 so that rotation_z,
annulus arcs and anchor yaws reproduce glibc's std::sin / std::cos / std::atan2 bits."""
import ctypes as C
import math

import numpy as np
import pytest

from paper_2512_16896_b200 import _capi as A

pytestmark = pytest.mark.gpu


def device(fn, x):
    x = np.ascontiguousarray(x, np.float64)
    n = len(x) // 2 if fn == 2 else len(x)
    out = np.zeros(n)
    A.check(A.lib().sb_device_math(fn, x.ctypes.data_as(C.POINTER(C.c_double)), n,
                                   out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def test_sincos_matches_glibc_and_is_correctly_rounded(gpu):
    import mpmath as mp

    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(0, 2 * math.pi, 200000),          # yaws
                        rng.uniform(-7, 10, 50000),                    # arc angles
                        np.array([0.0, math.pi / 2, math.pi, 2 * math.pi, 1e-9, -1e-7])])
    s, c = device(0, x), device(1, x)
    gs = np.array([math.sin(v) for v in x])
    gc = np.array([math.cos(v) for v in x])
    ms, mc = (s != gs).mean(), (c != gc).mean()
    assert ms < 3e-3 and mc < 3e-3, (ms, mc)  # glibc itself misrounds ~1e-3
    mp.mp.prec = 200
    sub = rng.choice(len(x), 3000, replace=False)
    cr_s = sum(s[i] != float(mp.sin(mp.mpf(x[i]))) for i in sub)
    cr_c = sum(c[i] != float(mp.cos(mp.mpf(x[i]))) for i in sub)
    assert cr_s == 0 and cr_c == 0


def test_atan2_matches_glibc_and_is_correctly_rounded(gpu):
    import mpmath as mp

    rng = np.random.default_rng(1)
    yx = rng.uniform(-1, 1, (100000, 2))
    special = np.array([[0, 1], [1, 0], [0, -1], [-1, 0], [-0.0, -1], [1, 1], [-1, -1],
                        [0.3, -0.4], [1e-300, 1.0], [1.0, 1e-300]])
    yx = np.concatenate([yx, special])
    a = device(2, yx.reshape(-1))
    g = np.array([math.atan2(y, x) for y, x in yx])
    assert (a != g).mean() < 3e-3
    assert np.array_equal(a[-len(special):], g[-len(special):])
    mp.mp.prec = 200
    sub = rng.choice(len(yx), 3000, replace=False)
    assert sum(a[i] != float(mp.atan2(mp.mpf(yx[i, 0]), mp.mpf(yx[i, 1]))) for i in sub) == 0
