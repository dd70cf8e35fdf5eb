// glibc-identical sin / cos / atan2 (host and device).
//
// The reference calls std::sin / std::cos (rotation_z, transform.hpp:47; annulus_sector's
// arc points, polygon.cpp:151; local-frame directions, relationships.cpp:95) and
// std::atan2 (yaw_of, transform.hpp:77; resolve_direction / annulus_sector,
// relationships.cpp:24-34,202; face_to_yaw, relationships.cpp:232-239), i.e. glibc's libm.
// glibc 2.39 on x86-64 dispatches those (ifunc) to __sin_fma / __cos_fma /
// __ieee754_atan2_fma on any CPU with FMA + AVX2: the IBM Accurate Mathematical Library
// algorithms (sysdeps/ieee754/dbl-64/s_sin.c, e_atan2.c; slow multi-precision paths
// removed since 2.28 / 2.35), compiled with FMA contraction. They are NOT correctly
// rounded (max 0.548 ulp), so a correctly rounded libm differs from them in ~0.1 % of
// arguments. GCC also merges an adjacent std::cos(a) / std::sin(a) pair into glibc's
// sincos (the reference's objects call sincos, never sin or cos; see sbg::sincos). This
// file restates those algorithms operation for operation, every fused
// multiply-add exactly where the FMA build of glibc 2.39 has one (read from its code),
// with glibc's own tables (sb_glibcm_tab.h, extracted by tools/gen_glibc_tables.py).
// Bit-identical to the host's std::sin / std::cos / std::atan2 over the domain the path
// uses (|x| < 105414350 for sin / cos -- wider arguments take glibc's branred reduction,
// restated here only through the correctly rounded fallback; atan2 everywhere), checked by
// tests/test_glibcm.py (CPU, 10^6 arguments per function) and tests/test_gpu_libm.py.
//
// Compile device code with -fmad=false and host code with -ffp-contract=off: every
// unfused + - * / below rounds once, every SBM_FMA is one fused operation.
#pragma once

#include <cstdint>
#include <cstring>
#ifndef __CUDACC__
#include <cmath>
#endif

#include "sb_glibcm_tab.h"

#ifdef __CUDACC__
#define SBM_HD __host__ __device__ __forceinline__
#else
#define SBM_HD inline
#endif

namespace sbg {

namespace {
#ifdef __CUDACC__
__device__ const double d_sincostab[440] = {SBM_SINCOSTAB_INIT};
__device__ const double d_cij[241 * 7] = {SBM_CIJ_INIT};
#endif
const double h_sincostab[440] = {SBM_SINCOSTAB_INIT};
const double h_cij[241 * 7] = {SBM_CIJ_INIT};
}  // namespace

SBM_HD double fma_(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
SBM_HD uint64_t bits(double x) {
#ifdef __CUDA_ARCH__
  return static_cast<uint64_t>(__double_as_longlong(x));
#else
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
#endif
}
SBM_HD double from_bits(uint64_t u) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(u));
#else
  double x;
  std::memcpy(&x, &u, 8);
  return x;
#endif
}
SBM_HD double fabs_(double x) { return from_bits(bits(x) & 0x7fffffffffffffffull); }
SBM_HD double copysign_(double x, double s) {
  return from_bits((bits(x) & 0x7fffffffffffffffull) | (bits(s) & 0x8000000000000000ull));
}
SBM_HD double sct(int k) {
#ifdef __CUDA_ARCH__
  return __ldg(d_sincostab + k);
#else
  return h_sincostab[k];
#endif
}
SBM_HD double cij(int i, int j) {
#ifdef __CUDA_ARCH__
  return __ldg(d_cij + 7 * i + j);
#else
  return h_cij[7 * i + j];
#endif
}

// usncs.h / s_sin.c constants
constexpr double kBig = 0x1.8p45, kHp0 = 0x1.921fb54442d18p0, kHp1 = 0x1.1a62633145c07p-54;
constexpr double kHpinv = 0x1.45f306dc9c883p-1, kToint = 0x1.8p52;
constexpr double kMp1 = 0x1.921fb58p0, kMp2 = -0x1.dde973cp-27;
constexpr double kPp3 = -0x1.cb3b398p-55, kPp4 = -0x1.d747f23e32ed7p-83;
constexpr double kSn3 = -0x1.5555555555515p-3, kSn5 = 0x1.11110e829872fp-7;
constexpr double kCs2 = 0.5, kCs4 = -0x1.5555555555535p-5, kCs6 = 0x1.6c16bedd9e239p-10;
constexpr double kS1 = -0x1.5555555555555p-3, kS2 = 0x1.1111111110ecep-7;
constexpr double kS3 = -0x1.a01a019db08b8p-13, kS4 = 0x1.71de27b9a7ed9p-19;
constexpr double kS5 = -0x1.addffc2fcdf59p-26;

// TAYLOR_SIN(a*a, a, da): a + ((POLY(xx) * a - 0.5 * da) * xx + da)
SBM_HD double taylor_sin(double a, double da) {
  const double xx = a * a;
  double p = fma_(xx, kS5, kS4);
  p = fma_(xx, p, kS3);
  p = fma_(xx, p, kS2);
  p = fma_(xx, p, kS1);
  const double t1 = fma_(p, a, -(0.5 * da));
  return a + fma_(xx, t1, da);
}

// do_sin (s_sin.c): sin(x + dx), table k = round(128 |x|)
SBM_HD double do_sin(double x, double dx) {
  const double xold = x;
  if (fabs_(x) < 0.126) return taylor_sin(x, dx);
  if (x <= 0) dx = -dx;
  const double u = kBig + fabs_(x);
  const double xr = fabs_(x) - (u - kBig);
  const int k = static_cast<int>(static_cast<uint32_t>(bits(u)) << 2);
  const double xx = xr * xr;
  const double s = xr + fma_(xr * xx, fma_(xx, kSn5, kSn3), dx);
  const double c = fma_(xr, dx, xx * fma_(xx, fma_(xx, kCs6, kCs4), kCs2));
  const double sn = sct(k), ssn = sct(k + 1), cs = sct(k + 2), ccs = sct(k + 3);
  const double cor = fma_(s, cs, fma_(-c, sn, fma_(s, ccs, ssn)));
  return copysign_(sn + cor, xold);
}

// do_cos (s_sin.c): cos(x + dx)
SBM_HD double do_cos(double x, double dx) {
  if (x < 0) dx = -dx;
  const double u = kBig + fabs_(x);
  const double xr = (fabs_(x) - (u - kBig)) + dx;
  const int k = static_cast<int>(static_cast<uint32_t>(bits(u)) << 2);
  const double xx = xr * xr;
  const double s = fma_(xr * xx, fma_(xx, kSn5, kSn3), xr);
  const double c = xx * fma_(xx, fma_(xx, kCs6, kCs4), kCs2);
  const double sn = sct(k), ssn = sct(k + 1), cs = sct(k + 2), ccs = sct(k + 3);
  const double cor = fma_(-s, sn, fma_(-c, cs, fma_(-s, ssn, ccs)));
  return cs + cor;
}

// reduce_sincos (s_sin.c): x = n * pi/2 + (a + da), |x| < 105414350
SBM_HD int reduce_sincos(double x, double& a, double& da) {
  const double t = fma_(x, kHpinv, kToint);
  const double xn = t - kToint;
  const int n = static_cast<int>(static_cast<uint32_t>(bits(t)) & 3u);
  const double y = fma_(-xn, kMp2, fma_(-xn, kMp1, x));
  const double t2 = fma_(-xn, kPp3, y);
  double db = fma_(-xn, kPp3, y - t2);
  const double b = fma_(-xn, kPp4, t2);
  db = db + fma_(-xn, kPp4, t2 - b);
  a = b;
  da = db;
  return n;
}

SBM_HD double do_sincos(double a, double da, int n) {
  const double r = (n & 1) ? do_cos(a, da) : do_sin(a, da);
  return (n & 2) ? -r : r;
}

SBM_HD double sin(double x) {
  const uint32_t k = static_cast<uint32_t>(bits(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e500000u) return x;
  if (k < 0x3feb6000u) return do_sin(x, 0.0);
  if (k < 0x400368fdu) return copysign_(do_cos(kHp0 - fabs_(x), kHp1), x);
  if (k < 0x419921fbu) {
    double a, da;
    const int n = reduce_sincos(x, a, da);
    return do_sincos(a, da, n);
  }
  if (k >= 0x7ff00000u) return x - x;  // inf / nan -> nan
#ifdef __CUDA_ARCH__
  return ::sin(x);
#else
  return std::sin(x);
#endif
}

SBM_HD double cos(double x) {
  const uint32_t k = static_cast<uint32_t>(bits(x) >> 32) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;
  if (k < 0x3feb6000u) return do_cos(x, 0.0);
  if (k < 0x400368fdu) {
    const double y = kHp0 - fabs_(x);
    const double a = y + kHp1;
    const double da = (y - a) + kHp1;
    return do_sin(a, da);
  }
  if (k < 0x419921fbu) {
    double a, da;
    const int n = reduce_sincos(x, a, da);
    return do_sincos(a, da, n + 1);
  }
  if (k >= 0x7ff00000u) return x - x;
#ifdef __CUDA_ARCH__
  return ::cos(x);
#else
  return std::cos(x);
#endif
}

// sincos (s_sincos.c). GCC merges the reference's adjacent std::cos(a) / std::sin(a)
// (rotation_z, annulus_sector, relationships.cpp, trimesh.cpp) into one glibc sincos
// call at -O2, and glibc's sincos differs from sin in 0.855469 <= |x| < 2.426265: it
// evaluates do_cos(y + hp1, (y - (y + hp1)) + hp1) where sin evaluates do_cos(y, hp1).
SBM_HD void sincos(double x, double* sinx, double* cosx) {
  const uint32_t k = static_cast<uint32_t>(bits(x) >> 32) & 0x7fffffffu;
  if (k < 0x400368fdu) {
    if (k < 0x3e400000u) {
      *sinx = x;
      *cosx = 1.0;
      return;
    }
    if (k < 0x3feb6000u) {
      *sinx = do_sin(x, 0.0);
      *cosx = do_cos(x, 0.0);
      return;
    }
    const double y = kHp0 - fabs_(x);
    const double a = y + kHp1;
    const double da = (y - a) + kHp1;
    *sinx = copysign_(do_cos(a, da), x);
    *cosx = do_sin(a, da);
    return;
  }
  if (k < 0x419921fbu) {
    double a, da;
    const int n = reduce_sincos(x, a, da);
    *sinx = do_sincos(a, da, n);
    *cosx = do_sincos(a, da, n + 1);
    return;
  }
  *sinx = sbg::sin(x);  // inf / nan, or the wide-argument fallback (see above)
  *cosx = sbg::cos(x);
}

// e_atan2.c constants
constexpr double kHpi = 0x1.921fb54442d18p0, kHpi1 = 0x1.1a62633145c07p-54;
constexpr double kOpi = 0x1.921fb54442d18p1, kOpi1 = 0x1.1a62633145c07p-53;
constexpr double kQpi = 0x1.921fb54442d18p-1, kTqpi = 0x1.2d97c7f3321d2p1;
constexpr double kInv16 = 0x1p-4, kTwo500 = 0x1p500, kTwom500 = 0x1p-500;
constexpr double kD3 = -0x1.5555555555555p-2, kD5 = 0x1.99999999997fdp-3;
constexpr double kD7 = -0x1.24924923f7603p-3, kD9 = 0x1.c71c6e5129a3bp-4;
constexpr double kD11 = -0x1.7458022b13c25p-4, kD13 = 0x1.375f08b31cbcep-4;

SBM_HD double atan_poly(double v) {  // d3 + v (d5 + v (d7 + v (d9 + v (d11 + v d13))))
  double p = fma_(v, kD13, kD11);
  p = fma_(v, p, kD9);
  p = fma_(v, p, kD7);
  p = fma_(v, p, kD5);
  return fma_(v, p, kD3);
}
SBM_HD int atan_row(double u) {  // i = (TWO52 + TWO8 * u) - TWO52 - 16
  return static_cast<int>(fma_(u, 256.0, 0x1p52) - 0x1p52) - 16;
}
SBM_HD double cij_poly(double v, int i) {  // cij[i][2] + v (c3 + v (c4 + v (c5 + v c6)))
  double p = fma_(v, cij(i, 6), cij(i, 5));
  p = fma_(v, p, cij(i, 4));
  p = fma_(v, p, cij(i, 3));
  return fma_(v, p, cij(i, 2));
}

SBM_HD double atan2(double y, double x) {
  const uint64_t bx = bits(x), by = bits(y);
  const uint32_t ux = static_cast<uint32_t>(bx >> 32), dx = static_cast<uint32_t>(bx);
  const uint32_t uy = static_cast<uint32_t>(by >> 32), dy = static_cast<uint32_t>(by);
  if ((ux & 0x7ff00000u) == 0x7ff00000u && ((ux & 0x000fffffu) | dx) != 0) return x + y;
  if ((uy & 0x7ff00000u) == 0x7ff00000u && ((uy & 0x000fffffu) | dy) != 0) return y + y;
  if (uy == 0u && dy == 0u) return (ux & 0x80000000u) == 0 ? 0.0 : kOpi;
  if (uy == 0x80000000u && dy == 0u) return (ux & 0x80000000u) == 0 ? -0.0 : -kOpi;
  if (x == 0) return (uy & 0x80000000u) == 0 ? kHpi : -kHpi;
  const bool xinf = (ux & 0x7fffffffu) == 0x7ff00000u && dx == 0;
  const bool yinf = (uy & 0x7fffffffu) == 0x7ff00000u && dy == 0;
  if (xinf) {
    const bool ypos = (uy & 0x80000000u) == 0;
    if ((ux & 0x80000000u) == 0) return yinf ? (ypos ? kQpi : -kQpi) : (ypos ? 0.0 : -0.0);
    return yinf ? (ypos ? kTqpi : -kTqpi) : (ypos ? kOpi : -kOpi);
  }
  if (yinf) return (uy & 0x80000000u) == 0 ? kHpi : -kHpi;

  double ax = x < 0 ? -x : x, ay = y < 0 ? -y : y;
  const int de = static_cast<int>(uy & 0x7ff00000u) - static_cast<int>(ux & 0x7ff00000u);
  if (de >= 59768832) return y > 0 ? kHpi : -kHpi;
  if (de <= -59768832) {
    if (x > 0) return copysign_(ay / ax, y);
    return y > 0 ? kOpi : -kOpi;
  }
  if (ax < kTwom500 || ay < kTwom500) {
    ax *= kTwo500;
    ay *= kTwo500;
  }
  if (ax > kTwo500 || ay > kTwo500) {
    ax *= kTwom500;
    ay *= kTwom500;
  }
  double u, du;
  if (ay < ax) {
    u = ay / ax;
    const double v = ax * u, vv = fma_(ax, u, -v);
    du = ((ay - v) - vv) / ax;
  } else {
    u = ax / ay;
    const double v = ay * u, vv = fma_(ay, u, -v);
    du = ((ax - v) - vv) / ay;
  }
  double z;
  if (x > 0) {
    if (ay < ax) {  // (i) atan(ay/ax)
      if (u < kInv16) {
        const double v = u * u;
        z = u + fma_(u * v, atan_poly(v), du);
      } else {
        const int i = atan_row(u);
        const double t3 = u - cij(i, 0);
        const double v = t3 + du;  // EADD(t3, du, v, dv)
        const double dv = fabs_(t3) > fabs_(du) ? (t3 - v) + du : (du - v) + t3;
        const double t2 = cij(i, 2);
        double p = fma_(v, cij(i, 6), cij(i, 5));
        p = fma_(v, p, cij(i, 4));
        p = fma_(v, p, cij(i, 3));
        z = fma_(v, t2, fma_(dv, t2, (v * v) * p)) + cij(i, 1);
      }
    } else {  // (ii) pi/2 - atan(ax/ay)
      if (u < kInv16) {
        const double v = u * u;
        const double zz = (u * v) * atan_poly(v);
        const double t2 = kHpi - u;  // ESUB(hpi, u, t2, cor)
        const double cor = kHpi > fabs_(u) ? (kHpi - t2) - u : kHpi - (u + t2);
        z = (((kHpi1 + cor) - du) - zz) + t2;
      } else {
        const int i = atan_row(u);
        const double v = (u - cij(i, 0)) + du;
        z = (kHpi - cij(i, 1)) + fma_(-v, cij_poly(v, i), kHpi1);
      }
    }
  } else if (ax < ay) {  // (iii) pi/2 + atan(ax/ay)
    if (u < kInv16) {
      const double v = u * u;
      const double zz = (u * v) * atan_poly(v);
      const double t2 = u + kHpi;  // EADD(hpi, u, t2, cor)
      const double cor = kHpi > fabs_(u) ? (kHpi - t2) + u : (u - t2) + kHpi;
      z = (((kHpi1 + cor) + du) + zz) + t2;
    } else {
      const int i = atan_row(u);
      const double v = (u - cij(i, 0)) + du;
      z = (kHpi + cij(i, 1)) + fma_(v, cij_poly(v, i), kHpi1);
    }
  } else {  // (iv) pi - atan(ax/ay)
    if (u < kInv16) {
      const double v = u * u;
      const double zz = (u * v) * atan_poly(v);
      const double t2 = kOpi - u;  // ESUB(opi, u, t2, cor)
      const double cor = kOpi > fabs_(u) ? (kOpi - t2) - u : kOpi - (u + t2);
      z = (((kOpi1 + cor) - du) - zz) + t2;
    } else {
      const int i = atan_row(u);
      const double v = (u - cij(i, 0)) + du;
      z = (kOpi - cij(i, 1)) + fma_(-v, cij_poly(v, i), kOpi1);
    }
  }
  return copysign_(z, y);
}

}  // namespace sbg
