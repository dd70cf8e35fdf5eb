// Device-side restatements of the reference hot-path arithmetic (sm_100a, FP64).
//
// Compiled with -fmad=false: every +,-,*,/ rounds once, exactly as the reference's
// default x86-64 build (SSE2, no FMA) does, and every reduction follows the reference's
// Eigen expression order (left to right; oracle/shim/Eigen/Dense). sqrt and division are
// IEEE correctly rounded on both sides, so masks, accepted indices and sampled positions
// are bit-identical to the reference except where a libm transcendental (sin, cos, atan2)
// is involved -- see DESIGN.md "libm".
#pragma once

#include <stdint.h>

#include "sb_layout.h"

namespace sbd {

constexpr double kEps = 1e-12;  // collision.cpp:11

// ------------------------------------------------------------------------- RNG
constexpr uint64_t kPcgMult = 6364136223846793005ULL;
constexpr uint64_t kPcgSeq = 0xda3e39cb94b95bdbULL;
constexpr uint64_t kPcgInc = (kPcgSeq << 1u) | 1u;
constexpr uint64_t kCacheSalt = 0x63616368ULL;     // "cach" sampler.cpp:9
constexpr uint64_t kFallbackSalt = 0x66616c6cULL;  // "fall" sampler.cpp:10
constexpr uint64_t kYawSalt = 0x79617721ULL;       // "yaw!" sampler.cpp:11

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {  // rng.hpp:9-14
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// Pcg32 (rng.hpp:24-60). Only the state is carried; inc is the fixed default sequence.
struct Pcg {
  uint64_t state;

  // Pcg32(seed): state=0, step, state += seed, step (rng.hpp:26-31).
  __host__ __device__ __forceinline__ static Pcg seeded(uint64_t seed) {
    Pcg p{0};
    p.state = kPcgInc;  // 0 * mult + inc
    p.state += seed;
    p.state = p.state * kPcgMult + kPcgInc;
    return p;
  }
  __host__ __device__ __forceinline__ uint32_t next_u32() {
    uint64_t old = state;
    state = old * kPcgMult + kPcgInc;
    uint32_t xorshifted = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
    uint32_t rot = static_cast<uint32_t>(old >> 59u);
    return (xorshifted >> rot) | (xorshifted << ((32u - rot) & 31u));
  }
  // GCC evaluates the unsequenced operands left to right: first draw is the high word
  // (rng.hpp:42; pinned by the KAT Pcg32(12345).next_u64() = 8630b53a16ac2a2c).
  __host__ __device__ __forceinline__ uint64_t next_u64() {
    uint64_t hi = next_u32();
    uint64_t lo = next_u32();
    return (hi << 32) | lo;
  }
  __host__ __device__ __forceinline__ double next_double() {
    return static_cast<double>(next_u64() >> 11) * 0x1.0p-53;
  }
  // LCG jump-ahead by `delta` steps (Brown, "Random number generation with arbitrary
  // strides"): the j-th drained fast-path point is draw j, i.e. 6j steps in.
  __host__ __device__ __forceinline__ void advance(uint64_t delta) {
    uint64_t cur_mult = kPcgMult, cur_plus = kPcgInc, acc_mult = 1u, acc_plus = 0u;
    while (delta > 0) {
      if (delta & 1u) {
        acc_mult *= cur_mult;
        acc_plus = acc_plus * cur_mult + cur_plus;
      }
      cur_plus = (cur_mult + 1u) * cur_plus;
      cur_mult *= cur_mult;
      delta >>= 1u;
    }
    state = acc_mult * state + acc_plus;
  }
};

// LCG jump by whole fast-path draws (6 steps each) from a table of powers: entry
// [k][d] = {mult, plus} of the map "advance 6 * d * 256^k steps"; the jumps commute, so
// state(draw) = J3[b3] J2[b2] J1[b1] J0[b0] state0 for the bytes b of `draw` -- the same
// state advance(6 * draw) reaches (modular arithmetic, bit-exact), in 4 multiply-adds
// instead of ~21 squaring rounds. Built by pcg_jump_table_host; draws < 2^32.
__device__ __forceinline__ uint64_t pcg_jump_draws(const uint64_t* table, uint64_t state, uint64_t draw) {
#pragma unroll
  for (int k = 0; k < SB_PCG_JUMP_LEVELS; ++k) {
    const uint32_t d = static_cast<uint32_t>(draw >> (8 * k)) & 0xffu;
    if (d) {
      const ulonglong2 e = __ldg(reinterpret_cast<const ulonglong2*>(table) + (k * 256 + d));
      state = e.x * state + e.y;
    }
  }
  return state;
}

// make_stream(seed, {c0, c1, ...}) (rng.hpp:63-67)
__host__ __device__ __forceinline__ uint64_t stream_seed2(uint64_t seed, uint64_t c0, uint64_t c1) {
  return mix64(mix64(mix64(seed) ^ c0) ^ c1);
}
__host__ __device__ __forceinline__ uint64_t stream_seed4(uint64_t seed, uint64_t c0, uint64_t c1,
                                                          uint64_t c2, uint64_t c3) {
  return mix64(mix64(mix64(mix64(mix64(seed) ^ c0) ^ c1) ^ c2) ^ c3);
}

// ------------------------------------------------------------------ transforms
// Rigid pose as a 3x4 row-major block [R | t]; the bottom row is (0,0,0,1) by contract.
struct M34 {
  double m[12];
  __device__ __forceinline__ double r(int i, int j) const { return m[4 * i + j]; }
  __device__ __forceinline__ double t(int i) const { return m[4 * i + 3]; }
};

// Mat4 product A*B as the reference computes it (shim: ((a0 b0 + a1 b1) + a2 b2) + a3 b3),
// with both bottom rows (0,0,0,1); rows 0..2 only (row 3 is never read downstream).
__device__ __forceinline__ void mul34(const M34& A, const M34& B, M34& C) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double b3 = j == 3 ? 1.0 : 0.0;
      double s = A.m[4 * i + 0] * B.m[0 + j];
      s = s + A.m[4 * i + 1] * B.m[4 + j];
      s = s + A.m[4 * i + 2] * B.m[8 + j];
      s = s + A.m[4 * i + 3] * b3;
      C.m[4 * i + j] = s;
    }
  }
}

// inverse_rigid (transform.hpp:63-69): [R^T | (-R^T) t]
__device__ __forceinline__ void inverse_rigid(const M34& P, M34& I) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int k = 0; k < 3; ++k) I.m[4 * i + k] = P.m[4 * k + i];
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    double s = (-I.m[4 * i + 0]) * P.m[3];
    s = s + (-I.m[4 * i + 1]) * P.m[7];
    s = s + (-I.m[4 * i + 2]) * P.m[11];
    I.m[4 * i + 3] = s;
  }
}

// transform_point (transform.hpp:71-73): R p + t, left to right.
__device__ __forceinline__ void xform(const M34& M, double px, double py, double pz, double& ox,
                                      double& oy, double& oz) {
  ox = ((M.m[0] * px + M.m[1] * py) + M.m[2] * pz) + M.m[3];
  oy = ((M.m[4] * px + M.m[5] * py) + M.m[6] * pz) + M.m[7];
  oz = ((M.m[8] * px + M.m[9] * py) + M.m[10] * pz) + M.m[11];
}

// transform_aabb (aabb.hpp:54-62) from a precomputed center c / half extent h.
__device__ __forceinline__ void xform_aabb(const M34& M, const double c[3], const double h[3],
                                           double mn[3], double mx[3]) {
  double cx, cy, cz;
  xform(M, c[0], c[1], c[2], cx, cy, cz);
  double wx = (fabs(M.m[0]) * h[0] + fabs(M.m[1]) * h[1]) + fabs(M.m[2]) * h[2];
  double wy = (fabs(M.m[4]) * h[0] + fabs(M.m[5]) * h[1]) + fabs(M.m[6]) * h[2];
  double wz = (fabs(M.m[8]) * h[0] + fabs(M.m[9]) * h[1]) + fabs(M.m[10]) * h[2];
  mn[0] = cx - wx;
  mn[1] = cy - wy;
  mn[2] = cz - wz;
  mx[0] = cx + wx;
  mx[1] = cy + wy;
  mx[2] = cz + wz;
}

// Aabb3::overlaps with margin 0 (aabb.hpp:29-33): inclusive.
__device__ __forceinline__ bool overlaps(const double amn[3], const double amx[3],
                                         const double bmn[3], const double bmx[3]) {
  return amn[0] <= bmx[0] && bmn[0] <= amx[0] && amn[1] <= bmx[1] && bmn[1] <= amx[1] &&
         amn[2] <= bmx[2] && bmn[2] <= amx[2];
}

// ------------------------------------------------------- triangle-triangle test
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }  // std::min
__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }  // std::max

// isect_interval (collision.cpp:14-20)
__device__ __forceinline__ void isect_interval(double vv0, double vv1, double vv2, double d0,
                                               double d1, double d2, double& lo, double& hi) {
  double t0 = vv0 + (vv1 - vv0) * d0 / (d0 - d1);
  double t1 = vv2 + (vv1 - vv2) * d2 / (d2 - d1);
  lo = dmin(t0, t1);
  hi = dmax(t0, t1);
}

// compute_interval (collision.cpp:23-40); false = coplanar
__device__ __forceinline__ bool compute_interval(double p0, double p1, double p2, double d0,
                                                 double d1, double d2, double& lo, double& hi) {
  if (d0 * d1 > 0.0) {
    isect_interval(p0, p2, p1, d0, d2, d1, lo, hi);
  } else if (d0 * d2 > 0.0) {
    isect_interval(p0, p1, p2, d0, d1, d2, lo, hi);
  } else if (d1 * d2 > 0.0 || d0 != 0.0) {
    isect_interval(p1, p0, p2, d1, d0, d2, lo, hi);
  } else if (d1 != 0.0) {
    isect_interval(p0, p1, p2, d0, d1, d2, lo, hi);
  } else if (d2 != 0.0) {
    isect_interval(p0, p2, p1, d0, d2, d1, lo, hi);
  } else {
    return false;
  }
  return true;
}

__device__ __forceinline__ double orient2(double px, double py, double qx, double qy, double rx,
                                          double ry) {
  return (qx - px) * (ry - py) - (qy - py) * (rx - px);
}

// seg_seg_cross_2d (collision.cpp:42-51): strict crossing only
__device__ __forceinline__ bool seg_cross(double ax, double ay, double bx, double by, double cx,
                                          double cy, double dx, double dy) {
  double o1 = orient2(ax, ay, bx, by, cx, cy), o2 = orient2(ax, ay, bx, by, dx, dy);
  double o3 = orient2(cx, cy, dx, dy, ax, ay), o4 = orient2(cx, cy, dx, dy, bx, by);
  return ((o1 > kEps && o2 < -kEps) || (o1 < -kEps && o2 > kEps)) &&
         ((o3 > kEps && o4 < -kEps) || (o3 < -kEps && o4 > kEps));
}

// point_in_tri_2d (collision.cpp:53-61)
__device__ __forceinline__ bool point_in_tri(double px, double py, double ax, double ay, double bx,
                                             double by, double cx, double cy) {
  double d1 = orient2(ax, ay, bx, by, px, py);
  double d2 = orient2(bx, by, cx, cy, px, py);
  double d3 = orient2(cx, cy, ax, ay, px, py);
  bool has_neg = d1 < -kEps || d2 < -kEps || d3 < -kEps;
  bool has_pos = d1 > kEps || d2 > kEps || d3 > kEps;
  return !(has_neg && has_pos) && (has_neg || has_pos);
}

// coplanar_tri_tri (collision.cpp:63-83)
static __device__ __noinline__ bool coplanar_tri_tri(const double n[3], const double* p, const double* q) {
  int axis = 0;
  double an0 = fabs(n[0]), an1 = fabs(n[1]), an2 = fabs(n[2]);
  if (an1 > an0) axis = 1;
  if (an2 > (axis == 0 ? an0 : an1)) axis = 2;
  int u = (axis + 1) % 3, v = (axis + 2) % 3;
  double t1x[3] = {p[u], p[3 + u], p[6 + u]}, t1y[3] = {p[v], p[3 + v], p[6 + v]};
  double t2x[3] = {q[u], q[3 + u], q[6 + u]}, t2y[3] = {q[v], q[3 + v], q[6 + v]};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (seg_cross(t1x[i], t1y[i], t1x[(i + 1) % 3], t1y[(i + 1) % 3], t2x[j], t2y[j],
                    t2x[(j + 1) % 3], t2y[(j + 1) % 3]))
        return true;
  double c1x = (t1x[0] + t1x[1] + t1x[2]) / 3.0, c1y = (t1y[0] + t1y[1] + t1y[2]) / 3.0;
  double c2x = (t2x[0] + t2x[1] + t2x[2]) / 3.0, c2y = (t2y[0] + t2y[1] + t2y[2]) / 3.0;
  if (point_in_tri(c1x, c1y, t2x[0], t2y[0], t2x[1], t2y[1], t2x[2], t2y[2])) return true;
  if (point_in_tri(c2x, c2y, t1x[0], t1y[0], t1x[1], t1y[1], t1x[2], t1y[2])) return true;
  return false;
}

// tri_tri_intersect (collision.cpp:87-130), split into the stages the warp narrow phase
// runs as separate filter passes. Every quantity is computed with the reference's
// operations in the reference's order, so the staged and the monolithic forms agree bit
// for bit; only *when* a pure function of one triangle is evaluated changes.
struct TriPlane {
  double n[3];  // cross(v1 - v0, v2 - v0)
  double dc;    // -dot(n, v0)
  double tol;   // kEps * max(1, |n|)  (collision.cpp:95-98 / 108-110)
};

__device__ __forceinline__ TriPlane tri_plane(const double* t) {
  TriPlane P;
  double e1x = t[3] - t[0], e1y = t[4] - t[1], e1z = t[5] - t[2];
  double e2x = t[6] - t[0], e2y = t[7] - t[1], e2z = t[8] - t[2];
  P.n[0] = e1y * e2z - e1z * e2y;
  P.n[1] = e1z * e2x - e1x * e2z;
  P.n[2] = e1x * e2y - e1y * e2x;
  P.dc = -((P.n[0] * t[0] + P.n[1] * t[1]) + P.n[2] * t[2]);
  double scale = sqrt((P.n[0] * P.n[0] + P.n[1] * P.n[1]) + P.n[2] * P.n[2]);
  P.tol = kEps * dmax(1.0, scale);
  return P;
}

// Signed distances of t's vertices to plane (n, dc), snapped to 0 below tol.
__device__ __forceinline__ void plane_dists(const double* n, double dc, double tol, const double* t,
                                            double& d0, double& d1, double& d2) {
  d0 = ((n[0] * t[0] + n[1] * t[1]) + n[2] * t[2]) + dc;
  d1 = ((n[0] * t[3] + n[1] * t[4]) + n[2] * t[5]) + dc;
  d2 = ((n[0] * t[6] + n[1] * t[7]) + n[2] * t[8]) + dc;
  if (fabs(d0) < tol) d0 = 0.0;
  if (fabs(d1) < tol) d1 = 0.0;
  if (fabs(d2) < tol) d2 = 0.0;
}

// false = all three strictly on one side (the early-outs of collision.cpp:99,111)
__device__ __forceinline__ bool straddles(double d0, double d1, double d2) {
  return !((d0 > 0 && d1 > 0 && d2 > 0) || (d0 < 0 && d1 < 0 && d2 < 0));
}

// Rest of the test once both plane tests passed (collision.cpp:113-129).
__device__ __forceinline__ bool tri_tri_finish(const double* p, const double* q, const double n1[3],
                                               const double n2[3], double dp0, double dp1,
                                               double dp2, double dq0, double dq1, double dq2) {
  if (dp0 == 0 && dp1 == 0 && dp2 == 0) return coplanar_tri_tri(n1, p, q);

  double dir0 = n1[1] * n2[2] - n1[2] * n2[1];
  double dir1 = n1[2] * n2[0] - n1[0] * n2[2];
  double dir2 = n1[0] * n2[1] - n1[1] * n2[0];
  int axis = 0;
  double ad0 = fabs(dir0), ad1 = fabs(dir1), ad2 = fabs(dir2);
  if (ad1 > ad0) axis = 1;
  if (ad2 > (axis == 0 ? ad0 : ad1)) axis = 2;

  double lo1, hi1, lo2, hi2;
  if (!compute_interval(p[axis], p[3 + axis], p[6 + axis], dp0, dp1, dp2, lo1, hi1))
    return coplanar_tri_tri(n1, p, q);
  if (!compute_interval(q[axis], q[3 + axis], q[6 + axis], dq0, dq1, dq2, lo2, hi2))
    return coplanar_tri_tri(n1, p, q);
  return hi1 > lo2 + kEps && hi2 > lo1 + kEps;
}

// tri_tri_intersect (collision.cpp:87-130). p, q: 9 doubles each (three xyz vertices).
__device__ __forceinline__ bool tri_tri_intersect(const double* p, const double* q) {
  const TriPlane P2 = tri_plane(q);
  double dp0, dp1, dp2;
  plane_dists(P2.n, P2.dc, P2.tol, p, dp0, dp1, dp2);
  if (!straddles(dp0, dp1, dp2)) return false;
  const TriPlane P1 = tri_plane(p);
  double dq0, dq1, dq2;
  plane_dists(P1.n, P1.dc, P1.tol, q, dq0, dq1, dq2);
  if (!straddles(dq0, dq1, dq2)) return false;
  return tri_tri_finish(p, q, P1.n, P2.n, dp0, dp1, dp2, dq0, dq1, dq2);
}

// ------------------------------------------------ triangle distance (margin > 0)
// collision.cpp:136-212 with the shim's vector arithmetic (dot = ((x x' + y y') + z z'),
// element-wise +, -, scalar *). Only used when the world's margin is > 0.
struct V3 {
  double x, y, z;
};
__device__ __forceinline__ V3 v3(const double* p) { return {p[0], p[1], p[2]}; }
__device__ __forceinline__ V3 vsub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ V3 vadd(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ V3 vmul(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ double vdot(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__device__ __forceinline__ double vnorm(V3 a) { return sqrt(vdot(a, a)); }
__device__ __forceinline__ double clamp01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

static __device__ __noinline__ double seg_seg_distance(V3 p0, V3 p1, V3 q0, V3 q1) {
  const V3 d1 = vsub(p1, p0), d2 = vsub(q1, q0), r = vsub(p0, q0);
  const double a = vdot(d1, d1), e = vdot(d2, d2), f = vdot(d2, r);
  double s, t;
  if (a <= kEps && e <= kEps) return vnorm(r);
  if (a <= kEps) {
    s = 0.0;
    t = clamp01(f / e);
  } else {
    const double c = vdot(d1, r);
    if (e <= kEps) {
      t = 0.0;
      s = clamp01(-c / a);
    } else {
      const double b = vdot(d1, d2);
      const double denom = a * e - b * b;
      s = denom > kEps ? clamp01((b * f - c * e) / denom) : 0.0;
      t = (b * s + f) / e;
      if (t < 0.0) {
        t = 0.0;
        s = clamp01(-c / a);
      } else if (t > 1.0) {
        t = 1.0;
        s = clamp01((b - c) / a);
      }
    }
  }
  return vnorm(vsub(vadd(p0, vmul(d1, s)), vadd(q0, vmul(d2, t))));
}

static __device__ __noinline__ double point_tri_distance(V3 p, V3 a, V3 b, V3 c) {
  const V3 ab = vsub(b, a), ac = vsub(c, a), ap = vsub(p, a);
  const double d1 = vdot(ab, ap), d2 = vdot(ac, ap);
  if (d1 <= 0 && d2 <= 0) return vnorm(ap);
  const V3 bp = vsub(p, b);
  const double d3 = vdot(ab, bp), d4 = vdot(ac, bp);
  if (d3 >= 0 && d4 <= d3) return vnorm(bp);
  const double vc = d1 * d4 - d3 * d2;
  if (vc <= 0 && d1 >= 0 && d3 <= 0) {
    const double v = d1 / (d1 - d3);
    return vnorm(vsub(p, vadd(a, vmul(ab, v))));
  }
  const V3 cp = vsub(p, c);
  const double d5 = vdot(ab, cp), d6 = vdot(ac, cp);
  if (d6 >= 0 && d5 <= d6) return vnorm(cp);
  const double vb = d5 * d2 - d1 * d6;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) {
    const double w = d2 / (d2 - d6);
    return vnorm(vsub(p, vadd(a, vmul(ac, w))));
  }
  const double va = d3 * d6 - d5 * d4;
  if (va <= 0 && (d4 - d3) >= 0 && (d5 - d6) >= 0) {
    const double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    return vnorm(vsub(p, vadd(b, vmul(vsub(c, b), w))));
  }
  const double denom = 1.0 / (va + vb + vc);
  const double v = vb * denom, w = vc * denom;
  return vnorm(vsub(p, vadd(vadd(a, vmul(ab, v)), vmul(ac, w))));
}

// tri_tri_distance (collision.cpp:198-212); p, q: 9 doubles each.
static __device__ __noinline__ double tri_tri_distance(const double* p, const double* q) {
  if (tri_tri_intersect(p, q)) return 0.0;
  const V3 pa[3] = {v3(p), v3(p + 3), v3(p + 6)};
  const V3 qa[3] = {v3(q), v3(q + 3), v3(q + 6)};
  double best = __longlong_as_double(0x7ff0000000000000LL);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      best = dmin(best, seg_seg_distance(pa[i], pa[(i + 1) % 3], qa[j], qa[(j + 1) % 3]));
  for (int i = 0; i < 3; ++i) {
    best = dmin(best, point_tri_distance(pa[i], qa[0], qa[1], qa[2]));
    best = dmin(best, point_tri_distance(qa[i], pa[0], pa[1], pa[2]));
  }
  return best;
}

// Aabb3::overlaps with margin (aabb.hpp:29-33): a.min <= b.max + m && b.min <= a.max + m.
__device__ __forceinline__ bool overlaps_m(const double amn[3], const double amx[3],
                                           const double bmn[3], const double bmx[3], double m) {
  return amn[0] <= bmx[0] + m && bmn[0] <= amx[0] + m && amn[1] <= bmx[1] + m &&
         bmn[1] <= amx[1] + m && amn[2] <= bmx[2] + m && bmn[2] <= amx[2] + m;
}

// ---------------------------------------------------------- BVH-vs-BVH collide
// MeshBvh::collide (collision.cpp:285-329) over the effective DAGs of A (candidate, frame
// of reference) and B (placed object, posed by M = other_in_self). Each node pair is
// visited once (the reference revisits pairs reachable along several {left, left+1}
// paths; the boolean result is the same existential). Pairs are processed in
// lexicographic (a, b) order, which is a topological order of the pair DAG because every
// child id exceeds its parent's, so a pending bit is never set after it was consumed.
__device__ __forceinline__ bool collide(const SbNode* __restrict__ A, int nA,
                                        const SbNode* __restrict__ B,
                                        const SbTri* __restrict__ trisA,
                                        const SbTri* __restrict__ trisB, const M34& M,
                                        uint32_t& node_tests, uint32_t& pair_tests) {
  uint32_t pend[SB_MAX_NODES_PER_GEOM];
  for (int a = 0; a < nA; ++a) pend[a] = 0u;
  pend[0] = 1u;
  for (int a = 0; a < nA; ++a) {
    while (pend[a] != 0u) {
      const int b = __ffs(pend[a]) - 1;
      pend[a] &= pend[a] - 1u;
      const SbNode& na = A[a];
      const SbNode& nb = B[b];
      double bmn[3], bmx[3];
      ++node_tests;
      xform_aabb(M, nb.c, nb.h, bmn, bmx);
      if (!overlaps(na.bmin, na.bmax, bmn, bmx)) continue;
      const bool la = na.child0 < 0, lb = nb.child0 < 0;
      if (la && lb) {
        for (int j = 0; j < nb.tri_count; ++j) {
          const double* tb = trisB[nb.tri_start + j].v;
          double q[9];
          xform(M, tb[0], tb[1], tb[2], q[0], q[1], q[2]);
          xform(M, tb[3], tb[4], tb[5], q[3], q[4], q[5]);
          xform(M, tb[6], tb[7], tb[8], q[6], q[7], q[8]);
          for (int i = 0; i < na.tri_count; ++i) {
            ++pair_tests;
            if (tri_tri_intersect(trisA[na.tri_start + i].v, q)) return true;
          }
        }
      } else {
        bool descend_a = lb;
        if (!descend_a && !la) {
          double e0 = bmx[0] - bmn[0], e1 = bmx[1] - bmn[1], e2 = bmx[2] - bmn[2];
          descend_a = na.ext2 >= (e0 * e0 + e1 * e1) + e2 * e2;
        }
        if (descend_a) {
          pend[na.child0] |= 1u << b;
          pend[na.child1] |= 1u << b;
        } else {
          pend[a] |= (1u << nb.child0) | (1u << nb.child1);
        }
      }
    }
  }
  return false;
}

// ------------------------------------------------------------------ occupancy grid
__device__ __forceinline__ int cell_of(double v, double v0, double inv, int g) {
  const double f = floor((v - v0) * inv);
  if (!(f >= 0.0)) return 0;  // also NaN
  return f >= (double)g ? g - 1 : (int)f;
}

// Cell range [cx0, cx1] x [cy0, cy1] of a world box (min xyz, max xyz).
__device__ __forceinline__ void cell_range(const SbCellGrid& G, const double* mn, const double* mx,
                                           int& cx0, int& cx1, int& cy0, int& cy1) {
  cx0 = cell_of(mn[0], G.x0, G.inv_x, G.g);
  cx1 = cell_of(mx[0], G.x0, G.inv_x, G.g);
  cy0 = cell_of(mn[1], G.y0, G.inv_y, G.g);
  cy1 = cell_of(mx[1], G.y0, G.inv_y, G.g);
}

// Set object `obj`'s bit in the cells its world box (min xyz, max xyz) meets. The words of
// up to 8 cells are loaded before any is stored (a plain load -> or -> store per cell
// would serialise on the possible aliasing; RED atomics measured slower: C4 +14 %).
__device__ __forceinline__ void cell_insert(const SbCellGrid& G, uint64_t inst, int32_t obj,
                                            const double* mn, const double* mx) {
  int cx0, cx1, cy0, cy1;
  cell_range(G, mn, mx, cx0, cx1, cy0, cy1);
  uint32_t* base = G.cells + inst * (uint64_t)(G.g * G.g) * G.words + (obj >> 5);
  const uint32_t bit = 1u << (obj & 31);
  const int nc = (cx1 - cx0 + 1) * (cy1 - cy0 + 1);
  int cx = cx0, cy = cy0;  // walked row by row (no division per cell)
  for (int c0 = 0; c0 < nc; c0 += 8) {
    uint32_t v[8];
    uint32_t* a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a[u] = base + (uint64_t)(cy * G.g + cx) * G.words;
      v[u] = c0 + u < nc ? *a[u] : 0u;
      if (++cx > cx1) {
        cx = cx0;
        ++cy;
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (c0 + u < nc) *a[u] = v[u] | bit;
  }
}

// ------------------------------------------------------------------ world view
using WorldView = SbWorldView;

struct CheckCounters {
  uint32_t narrow;  // candidate/object pairs past the AABB broad phase
  uint32_t pairs;   // triangle-pair predicate evaluations
  uint32_t broad;   // enabled objects examined by the broad phase
  uint32_t nodes;   // BVH node-pair box tests
};

// Store an accepted pose: record + world box (update_transform, collision.cpp:408-412).
__device__ __forceinline__ void store_pose(const WorldView& w, int32_t obj, uint64_t inst,
                                           const M34& P) {
  double2* pp = reinterpret_cast<double2*>(w.pose + sb_pose_off(w, obj, inst));
#pragma unroll
  for (int k = 0; k < 6; ++k) pp[k] = make_double2(P.m[2 * k], P.m[2 * k + 1]);
  const SbGeom g = w.geoms[w.obj_geom[obj]];
  double mn[3], mx[3];
  xform_aabb(P, g.box_c, g.box_h, mn, mx);
  double2* bp = reinterpret_cast<double2*>(w.box + sb_box_off(w, obj, inst));
  bp[0] = make_double2(mn[0], mn[1]);
  bp[1] = make_double2(mn[2], mx[0]);
  bp[2] = make_double2(mx[1], mx[2]);
}

// Column-major Mat4 (16 doubles) -> 3x4 row-major record.
__device__ __forceinline__ void from_colmajor(const double* c, M34& P) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) P.m[4 * i + j] = c[4 * j + i];
}

}  // namespace sbd
