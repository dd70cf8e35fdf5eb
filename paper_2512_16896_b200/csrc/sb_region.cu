// Warp-cooperative per-instance constraint regions (relationships.cpp:161-218 with
// polygon.cpp:136-176 annulus_sector, the rect-clip stand-in for Boost intersect, and
// polygon.cpp:260-388 triangulate + PolygonSampler), one 16-lane group per instance (two
// instances per warp), all on device.
//
// Lanes compute the arc points, the Sutherland-Hodgman passes (prefix-sum compaction
// preserves the sequential output order) and the fan triangles in parallel; every step
// whose rounding depends on evaluation order (ring areas, the tolerance-based duplicate
// drop, the cumulative-area table) runs on g.gl 0 in the reference's order, so tables are
// bit-identical to sbp::* (the single-thread restatement) and to the reference.
#include <stdexcept>
#include <string>

#include "../../include/scenebatch_b200.h"
#include "sb_crmath.cuh"
#include "sb_glibcm.cuh"
#include "sb_dev.cuh"
#include "sb_pdl.cuh"
#include "sb_poly.h"
#include "sb_region.h"

using namespace sbd;

namespace sbk {
namespace {

constexpr int kRB = 128;            // threads per block
constexpr int kG = 16;              // lanes per instance group: two instances per warp
constexpr int kRW = kRB / kG;       // groups per block
constexpr int kCap = sbp::kCap;
#ifndef SB_REGION_MIN_BLOCKS
#define SB_REGION_MIN_BLOCKS 8
#endif
constexpr int kRegionMinBlocks = SB_REGION_MIN_BLOCKS;  // resident blocks per SM (register cap)

// The lanes of one instance group and its collectives (kG-wide shuffles, ballots, votes).
struct Grp {
  int gl;          // g.gl within the group
  int base;        // the group's first lane in the warp
  unsigned mask;   // the group's lanes
  __device__ __forceinline__ Grp()
      : gl(threadIdx.x & (kG - 1)), base((threadIdx.x & 31) & ~(kG - 1)),
        mask((kG == 32 ? 0xffffffffu : ((1u << kG) - 1u)) << ((threadIdx.x & 31) & ~(kG - 1))) {}
  __device__ __forceinline__ unsigned ballot(bool p) const {
    return (__ballot_sync(mask, p) >> base) & (kG == 32 ? 0xffffffffu : ((1u << kG) - 1u));
  }
  template <class T>
  __device__ __forceinline__ T bcast(T v, int src) const { return __shfl_sync(mask, v, src, kG); }
  __device__ __forceinline__ bool any(bool p) const { return __any_sync(mask, p); }
  __device__ __forceinline__ bool all(bool p) const { return __all_sync(mask, p); }
  __device__ __forceinline__ void sync() const { __syncwarp(mask); }
};

// Optional stage cycle profile (build with -DSB_REGION_PROF): [0] anchor state, [1] band /
// direction / bounds, [2] arc points, [3] orientation + 4 clips, [4] dedupe + area,
// [5] triangulate + fan test, [6] sampler table, [7] instances.
__device__ unsigned long long g_rprof[8];
#ifdef SB_REGION_PROF
#define SB_RP_MARK(var) const long long var = clock64()
#define SB_RP_ADD(k, a, b) \
  if (g.gl == 0) atomicAdd(&g_rprof[k], (unsigned long long)((b) - (a)))
#else
#define SB_RP_MARK(var)
#define SB_RP_ADD(k, a, b)
#endif

// Two ring buffers per instance group; the triangle areas / cumulative sums of the fan
// reuse whichever buffer the final ring is not in (24.6 KB of shared memory per block).
struct RegionScratch {
  double x[2][kCap], y[2][kCap];
};

// ring_area (polygon.cpp:58-66): the shoelace terms in parallel, their sum on g.gl 0 in
// the reference's left-to-right order (bit-identical to sbp::ring_area). All lanes call;
// every g.gl gets the result.
__device__ __noinline__ double warp_ring_area(const double* x, const double* y, int n, double* tmp) {
  const Grp g;
  for (int i = g.gl; i < n; i += kG) {
    const int j = i + 1 == n ? 0 : i + 1;
    tmp[i] = x[i] * y[j] - x[j] * y[i];
  }
  g.sync();
  double s = 0.0;
  if (g.gl == 0) {
#pragma unroll 8
    for (int i = 0; i < n; ++i) s += tmp[i];
  }
  s = g.bcast(s, 0);
  g.sync();
  return 0.5 * s;
}

// Exclusive group prefix count of `flag` over lanes; returns this lane's offset.
__device__ __forceinline__ int lane_rank(const Grp& g, bool flag, int& total) {
  const unsigned m = g.ballot(flag);
  total = __popc(m);
  return __popc(m & ((1u << g.gl) - 1u));
}

// One Sutherland-Hodgman pass (same arithmetic and output order as sbp::clip_half);
// returns the output size, or -1 on overflow.
__device__ __noinline__ int warp_clip(const double* ix, const double* iy, int n, double* ox, double* oy,
                         int axis, double bound, bool keep_ge) {
  const Grp g;
  int base = 0;
  for (int i0 = 0; i0 < n; i0 += kG) {
    const int i = i0 + g.gl;
    int cnt = 0;
    bool ci = false, pi = false;
    double cx = 0, cy = 0, qx = 0, qy = 0;
    if (i < n) {
      const int ip = (i + n - 1) % n;
      const double cur_a = axis == 0 ? ix[i] : iy[i];
      const double prv_a = axis == 0 ? ix[ip] : iy[ip];
      ci = keep_ge ? cur_a >= bound : cur_a <= bound;
      pi = keep_ge ? prv_a >= bound : prv_a <= bound;
      if (ci != pi) {
        const double prv_o = axis == 0 ? iy[ip] : ix[ip];
        const double cur_o = axis == 0 ? iy[i] : ix[i];
        const double t = (bound - prv_a) / (cur_a - prv_a);
        const double o = prv_o + t * (cur_o - prv_o);
        qx = axis == 0 ? bound : o;
        qy = axis == 0 ? o : bound;
        ++cnt;
      }
      if (ci) {
        cx = ix[i];
        cy = iy[i];
        ++cnt;
      }
    }
    // exclusive prefix of cnt across the group
    int incl = cnt;
#pragma unroll
    for (int d = 1; d < kG; d <<= 1) {
      const int v = __shfl_up_sync(g.mask, incl, d, kG);
      if (g.gl >= d) incl += v;
    }
    const int total = g.bcast(incl, kG - 1);
    int pos = base + incl - cnt;
    if (base + total <= kCap && i < n) {
      if (ci != pi) {
        ox[pos] = qx;
        oy[pos] = qy;
        ++pos;
      }
      if (ci) {
        ox[pos] = cx;
        oy[pos] = cy;
      }
    }
    base += total;
  }
  g.sync();
  return base <= kCap ? base : -1;
}

struct RegionStats {
  int status;  // sbp::RegionStatus
  int ntri;
};

// distance_band (relationships.cpp:101-122)
__device__ __forceinline__ void distance_band(const SbPlacementDev& pl, double& min_r, double& max_r) {
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  min_r = 0.0;
  max_r = inf;
  if (pl.distance_type == SB_DIST_GREATER) {
    min_r = pl.distance;
  } else if (pl.distance_type == SB_DIST_LESS) {
    max_r = pl.distance;
  } else if (pl.distance_type == SB_DIST_EQUAL) {
    const double half = dmax(0.05 * pl.distance, 0.01);
    min_r = dmax(0.0, pl.distance - half);
    max_r = pl.distance + half;
  }
}
// RelationshipSpec::effective_angle_threshold
__device__ __forceinline__ double region_theta(const SbPlacementDev& pl) {
  const double pi = 3.14159265358979323846;
  return pl.angle_threshold > 0.0 ? pl.angle_threshold
                                  : (pl.direction == SB_DIR_NONE ? pi : pi / 4.0);
}
// resolve_direction (relationships.cpp:78-99); (1, 0) without a direction
__device__ __forceinline__ void resolve_direction(const SbPlacementDev& pl, double ayaw, double& vx,
                                                  double& vy) {
  vx = 1.0;
  vy = 0.0;
  if (pl.direction == SB_DIR_NONE) return;
  switch (pl.direction) {
    case SB_DIR_LEFT: vx = -1; vy = 0; break;
    case SB_DIR_RIGHT: vx = 1; vy = 0; break;
    case SB_DIR_FRONT: vx = 0; vy = -1; break;
    case SB_DIR_BACK: vx = 0; vy = 1; break;
    default: {
      const double nrm = sqrt(pl.direction_vector[0] * pl.direction_vector[0] +
                              pl.direction_vector[1] * pl.direction_vector[1]);
      vx = pl.direction_vector[0] / nrm;
      vy = pl.direction_vector[1] / nrm;
    }
  }
  if (pl.frame == SB_FRAME_LOCAL) {
    double c, s;
    sbg::sincos(ayaw, &s, &c);
    const double nx = c * vx - s * vy, ny = s * vx + c * vy;
    vx = nx;
    vy = ny;
  }
}

__device__ __forceinline__ int arc_count(double a0, double a1) {
  const double step = 5.0 * 3.14159265358979323846 / 180.0;
  const int n = (int)ceil(fabs(a1 - a0) / step);
  return n < 1 ? 1 : n;
}
// arc k's endpoints for direction (vx, vy); false if there is no arc k
__device__ __forceinline__ bool arc_ends(const SbPlacementDev& pl, double vx, double vy, int k,
                                         double& a0, double& a1) {
  const double pi = 3.14159265358979323846;
  const double theta = region_theta(pl);
  double min_r, max_r;
  distance_band(pl, min_r, max_r);
  if (theta >= pi - 1e-12) {  // full: one circle (the hole case has its own kernel)
    a0 = 0.0;
    a1 = 2.0 * pi;
    return k == 0;
  }
  const double base = sbg::atan2(vy, vx);
  if (k == 0) {
    a0 = base - theta;
    a1 = base + theta;
    return true;
  }
  a0 = base + theta;
  a1 = base - theta;
  return min_r > 0.0;
}
// Region for one anchor state into (tris, cum) with capacity `cap`. All lanes call.
// arcs: the placement's shared arc table (arc_table_host), or NULL when the arcs depend on
// the anchor yaw.
__device__ RegionStats warp_region(const SbPlacementDev& pl, double ax, double ay, double ayaw,
                                   SbRegionTri* tris, double* cum, int cap, RegionScratch& sc,
                                   const SbArcTable* arcs) {
  const Grp g;
  SB_RP_MARK(rp0);
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double min_r, max_r;
  distance_band(pl, min_r, max_r);
  const double pi = 3.14159265358979323846;
  const double theta = region_theta(pl);
  double vx, vy;
  if (!arcs) resolve_direction(pl, ayaw, vx, vy);  // only the arcs need the direction
  // clip bound = bounds(support) expanded by the anchor; only used for infinite max_r
  const double* rc = pl.rect;
  double bx0 = inf, by0 = inf, bx1 = -inf, by1 = -inf;
  const double vxs[5] = {rc[0], rc[2], rc[2], rc[0], ax};
  const double vys[5] = {rc[1], rc[1], rc[3], rc[3], ay};
  for (int k = 0; k < 5; ++k) {
    bx0 = dmin(bx0, vxs[k]);
    by0 = dmin(by0, vys[k]);
    bx1 = dmax(bx1, vxs[k]);
    by1 = dmax(by1, vys[k]);
  }
  const double ddx = bx1 - bx0, ddy = by1 - by0;
  const double diag = bx0 > bx1 ? 0.0 : sqrt(ddx * ddx + ddy * ddy);

  SB_RP_MARK(rp1);
  SB_RP_ADD(1, rp0, rp1);
  // ---- annulus_sector (polygon.cpp:136-176), arc points in parallel
  if (!(theta > 0.0) || theta > pi + 1e-12) return {sbp::kRegionBadArg, 0};
  if (isinf(max_r)) max_r = fmax(diag, min_r + 1e-6);
  if (!(min_r < max_r)) return {sbp::kRegionBadArg, 0};
  const bool full = theta >= pi - 1e-12;
  if (full && min_r > 0.0) return {sbp::kRegionBadArg, 0};  // hole: k_relation_regions<true>
  double* X = sc.x[0];
  double* Y = sc.y[0];
  int n = 0;
  auto arc = [&](int k, double radius, int off) -> int {
    double a0 = 0.0, a1 = 0.0;
    int na;
    if (arcs) {
      na = __ldg(&arcs->na[k]);
    } else {
      arc_ends(pl, vx, vy, k, a0, a1);
      na = arc_count(a0, a1);
    }
    if (off + na + 1 > kCap) return -1;
    for (int i = g.gl; i <= na; i += kG) {
      double sa, ca;
      if (arcs) {
        ca = __ldg(&arcs->c[k][i]);
        sa = __ldg(&arcs->s[k][i]);
      } else {
        const double a = a0 + (a1 - a0) * (double)i / (double)na;
        sbg::sincos(a, &sa, &ca);
      }
      X[off + i] = ax + radius * ca;
      Y[off + i] = ay + radius * sa;
    }
    return off + na + 1;
  };
  if (full) {
    n = arc(0, max_r, 0);
    if (n < 0) return {sbp::kRegionOverflow, 0};
    n -= 1;
  } else {
    n = arc(0, max_r, 0);
    if (n < 0) return {sbp::kRegionOverflow, 0};
    if (min_r > 0.0) {
      n = arc(1, min_r, n);
      if (n < 0) return {sbp::kRegionOverflow, 0};
    } else {
      if (n + 1 > kCap) return {sbp::kRegionOverflow, 0};
      if (g.gl == 0) {
        X[n] = ax;
        Y[n] = ay;
      }
      ++n;
    }
  }
  g.sync();

  SB_RP_MARK(rp2);
  SB_RP_ADD(2, rp1, rp2);
  // ---- intersect with the support rect (oracle Boost stand-in): correct() orientation
  if (n < 3) return {sbp::kRegionEmpty, 0};
  const double ar = warp_ring_area(X, Y, n, sc.x[1]);
  if (ar < 0.0) {  // reverse the closed ring: p0 stays first
    for (int i = 1 + g.gl; i < n - i; i += kG) {
      const int j = n - i;
      const double tx = X[i], ty = Y[i];
      X[i] = X[j];
      Y[i] = Y[j];
      X[j] = tx;
      Y[j] = ty;
    }
    g.sync();
  }
  const double x0 = fmin(rc[0], rc[2]), x1 = fmax(rc[0], rc[2]);
  const double y0 = fmin(rc[1], rc[3]), y1 = fmax(rc[1], rc[3]);
  // Sutherland-Hodgman passes x >= x0, x <= x1, y >= y0, y <= y1. A pass that keeps every
  // vertex outputs its input unchanged (no crossings, same order), so it is skipped; the
  // ring stays in buffer cb.
  int cb = 0;
  auto pass = [&](int axis, double bound, bool keep_ge) {
    if (n < 0) return;
    bool inside = true;
    for (int i = g.gl; i < n; i += kG) {
      const double a = axis == 0 ? sc.x[cb][i] : sc.y[cb][i];
      if (!(keep_ge ? a >= bound : a <= bound)) inside = false;
    }
    if (g.all(inside)) return;
    n = warp_clip(sc.x[cb], sc.y[cb], n, sc.x[cb ^ 1], sc.y[cb ^ 1], axis, bound, keep_ge);
    cb ^= 1;
  };
  pass(0, x0, true);
  pass(0, x1, false);
  pass(1, y0, true);
  pass(1, y1, false);
  if (n < 0) return {sbp::kRegionOverflow, 0};
  X = sc.x[cb];
  Y = sc.y[cb];
  SB_RP_MARK(rp3);
  SB_RP_ADD(3, rp2, rp3);
  // drop consecutive exact duplicates (keep the first of each run; == is transitive, so
  // comparing with the previous vertex equals comparing with the last kept one), then
  // trailing copies of vertex 0. Out of place: buffer cb -> buffer cb ^ 1.
  double* X1 = sc.x[cb ^ 1];
  double* Y1 = sc.y[cb ^ 1];
  double* const FA = sc.x[cb];  // free once the ring is copied out: fan areas
  double* const FC = sc.y[cb];  // and cumulative sums
  int m = 0;
  for (int i0 = 0; i0 < n; i0 += kG) {
    const int i = i0 + g.gl;
    bool keep = false;
    double xi = 0.0, yi = 0.0;
    if (i < n) {
      xi = X[i];
      yi = Y[i];
      keep = i == 0 || xi != X[i - 1] || yi != Y[i - 1];
    }
    int tot;
    const int r = lane_rank(g, keep, tot);
    if (keep) {
      X1[m + r] = xi;
      Y1[m + r] = yi;
    }
    m += tot;
  }
  g.sync();
  if (g.gl == 0)
    while (m > 1 && X1[0] == X1[m - 1] && Y1[0] == Y1[m - 1]) --m;
  m = g.bcast(m, 0);
  double area1 = 0.0;
  if (m >= 3) {
    area1 = warp_ring_area(X1, Y1, m, FA);
    if (area1 == 0.0) m = 0;
  }
  if (m < 3) return {sbp::kRegionEmpty, 0};
  if (pl.erode_r > 0.0) {
    // apply_ratio_on_support -> erode (relationships.cpp:220-230, polygon.cpp:101-113) as the
    // oracle's Boost stand-in defines buffer(-r) on a convex ring (sbh::erode_convex): lane i
    // rebuilds the offset lines of edges i-1 and i and intersects them.
    const double r = pl.erode_r;
    bool convex = true;
    for (int i = g.gl; i < m; i += kG) {
      const int h = i == 0 ? m - 1 : i - 1, q = i + 1 == m ? 0 : i + 1;
      const double ox = X1[h], oy = Y1[h], px = X1[i], py = Y1[i], qx = X1[q], qy = Y1[q];
      if ((px - ox) * (qy - oy) - (py - oy) * (qx - ox) < 0.0) convex = false;
      const double dxh = px - ox, dyh = py - oy, dxi = qx - px, dyi = qy - py;
      const double lh = sqrt(dxh * dxh + dyh * dyh), li = sqrt(dxi * dxi + dyi * dyi);
      const double axh = ox + (-dyh / lh) * r, ayh = oy + (dxh / lh) * r;
      const double axi = px + (-dyi / li) * r, ayi = py + (dxi / li) * r;
      const double den = dxh * dyi - dyh * dxi;
      const double t = ((axi - axh) * dyi - (ayi - ayh) * dxi) / den;
      FA[i] = axh + t * dxh;
      FC[i] = ayh + t * dyh;
    }
    if (!g.all(convex)) return {sbp::kRegionBadArg, 0};  // concave region: out of scope
    g.sync();
    bool alive = true;  // every offset edge keeps its direction, else eroded away
    for (int i = g.gl; i < m; i += kG) {
      const int q = i + 1 == m ? 0 : i + 1;
      if (!((FA[q] - FA[i]) * (X1[q] - X1[i]) + (FC[q] - FC[i]) * (Y1[q] - Y1[i]) > 0.0))
        alive = false;
    }
    if (!g.all(alive)) return {sbp::kRegionEmpty, 0};
    g.sync();
    for (int i = g.gl; i < m; i += kG) {
      X1[i] = FA[i];
      Y1[i] = FC[i];
    }
    g.sync();
    area1 = warp_ring_area(X1, Y1, m, FA);
  }

  SB_RP_MARK(rp4);
  SB_RP_ADD(4, rp3, rp4);
  // ---- triangulate (polygon.cpp:344-368) + ear_clip_ring (:260-340): orientation (same
  // ring, same area), tolerance-based duplicate drop, then the fan fast path
  if (area1 < 0.0) {
    for (int i = g.gl; i < m - 1 - i; i += kG) {
      const int j = m - 1 - i;
      const double tx = X1[i], ty = Y1[i];
      X1[i] = X1[j];
      Y1[i] = Y1[j];
      X1[j] = tx;
      Y1[j] = ty;
    }
    g.sync();
  }
  // The drop compares each vertex with the last KEPT one (not transitive): if no
  // consecutive pair is within tolerance nothing is dropped; otherwise g.gl 0 runs the
  // sequential loop.
  bool close = false;
  for (int i = 1 + g.gl; i < m; i += kG) {
    const double dx = X1[i] - X1[i - 1], dy = Y1[i] - Y1[i - 1];
    if (!(dx * dx + dy * dy > 1e-24)) close = true;
  }
  int k = m;
  if (g.any(close)) {
    if (g.gl == 0) {
      k = 0;
      for (int i = 0; i < m; ++i) {
        if (k > 0) {
          const double dx = X1[i] - X1[k - 1], dy = Y1[i] - Y1[k - 1];
          if (!(dx * dx + dy * dy > 1e-24)) continue;
        }
        X1[k] = X1[i];
        Y1[k] = Y1[i];
        ++k;
      }
    }
    k = g.bcast(k, 0);
    g.sync();
  }
  if (g.gl == 0) {
    while (k > 1) {
      const double dx = X1[0] - X1[k - 1], dy = Y1[0] - Y1[k - 1];
      if (dx * dx + dy * dy <= 1e-24) --k;
      else break;
    }
  }
  k = g.bcast(k, 0);
  g.sync();
  X = X1;
  Y = Y1;
  if (k < 3) return {sbp::kRegionOk, 0};  // valid() == false -> placeable = 0
  bool ok = true;
  for (int i = g.gl; i < k; i += kG) {
    const int a = i == 0 ? k - 1 : i - 1, c = i + 1 == k ? 0 : i + 1;
    if (sbp::cross2(X[a], Y[a], X[i], Y[i], X[c], Y[c]) < 0.0) ok = false;
    if (i + 3 < k) {
      const double cr = sbp::cross2(X[k - 1], Y[k - 1], X[i], Y[i], X[i + 1], Y[i + 1]);
      if (cr < 0.0 || fabs(cr) < 1e-18) ok = false;
    }
  }
  const bool fan = g.all(ok);
  SB_RP_MARK(rp5);
  SB_RP_ADD(5, rp4, rp5);
  int ntri = 0;
  if (fan) {
    // triangle i = (k-1, i, i+1); keep area > 0 (PolygonSampler ctor, polygon.cpp:374-375):
    // areas and output slots in parallel, the running total on g.gl 0 in order, the
    // normalisation (polygon.cpp:381-387) in parallel again.
    const int nt = k - 2;
    int slot[(kCap + kG - 1) / kG];
    for (int i0 = 0, c = 0; i0 < nt; i0 += kG, ++c) {
      const int i = i0 + g.gl;
      double a = 0.0;
      if (i < nt) a = 0.5 * fabs(sbp::cross2(X[k - 1], Y[k - 1], X[i], Y[i], X[i + 1], Y[i + 1]));
      int tot;
      const int r = lane_rank(g, a > 0.0, tot);
      slot[c] = a > 0.0 ? ntri + r : -1;
      if (a > 0.0) FA[ntri + r] = a;
      ntri += tot;
    }
    g.sync();
    if (ntri > cap) return {sbp::kRegionOverflow, 0};
    double total = 0.0;
    if (g.gl == 0) {
#pragma unroll 8
      for (int j = 0; j < ntri; ++j) {
        total += FA[j];
        FC[j] = total;
      }
    }
    total = g.bcast(total, 0);
    g.sync();
    if (ntri > 0 && !(total > 0.0)) ntri = 0;
    for (int i0 = 0, c = 0; i0 < nt; i0 += kG, ++c) {
      const int i = i0 + g.gl;
      const int j = slot[c];
      if (i < nt && j >= 0 && ntri > 0) {
        SbRegionTri& t = tris[j];
        t.a[0] = X[k - 1];
        t.a[1] = Y[k - 1];
        t.b[0] = X[i];
        t.b[1] = Y[i];
        t.c[0] = X[i + 1];
        t.c[1] = Y[i + 1];
        cum[j] = j == ntri - 1 ? 1.0 : FC[j] / total;
      }
    }
  } else if (g.gl == 0) {  // general ear clipping (reflex or sliver corners): restatement
    sbp::Ring r;
    r.n = k;
    for (int i = 0; i < k; ++i) {
      r.x[i] = X[i];
      r.y[i] = Y[i];
    }
    sbp::TableSink sink{tris, cum, 0, cap, 0.0};
    if (!sbp::ear_clip_into(r, sink)) ntri = -1;
    else ntri = sbp::finish_table(sink);
  }
  ntri = g.bcast(ntri, 0);
  g.sync();
  if (ntri < 0) return {sbp::kRegionOverflow, 0};
  SB_RP_MARK(rp6);
  SB_RP_ADD(6, rp5, rp6);
  SB_RP_ADD(7, 0, 1);
  return {sbp::kRegionOk, ntri};
}

// libm policy of the hole path on the device: the correctly rounded sin/cos/atan2.
struct DevMath {
  __device__ static void sincos(double a, double* s, double* c) { sbg::sincos(a, s, c); }
  __device__ static double atan2(double y, double x) { return sbg::atan2(y, x); }
};

// Shapes whose ring outgrows the group path's kCap -- the full annulus with a hole (theta =
// pi, min_r > 0) and wide annular sectors: one lane per instance runs the restated pipeline
// (sbp::hole_annulus_table / sbp::big_region_table) on 2 * kCap + 2 vertex rings in local
// memory; such rings are never convex, so the lane-parallel fan path would not apply.
__device__ __noinline__ RegionStats big_region_lane(const SbPlacementDev& pl, double ax, double ay,
                                                    double ayaw, const double* mx, const double* my,
                                                    SbRegionTri* tris, double* cum, int cap) {
  const sbp::SupportClip clip{pl.rect, pl.poly_n, pl.poly_x, pl.poly_y};
  sbp::TableSink sink{tris, cum, 0, cap, 0.0};
  if (pl.distance_type == SB_DIST_MIDDLE) {  // relationships.cpp:192-196
    sbp::Ring r, tmp;
    const int st = sbp::middle_region_table<DevMath>(mx, my, pl.n_anchors, clip, pl.erode_r, r, tmp, sink);
    if (st != sbp::kRegionOk) return {st, 0};
    return {sbp::kRegionOk, sbp::finish_table(sink)};
  }
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double min_r, max_r;
  distance_band(pl, min_r, max_r);
  const double pi = 3.14159265358979323846;
  const double theta = region_theta(pl);
  double vx, vy;
  resolve_direction(pl, ayaw, vx, vy);
  // clip bound = bounds(support) expanded by the anchor (relationships.cpp:188-203)
  const double* bd = pl.bounds;
  const double bx0 = dmin(bd[0], ax), by0 = dmin(bd[1], ay);
  const double bx1 = dmax(bd[2], ax), by1 = dmax(bd[3], ay);
  const double ddx = bx1 - bx0, ddy = by1 - by0;
  const double diag = bx0 > bx1 ? 0.0 : sqrt(ddx * ddx + ddy * ddy);
  (void)inf;
  if (!(theta > 0.0) || theta > pi + 1e-12) return {sbp::kRegionBadArg, 0};
  if (isinf(max_r)) max_r = fmax(diag, min_r + 1e-6);
  if (!(min_r < max_r)) return {sbp::kRegionBadArg, 0};
  sbp::HoleScratch sc;
  const bool full = theta >= pi - 1e-12;
  int st;
  if (full && min_r > 0.0) {
    st = sbp::hole_annulus_table<DevMath>(ax, ay, min_r, max_r, clip, pl.erode_r, sc, sink);
  } else {
    st = sbp::big_region_table<DevMath>(ax, ay, vx, vy, theta, min_r, max_r, clip, pl.erode_r,
                                        sc, sink);
  }
  if (st != sbp::kRegionOk) return {st, 0};
  return {sbp::kRegionOk, sbp::finish_table(sink)};
}

// Group-level dispatch: the hole path on lane 0, broadcast to the group.
template <bool kHole>
__device__ __forceinline__ RegionStats group_region(const SbPlacementDev& pl, double ax, double ay,
                                                    double ayaw, SbRegionTri* tris, double* cum,
                                                    int cap, RegionScratch& sc,
                                                    const SbArcTable* arcs,
                                                    const double* mx = nullptr,
                                                    const double* my = nullptr) {
  if constexpr (kHole) {
    const Grp g;
    RegionStats r{0, 0};
    if (g.gl == 0) r = big_region_lane(pl, ax, ay, ayaw, mx, my, tris, cum, cap);
    r.status = g.bcast(r.status, 0);
    r.ntri = g.bcast(r.ntri, 0);
    return r;
  } else {
    return warp_region(pl, ax, ay, ayaw, tris, cum, cap, sc, arcs);
  }
}

// Warp per local instance: anchor state in the support frame (inverse_rigid(support) *
// anchor pose, yaw_of), the variation test against instance 0 (relationships.cpp:178-186)
// and the region table. Instance 0's state comes from `s0` (sharded runs) or, when this
// shard owns global instance 0, is recomputed per warp from local instance 0.
template <bool kHole>
__global__ void __launch_bounds__(kRB, kRegionMinBlocks) k_relation_regions(RelationRegionParams p) {
  pdl_enter();
  __shared__ RegionScratch scratch[kRW];
  const SbArcTable* arcs = kHole ? nullptr : p.arcs;
  const Grp g;
  const uint64_t warp = (blockIdx.x * (uint64_t)kRB + threadIdx.x) / kG;  // instance group
  const uint64_t nwarps = (uint64_t)gridDim.x * kRW;
  RegionScratch& sc = scratch[threadIdx.x / kG];
  M34 inv;
#pragma unroll
  for (int k = 0; k < 12; ++k) inv.m[k] = p.inv_support[k];
  // Anchor position (and, only when it can matter, yaw) in the support frame. The yaw
  // feeds a local-frame direction and the variation test; the latter only needs it when
  // the positions agree (relationships.cpp:180-181), so atan2 is skipped otherwise.
  const bool yaw_used = p.pl.direction != SB_DIR_NONE && p.pl.frame == SB_FRAME_LOCAL;
  auto rel_of = [&](int32_t obj, uint64_t inst, M34& rel) {  // inverse_rigid(support_world[i]) * anchor pose
    const double* pp = p.w.pose + sb_pose_off(p.w, obj, inst);
    M34 P;
#pragma unroll
    for (int k = 0; k < 12; ++k) P.m[k] = pp[k];
    if (p.pl.inv_support_inst) {
      M34 Ii;
#pragma unroll
      for (int k = 0; k < 12; ++k) Ii.m[k] = p.pl.inv_support_inst[inst * 12 + k];
      mul34(Ii, P, rel);
    } else {
      mul34(inv, P, rel);
    }
  };
  auto yaw_of = [](const M34& rel) { return sbg::atan2(rel.m[4], rel.m[0]); };  // transform.hpp:77
  // several anchors (middle, or the multi-anchor variation test) take the serial path
  const int na = kHole && p.pl.n_anchors > 1 ? p.pl.n_anchors : 1;
  if (p.from_s0) {  // canonical region_for(0) from the exchanged instance-0 states
    if (warp == 0) {
      double mx[SB_MAX_ANCHORS], my[SB_MAX_ANCHORS];
      for (int k = 0; k < na; ++k) {
        mx[k] = p.s0[3 * k];
        my[k] = p.s0[3 * k + 1];
      }
      const RegionStats r = group_region<kHole>(p.pl, p.s0[0], p.s0[1], p.s0[2], p.tris, p.cum,
                                                p.cap, sc, arcs, mx, my);
      if (g.gl == 0) {
        const bool good = r.status == sbp::kRegionOk || r.status == sbp::kRegionEmpty;
        p.ntri[0] = good ? r.ntri : 0;
        if (!good) atomicMax(p.flags + 1, r.status);
      }
    }
    return;
  }
  if (p.states) {  // AnchorState batch given directly (build_constraint_region's input)
    const double x0 = p.states[0], y0 = p.states[1], yaw0 = p.states[2];
    bool vary = false;
    int worst = 0;
    for (uint64_t i = warp; i < p.w.n; i += nwarps) {
      const double ax = p.states[3 * i], ay = p.states[3 * i + 1], ayaw = p.states[3 * i + 2];
      const double dx = ax - x0, dy = ay - y0;  // relationships.cpp:178-186
      vary = vary || sqrt(dx * dx + dy * dy) > 1e-12 || fabs(ayaw - yaw0) > 1e-12;
      const RegionStats r = group_region<kHole>(p.pl, ax, ay, ayaw, p.tris + i * p.cap,
                                                p.cum + i * p.cap, p.cap, sc, arcs);
      if (g.gl == 0) {
        p.ntri[i] = r.status == sbp::kRegionOk || r.status == sbp::kRegionEmpty ? r.ntri : 0;
        if (r.status != sbp::kRegionOk && r.status != sbp::kRegionEmpty && r.status > worst)
          worst = r.status;
      }
    }
    if (g.gl == 0) {
      if (vary) atomicOr(p.flags + 0, 1);
      if (worst) atomicMax(p.flags + 1, worst);
    }
    return;
  }
  // instance 0's anchor states: recomputed from local instance 0, or exchanged (s0)
  double x0[SB_MAX_ANCHORS], y0[SB_MAX_ANCHORS];
  M34 rel0;
  for (int k = 0; k < na; ++k) {
    if (p.owns_instance0) {
      rel_of(p.pl.anchor_objects[k], 0, rel0);
      x0[k] = rel0.m[3];
      y0[k] = rel0.m[7];
    } else {
      x0[k] = p.s0[3 * k];
      y0[k] = p.s0[3 * k + 1];
    }
  }
  auto yaw0_of = [&](int k) {
    if (!p.owns_instance0) return p.s0[3 * k + 2];
    M34 r0;
    rel_of(p.pl.anchor_objects[k], 0, r0);
    return yaw_of(r0);
  };
  bool vary = false;
  int worst = 0;
  for (uint64_t i = warp; i < p.w.n; i += nwarps) {
    SB_RP_MARK(ra0);
    double ax = 0.0, ay = 0.0, ayaw = 0.0;
    double mx[SB_MAX_ANCHORS], my[SB_MAX_ANCHORS];
    for (int k = 0; k < na; ++k) {  // relationships.cpp:178-186, every anchor
      M34 rel;
      rel_of(p.pl.anchor_objects[k], i, rel);
      const double kx = rel.m[3], ky = rel.m[7];
      const double dx = kx - x0[k], dy = ky - y0[k];
      const bool pos_vary = sqrt(dx * dx + dy * dy) > 1e-12;
      double kyaw = 0.0;
      if ((k == 0 && yaw_used) || !pos_vary) kyaw = yaw_of(rel);
      if (!pos_vary && !vary) vary = fabs(kyaw - yaw0_of(k)) > 1e-12;
      vary = vary || pos_vary;
      mx[k] = kx;
      my[k] = ky;
      if (k == 0) {
        ax = kx;
        ay = ky;
        ayaw = kyaw;
      }
    }
    SB_RP_MARK(ra1);
    SB_RP_ADD(0, ra0, ra1);
    const RegionStats r = group_region<kHole>(p.pl, ax, ay, ayaw, p.tris + i * p.cap,
                                              p.cum + i * p.cap, p.cap, sc, arcs, mx, my);
    if (g.gl == 0) {
      p.ntri[i] = r.status == sbp::kRegionOk || r.status == sbp::kRegionEmpty ? r.ntri : 0;
      if (r.status != sbp::kRegionOk && r.status != sbp::kRegionEmpty && r.status > worst)
        worst = r.status;
    }
  }
  if (g.gl == 0) {
    if (vary) atomicOr(p.flags + 0, 1);
    if (worst) atomicMax(p.flags + 1, worst);
  }
}

}  // namespace

void region_profile(unsigned long long out[8], bool reset) {
  if (cudaMemcpyFromSymbol(out, g_rprof, 8 * sizeof(unsigned long long)) != cudaSuccess)
    throw std::runtime_error("region_profile");
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (cudaMemcpyToSymbol(g_rprof, z, sizeof z) != cudaSuccess) throw std::runtime_error("region_profile reset");
  }
}

void relation_regions(const RelationRegionParams& p, int num_sms, sb_stream_t s) {
  unsigned blocks = (unsigned)((p.w.n + kRW - 1) / kRW);
  const unsigned cap_blocks = (unsigned)(num_sms * 16);
  if (blocks > cap_blocks) blocks = cap_blocks;
  if (blocks == 0) blocks = 1;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
  if (p.hole) launch_pdl(k_relation_regions<true>, blocks, kRB, 0, st, p);
  else launch_pdl(k_relation_regions<false>, blocks, kRB, 0, st, p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("relation_regions: ") + cudaGetErrorString(e));
}

}  // namespace sbk
