// Constraint-region polygon pipeline, shared by host preparation (g++) and the
// per-instance region kernel (nvcc): annulus sector -> clip to the support rect ->
// ear-clipping triangulation -> exact-uniform sampler table -> draw.
//
// Each function restates the reference operation by operation (no FMA: host built with
// -ffp-contract=off, device with -fmad=false) so a region built here is bit-identical to
// the reference's, up to the libm used for sin/cos/atan2.
// Fixed-capacity arrays (SB_REGION_MAX_VERTS) keep it allocation-free on the device.
#pragma once

#include <math.h>
#include <stdint.h>

#include "sb_layout.h"

#ifdef __CUDACC__
#define SB_HD __host__ __device__ __forceinline__
#else
#define SB_HD inline
#endif

namespace sbp {

constexpr double kPi = 3.14159265358979323846;  // M_PI
constexpr int kCap = SB_REGION_MAX_VERTS;

template <int Cap>
struct RingT {
  static constexpr int cap = Cap;
  double x[Cap];
  double y[Cap];
  int n;
};
using Ring = RingT<kCap>;
// Merged ring of an annulus clipped to a rect with its hole bridged in
// (bridge_hole, polygon.cpp:197-258): outer + hole + 2 bridge vertices.
constexpr int kHoleCap = 2 * kCap + 2;
using HoleRing = RingT<kHoleCap>;

enum RegionStatus { kRegionOk = 0, kRegionEmpty = 1, kRegionOverflow = 2, kRegionBadArg = 3 };

// cross2 (polygon.cpp:54-56)
SB_HD double cross2(double ox, double oy, double ax, double ay, double bx, double by) {
  return (ax - ox) * (by - oy) - (ay - oy) * (bx - ox);
}

// ring_area (polygon.cpp:58-66); shoelace, left to right.
template <int Cap>
SB_HD double ring_area(const RingT<Cap>& r) {
  double s = 0.0;
  for (int i = 0; i < r.n; ++i) {
    int j = (i + 1) % r.n;
    s += r.x[i] * r.y[j] - r.x[j] * r.y[i];
  }
  return 0.5 * s;
}

template <int Cap>
SB_HD void reverse_ring(RingT<Cap>& r) {
  for (int i = 0, j = r.n - 1; i < j; ++i, --j) {
    double tx = r.x[i], ty = r.y[i];
    r.x[i] = r.x[j];
    r.y[i] = r.y[j];
    r.x[j] = tx;
    r.y[j] = ty;
  }
}

template <int Cap>
SB_HD bool push(RingT<Cap>& r, double x, double y) {
  if (r.n >= Cap) return false;
  r.x[r.n] = x;
  r.y[r.n] = y;
  ++r.n;
  return true;
}

// annulus_sector (polygon.cpp:136-176) for the non-full case and the full disc without
// a hole. clip_diag = clip_bound.diagonal() (only used when max_r is infinite).
SB_HD int annulus_sector(double cx, double cy, double vx, double vy, double theta, double min_r,
                         double max_r, double clip_diag, Ring& out) {
  out.n = 0;
  if (!(theta > 0.0) || theta > kPi + 1e-12) return kRegionBadArg;
  if (isinf(max_r)) max_r = fmax(clip_diag, min_r + 1e-6);
  if (!(min_r < max_r)) return kRegionBadArg;
  double base = atan2(vy, vx);
  bool full = theta >= kPi - 1e-12;
  double step = 5.0 * kPi / 180.0;
  auto arc = [&](double radius, double a0, double a1) -> bool {
    double span = fabs(a1 - a0) / step;
    int n = (int)ceil(span);
    if (n < 1) n = 1;
    for (int i = 0; i <= n; ++i) {
      double a = a0 + (a1 - a0) * (double)i / (double)n;
      if (!push(out, cx + radius * cos(a), cy + radius * sin(a))) return false;
    }
    return true;
  };
  if (full) {
    if (min_r > 0.0) return kRegionBadArg;  // annulus with a hole: not on the device path
    if (!arc(max_r, 0.0, 2.0 * kPi)) return kRegionOverflow;
    out.n -= 1;  // closing vertex
    return kRegionOk;
  }
  if (!arc(max_r, base - theta, base + theta)) return kRegionOverflow;
  if (min_r > 0.0) {
    if (!arc(min_r, base + theta, base - theta)) return kRegionOverflow;
  } else {
    if (!push(out, cx, cy)) return kRegionOverflow;
  }
  return kRegionOk;
}

// One Sutherland-Hodgman pass against an axis-aligned half plane; the stand-in for
// Boost intersection documented in oracle/shim/boost/geometry.hpp (same operation order).
template <int Cap>
SB_HD bool clip_half(const RingT<Cap>& in, RingT<Cap>& out, int axis, double bound, bool keep_ge) {
  out.n = 0;
  int n = in.n;
  for (int i = 0; i < n; ++i) {
    int ip = (i + n - 1) % n;
    double cur_a = axis == 0 ? in.x[i] : in.y[i];
    double prv_a = axis == 0 ? in.x[ip] : in.y[ip];
    bool ci = keep_ge ? cur_a >= bound : cur_a <= bound;
    bool pi = keep_ge ? prv_a >= bound : prv_a <= bound;
    if (ci != pi) {
      double prv_o = axis == 0 ? in.y[ip] : in.x[ip];
      double cur_o = axis == 0 ? in.y[i] : in.x[i];
      double t = (bound - prv_a) / (cur_a - prv_a);
      double o = prv_o + t * (cur_o - prv_o);
      bool ok = axis == 0 ? push(out, bound, o) : push(out, o, bound);
      if (!ok) return false;
    }
    if (ci && !push(out, in.x[i], in.y[i])) return false;
  }
  return true;
}

// intersect(ring, rect) as the oracle stand-in defines it: correct() orientation,
// 4 half-plane passes (x>=x0, x<=x1, y>=y0, y<=y1), drop consecutive exact duplicates,
// discard < 3 vertices or zero area. Result in `r` (open ring). Uses `tmp` as scratch.
// hole: correct() orients holes clockwise instead of counter-clockwise.
template <int Cap>
SB_HD int intersect_rect(RingT<Cap>& r, RingT<Cap>& tmp, const double rect[4], bool hole = false) {
  if (r.n < 3) return kRegionEmpty;
  // bg::correct (via to_boost, polygon.cpp:27-36) reverses the CLOSED ring, which keeps
  // vertex 0 first: [p0, p(n-1), ..., p1].
  if (hole ? ring_area(r) > 0.0 : ring_area(r) < 0.0) {
    for (int i = 1, j = r.n - 1; i < j; ++i, --j) {
      double tx = r.x[i], ty = r.y[i];
      r.x[i] = r.x[j];
      r.y[i] = r.y[j];
      r.x[j] = tx;
      r.y[j] = ty;
    }
  }
  double x0 = fmin(rect[0], rect[2]);
  double x1 = fmax(rect[0], rect[2]);
  double y0 = fmin(rect[1], rect[3]);
  double y1 = fmax(rect[1], rect[3]);
  if (!clip_half(r, tmp, 0, x0, true)) return kRegionOverflow;
  if (!clip_half(tmp, r, 0, x1, false)) return kRegionOverflow;
  if (!clip_half(r, tmp, 1, y0, true)) return kRegionOverflow;
  if (!clip_half(tmp, r, 1, y1, false)) return kRegionOverflow;
  int m = 0;
  for (int i = 0; i < r.n; ++i) {
    if (m == 0 || r.x[i] != r.x[m - 1] || r.y[i] != r.y[m - 1]) {
      r.x[m] = r.x[i];
      r.y[m] = r.y[i];
      ++m;
    }
  }
  while (m > 1 && r.x[0] == r.x[m - 1] && r.y[0] == r.y[m - 1]) --m;
  r.n = m;
  if (r.n < 3 || ring_area(r) == 0.0) return kRegionEmpty;
  return kRegionOk;
}

// One Sutherland-Hodgman pass against the half plane left of the clip edge a->b (convex
// support polygon; oracle shim clip_edge): side(p) = (b-a) x (p-a), inside iff >= 0,
// crossing point prev + t (cur - prev), t = side(prev) / (side(prev) - side(cur)).
template <int Cap>
SB_HD bool clip_edge(const RingT<Cap>& in, RingT<Cap>& out, double ax, double ay, double bx,
                     double by) {
  out.n = 0;
  const int n = in.n;
  const double ex = bx - ax, ey = by - ay;
  for (int i = 0; i < n; ++i) {
    const int ip = (i + n - 1) % n;
    const double sc = ex * (in.y[i] - ay) - ey * (in.x[i] - ax);
    const double sp = ex * (in.y[ip] - ay) - ey * (in.x[ip] - ax);
    const bool ci = sc >= 0.0, pi = sp >= 0.0;
    if (ci != pi) {
      const double t = sp / (sp - sc);
      if (!push(out, in.x[ip] + t * (in.x[i] - in.x[ip]), in.y[ip] + t * (in.y[i] - in.y[ip])))
        return false;
    }
    if (ci && !push(out, in.x[i], in.y[i])) return false;
  }
  return true;
}

// The support polygon as the intersection's clip operand (oracle shim `intersection`):
// n == 0: the axis-aligned rect `rect`; else a convex counter-clockwise ring (x, y).
struct SupportClip {
  const double* rect;
  int n;
  const double* x;
  const double* y;
};

// intersect(ring, support) as the oracle stand-in defines it (rect: intersect_rect; convex
// polygon: correct() orientation, one clip_edge pass per support edge in ring order, the
// same duplicate / area filter). Result in `r`.
template <int Cap>
SB_HD int intersect_support(RingT<Cap>& r, RingT<Cap>& tmp, const SupportClip& c, bool hole = false) {
  if (c.n == 0) return intersect_rect(r, tmp, c.rect, hole);
  if (r.n < 3) return kRegionEmpty;
  if (hole ? ring_area(r) > 0.0 : ring_area(r) < 0.0) {  // bg::correct keeps vertex 0 first
    for (int i = 1, j = r.n - 1; i < j; ++i, --j) {
      double tx = r.x[i], ty = r.y[i];
      r.x[i] = r.x[j];
      r.y[i] = r.y[j];
      r.x[j] = tx;
      r.y[j] = ty;
    }
  }
  for (int e = 0; e < c.n; ++e) {
    const int f = e + 1 == c.n ? 0 : e + 1;
    if (!clip_edge(r, tmp, c.x[e], c.y[e], c.x[f], c.y[f])) return kRegionOverflow;
    r.n = tmp.n;
    for (int i = 0; i < tmp.n; ++i) {
      r.x[i] = tmp.x[i];
      r.y[i] = tmp.y[i];
    }
  }
  int m = 0;
  for (int i = 0; i < r.n; ++i) {
    if (m == 0 || r.x[i] != r.x[m - 1] || r.y[i] != r.y[m - 1]) {
      r.x[m] = r.x[i];
      r.y[m] = r.y[i];
      ++m;
    }
  }
  while (m > 1 && r.x[0] == r.x[m - 1] && r.y[0] == r.y[m - 1]) --m;
  r.n = m;
  if (r.n < 3 || ring_area(r) == 0.0) return kRegionEmpty;
  return kRegionOk;
}

// erode() of a convex counter-clockwise ring by r (the oracle shim's buffer(-r), restated by
// sbh::erode_convex): in place; kRegionBadArg if concave, kRegionEmpty if eroded away.
template <int Cap>
SB_HD int erode_convex_ring(RingT<Cap>& ring, RingT<Cap>& tmp, double r) {
  const int n = ring.n;
  if (n < 3) return kRegionEmpty;
  for (int i = 0; i < n; ++i) {
    const int h = (i + n - 1) % n, q = (i + 1) % n;
    const double ox = ring.x[h], oy = ring.y[h], px = ring.x[i], py = ring.y[i];
    const double qx = ring.x[q], qy = ring.y[q];
    if ((px - ox) * (qy - oy) - (py - oy) * (qx - ox) < 0.0) return kRegionBadArg;
    const double dxh = px - ox, dyh = py - oy, dxi = qx - px, dyi = qy - py;
    const double lh = sqrt(dxh * dxh + dyh * dyh), li = sqrt(dxi * dxi + dyi * dyi);
    const double axh = ox + (-dyh / lh) * r, ayh = oy + (dxh / lh) * r;
    const double axi = px + (-dyi / li) * r, ayi = py + (dxi / li) * r;
    const double den = dxh * dyi - dyh * dxi;
    const double t = ((axi - axh) * dyi - (ayi - ayh) * dxi) / den;
    tmp.x[i] = axh + t * dxh;
    tmp.y[i] = ayh + t * dyh;
  }
  tmp.n = n;
  for (int i = 0; i < n; ++i) {
    const int q = (i + 1) % n;
    if (!((tmp.x[q] - tmp.x[i]) * (ring.x[q] - ring.x[i]) + (tmp.y[q] - tmp.y[i]) * (ring.y[q] - ring.y[i]) > 0.0))
      return kRegionEmpty;
  }
  for (int i = 0; i < n; ++i) {
    ring.x[i] = tmp.x[i];
    ring.y[i] = tmp.y[i];
  }
  return kRegionOk;
}

// ------------------------------------------------------------ middle (multi-anchor)
// is_valid_polygon (polygon.cpp:407-410) as the oracle shim defines bg::is_valid: a simple
// ring -- >= 3 vertices after dropping consecutive exact duplicates, finite, non-zero
// area, no two non-adjacent edges meeting (closed segments, exact orientation signs).
SB_HD int orient_sign(double ax, double ay, double bx, double by, double cx, double cy) {
  const double c = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
  return c > 0.0 ? 1 : (c < 0.0 ? -1 : 0);
}
SB_HD bool on_box(double ax, double ay, double bx, double by, double cx, double cy) {
  return fmin(ax, bx) <= cx && cx <= fmax(ax, bx) && fmin(ay, by) <= cy && cy <= fmax(ay, by);
}
SB_HD bool segments_meet(double px, double py, double qx, double qy, double rx, double ry,
                         double sx, double sy) {
  const int o1 = orient_sign(px, py, qx, qy, rx, ry), o2 = orient_sign(px, py, qx, qy, sx, sy);
  const int o3 = orient_sign(rx, ry, sx, sy, px, py), o4 = orient_sign(rx, ry, sx, sy, qx, qy);
  if (o1 != o2 && o3 != o4) return true;
  if (o1 == 0 && on_box(px, py, qx, qy, rx, ry)) return true;
  if (o2 == 0 && on_box(px, py, qx, qy, sx, sy)) return true;
  if (o3 == 0 && on_box(rx, ry, sx, sy, px, py)) return true;
  if (o4 == 0 && on_box(rx, ry, sx, sy, qx, qy)) return true;
  return false;
}
template <int Cap>
SB_HD bool simple_ring(const RingT<Cap>& in, RingT<Cap>& r) {
  // to_boost: correct() (orientation only -- irrelevant to simplicity) then the open ring
  r.n = 0;
  for (int i = 0; i < in.n; ++i)
    if (r.n == 0 || in.x[i] != r.x[r.n - 1] || in.y[i] != r.y[r.n - 1]) push(r, in.x[i], in.y[i]);
  while (r.n > 1 && r.x[0] == r.x[r.n - 1] && r.y[0] == r.y[r.n - 1]) --r.n;
  const int n = r.n;
  if (n < 3) return false;
  for (int i = 0; i < n; ++i)
    if (!isfinite(r.x[i]) || !isfinite(r.y[i])) return false;
  if (ring_area(r) == 0.0) return false;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      if (j == i + 1 || (i == 0 && j == n - 1)) continue;
      const int i1 = (i + 1) % n, j1 = (j + 1) % n;
      if (segments_meet(r.x[i], r.y[i], r.x[i1], r.y[i1], r.x[j], r.y[j], r.x[j1], r.y[j1]))
        return false;
    }
  return true;
}

// convex_hull (polygon.cpp:412-420) as the oracle shim defines bg::convex_hull: Andrew's
// monotone chain over the points sorted by (x, y) (stable insertion sort; equal points
// are interchangeable), collinear and duplicate points dropped, counter-clockwise from the
// lowest (x, y); ring_to_vec drops the closing vertex.
template <int Cap>
SB_HD void convex_hull_ring(const double* px, const double* py, int m, RingT<Cap>& out) {
  double sx[SB_MAX_ANCHORS], sy[SB_MAX_ANCHORS];
  for (int i = 0; i < m; ++i) {
    double x = px[i], y = py[i];
    int j = i;
    while (j > 0 && (x < sx[j - 1] || (x == sx[j - 1] && y < sy[j - 1]))) {
      sx[j] = sx[j - 1];
      sy[j] = sy[j - 1];
      --j;
    }
    sx[j] = x;
    sy[j] = y;
  }
  auto turn = [](double ox, double oy, double ax, double ay, double bx, double by) {
    return (ax - ox) * (by - oy) - (ay - oy) * (bx - ox);
  };
  out.n = 0;
  for (int i = 0; i < m; ++i) {
    while (out.n >= 2 && turn(out.x[out.n - 2], out.y[out.n - 2], out.x[out.n - 1], out.y[out.n - 1], sx[i], sy[i]) <= 0.0)
      --out.n;
    push(out, sx[i], sy[i]);
  }
  const int lower = out.n + 1;
  for (int i = m - 1; i >= 0; --i) {
    while (out.n >= lower && turn(out.x[out.n - 2], out.y[out.n - 2], out.x[out.n - 1], out.y[out.n - 1], sx[i], sy[i]) <= 0.0)
      --out.n;
    push(out, sx[i], sy[i]);
  }
  if (out.n > 1) --out.n;  // the start point again
  // close_ring + ring_to_vec: the closing copy is dropped again; a 1-point hull keeps its
  // point (ring_to_vec drops only a distinct-looking closing vertex within 1e-15)
}

// stadium (relationships.cpp:17-40): the capsule of radius `radius` around segment a-b
// (a disc of 72 points if a == b), cap at b then cap at a, 37 points each.
template <class M, int Cap>
SB_HD bool stadium_ring(double ax, double ay, double bx, double by, double radius, RingT<Cap>& out) {
  out.n = 0;
  const double dx = bx - ax, dy = by - ay;
  const double len = sqrt(dx * dx + dy * dy);
  if (len < 1e-12) {
    for (int i = 0; i < 72; ++i) {
      const double ang = 2.0 * kPi * (double)i / 72;
      double sa, ca;
      M::sincos(ang, &sa, &ca);
      if (!push(out, ax + radius * ca, ay + radius * sa)) return false;
    }
    return true;
  }
  const double ux = dx / len, uy = dy / len;
  const double base = M::atan2(uy, ux);
  auto cap = [&](double cx, double cy, double a0, double a1) -> bool {
    const int steps = 36;
    for (int i = 0; i <= steps; ++i) {
      const double ang = a0 + (a1 - a0) * (double)i / (double)steps;
      double sa, ca;
      M::sincos(ang, &sa, &ca);
      if (!push(out, cx + radius * ca, cy + radius * sa)) return false;
    }
    return true;
  };
  if (!cap(bx, by, base - kPi / 2, base + kPi / 2)) return false;
  return cap(ax, ay, base + kPi / 2, base + 3 * kPi / 2);
}

// middle_polygon (relationships.cpp:124-157) of m >= 2 anchor positions.
template <class M, int Cap>
SB_HD int middle_ring(const double* px, const double* py, int m, RingT<Cap>& out, RingT<Cap>& tmp) {
  if (m < 2 || m > SB_MAX_ANCHORS) return kRegionBadArg;
  const double inf = INFINITY;
  double bx0 = inf, by0 = inf, bx1 = -inf, by1 = -inf;
  for (int i = 0; i < m; ++i) {
    bx0 = fmin(bx0, px[i]);
    by0 = fmin(by0, py[i]);
    bx1 = fmax(bx1, px[i]);
    by1 = fmax(by1, py[i]);
  }
  double diag = 0.0;
  if (!(bx0 > bx1)) {
    const double ddx = bx1 - bx0, ddy = by1 - by0;
    diag = sqrt(ddx * ddx + ddy * ddy);
  }
  const double scale = fmax(1e-9, diag);
  bool collinear = true;  // relationships.cpp:42-50
  if (m >= 3) {
    const double ex = px[1] - px[0], ey = py[1] - py[0];
    for (int i = 2; i < m && collinear; ++i) {
      const double c = ex * (py[i] - py[0]) - ey * (px[i] - px[0]);
      if (fabs(c) > 1e-9 * scale * scale) collinear = false;
    }
  }
  if (m == 2 || collinear) {  // inflated extreme segment (lexicographic lo / hi)
    int lo = 0, hi = 0;
    for (int i = 0; i < m; ++i) {
      if (px[i] < px[lo] || (px[i] == px[lo] && py[i] < py[lo])) lo = i;
      if (px[i] > px[hi] || (px[i] == px[hi] && py[i] > py[hi])) hi = i;
    }
    const double sx = px[hi] - px[lo], sy = py[hi] - py[lo];
    const double sep = sqrt(sx * sx + sy * sy);
    return stadium_ring<M>(px[lo], py[lo], px[hi], py[hi], fmax(1e-6, 0.1 * sep), out) ? kRegionOk
                                                                                      : kRegionOverflow;
  }
  double cx = 0.0, cy = 0.0;
  for (int i = 0; i < m; ++i) {
    cx = cx + px[i];
    cy = cy + py[i];
  }
  cx = cx / (double)m;
  cy = cy / (double)m;
  // std::sort of <= 16 elements is libstdc++'s insertion sort: stable on equal angles
  double key[SB_MAX_ANCHORS];
  out.n = 0;
  for (int i = 0; i < m; ++i) {
    const double k = M::atan2(py[i] - cy, px[i] - cx);
    int j = out.n;
    push(out, 0.0, 0.0);
    while (j > 0 && k < key[j - 1]) {
      key[j] = key[j - 1];
      out.x[j] = out.x[j - 1];
      out.y[j] = out.y[j - 1];
      --j;
    }
    key[j] = k;
    out.x[j] = px[i];
    out.y[j] = py[i];
  }
  if (!simple_ring(out, tmp)) convex_hull_ring(px, py, m, out);  // equal-angle ties
  return kRegionOk;
}

// point_in_tri_strict (polygon.cpp:189-195)
SB_HD bool point_in_tri_strict(double px, double py, double ax, double ay, double bx, double by,
                               double cx, double cy) {
  const double eps = 1e-12;
  double d1 = cross2(ax, ay, bx, by, px, py);
  double d2 = cross2(bx, by, cx, cy, px, py);
  double d3 = cross2(cx, cy, ax, ay, px, py);
  return d1 > eps && d2 > eps && d3 > eps;
}

// Sampler table being built: triangles with positive area and their cumulative areas
// (PolygonSampler ctor, polygon.cpp:370-388). Caller provides storage for kCap-2 tris.
struct TableSink {
  SbRegionTri* tris;
  double* cum;
  int n;
  int cap;
  double total;
};

SB_HD bool sink_tri(TableSink& s, double ax, double ay, double bx, double by, double cx,
                    double cy) {
  double a = 0.5 * fabs(cross2(ax, ay, bx, by, cx, cy));
  if (a <= 0.0) return true;
  if (s.n >= s.cap) return false;
  SbRegionTri& t = s.tris[s.n];
  t.a[0] = ax;
  t.a[1] = ay;
  t.b[0] = bx;
  t.b[1] = by;
  t.c[0] = cx;
  t.c[1] = cy;
  s.total += a;
  s.cum[s.n] = s.total;
  ++s.n;
  return true;
}

// triangulate() of a hole-free polygon (polygon.cpp:344-368) feeding ear_clip_ring
// (polygon.cpp:260-340) straight into the sampler table. `r` is consumed. orient = false:
// ear_clip_ring alone (a ring triangulate() already oriented and bridged).
template <int Cap>
#ifdef __CUDACC__
static __host__ __device__ __noinline__
#else
inline
#endif
bool ear_clip_into(RingT<Cap>& r, TableSink& sink, bool orient = true) {
  if (r.n < 3) return true;
  if (orient && ring_area(r) < 0.0) reverse_ring(r);
  // drop consecutive duplicates (squared distance <= 1e-24)
  int n = 0;
  for (int i = 0; i < r.n; ++i) {
    if (n > 0) {
      double dx = r.x[i] - r.x[n - 1], dy = r.y[i] - r.y[n - 1];
      if (!(dx * dx + dy * dy > 1e-24)) continue;
    }
    r.x[n] = r.x[i];
    r.y[n] = r.y[i];
    ++n;
  }
  while (n > 1) {
    double dx = r.x[0] - r.x[n - 1], dy = r.y[0] - r.y[n - 1];
    if (dx * dx + dy * dy <= 1e-24) --n;
    else break;
  }
  if (n < 3) return true;
  // Fast path, exact: when no vertex is reflex and every ear the loop would clip passes
  // the sliver test, ear_clip_ring's sequence is cur = 0, 1, 2, ... with prev pinned at
  // vertex n-1, i.e. the fan (n-1, k, k+1) for k = 0..n-3 (the last one emitted by the
  // `remaining == 3` tail). Convex clipped sectors always take this path.
  {
    bool fan = true;
    for (int i = 0; i < n && fan; ++i) {
      const int a = (i + n - 1) % n, c = (i + 1) % n;
      if (cross2(r.x[a], r.y[a], r.x[i], r.y[i], r.x[c], r.y[c]) < 0.0) fan = false;
    }
    for (int k = 0; k + 3 < n && fan; ++k) {
      const double cr = cross2(r.x[n - 1], r.y[n - 1], r.x[k], r.y[k], r.x[k + 1], r.y[k + 1]);
      if (cr < 0.0 || fabs(cr) < 1e-18) fan = false;
    }
    if (fan) {
      for (int k = 0; k + 2 < n; ++k)
        if (!sink_tri(sink, r.x[n - 1], r.y[n - 1], r.x[k], r.y[k], r.x[k + 1], r.y[k + 1]))
          return false;
      return true;
    }
  }
  int prv[Cap], nxt[Cap];
  bool reflex[Cap];
  for (int i = 0; i < n; ++i) {
    prv[i] = (i + n - 1) % n;
    nxt[i] = (i + 1) % n;
  }
  auto update_reflex = [&](int i) {
    reflex[i] = cross2(r.x[prv[i]], r.y[prv[i]], r.x[i], r.y[i], r.x[nxt[i]], r.y[nxt[i]]) < 0.0;
  };
  for (int i = 0; i < n; ++i) update_reflex(i);
  auto is_ear = [&](int i) -> bool {
    if (reflex[i]) return false;
    int p = prv[i], q = nxt[i];
    double ax = r.x[p], ay = r.y[p], bx = r.x[i], by = r.y[i], cx = r.x[q], cy = r.y[q];
    if (fabs(cross2(ax, ay, bx, by, cx, cy)) < 1e-18) return false;
    for (int j = nxt[q]; j != p; j = nxt[j]) {
      if (reflex[j] && point_in_tri_strict(r.x[j], r.y[j], ax, ay, bx, by, cx, cy)) return false;
    }
    return true;
  };
  int remaining = n, cur = 0, since_clip = 0;
  while (remaining > 3) {
    if (is_ear(cur)) {
      int p = prv[cur], q = nxt[cur];
      if (!sink_tri(sink, r.x[p], r.y[p], r.x[cur], r.y[cur], r.x[q], r.y[q])) return false;
      nxt[p] = q;
      prv[q] = p;
      update_reflex(p);
      update_reflex(q);
      cur = q;
      --remaining;
      since_clip = 0;
      continue;
    }
    cur = nxt[cur];
    if (++since_clip > remaining) {
      int best = -1;
      double best_a = -1.0;
      for (int j = cur, k = 0; k < remaining; j = nxt[j], ++k) {
        if (reflex[j]) continue;
        double a = cross2(r.x[prv[j]], r.y[prv[j]], r.x[j], r.y[j], r.x[nxt[j]], r.y[nxt[j]]);
        if (a > best_a) {
          best_a = a;
          best = j;
        }
      }
      if (best < 0) break;
      int p = prv[best], q = nxt[best];
      if (!sink_tri(sink, r.x[p], r.y[p], r.x[best], r.y[best], r.x[q], r.y[q])) return false;
      nxt[p] = q;
      prv[q] = p;
      update_reflex(p);
      update_reflex(q);
      cur = q;
      --remaining;
      since_clip = 0;
    }
  }
  if (remaining == 3) {
    int p = prv[cur], q = nxt[cur];
    if (!sink_tri(sink, r.x[p], r.y[p], r.x[cur], r.y[cur], r.x[q], r.y[q])) return false;
  }
  return true;
}

// ------------------------------------------------------------ annulus with a hole
// libm policy for the hole path: glibc on the host (the reference's), the correctly
// rounded device functions in sb_region.cu.
struct HostMath {
  static inline void sincos(double a, double* s, double* c) {
    *s = ::sin(a);
    *c = ::cos(a);
  }
  static inline double atan2(double y, double x) { return ::atan2(y, x); }
};

// bridge_hole (polygon.cpp:197-258): merge the CW hole into the CCW outer ring at the
// hole's max-x vertex; a reflex outer vertex inside the bridge triangle takes over as
// the bridge end (the candidate and its triangle update as the scan proceeds).
template <class M>
SB_HD bool bridge_hole(const Ring& outer, const Ring& hole, HoleRing& out) {
  int mi = 0;
  for (int i = 1; i < hole.n; ++i)
    if (hole.x[i] > hole.x[mi]) mi = i;
  const double mx = hole.x[mi], my = hole.y[mi];
  const int n = outer.n;
  double best_x = INFINITY, hx = 0.0, hy = 0.0;
  int best_edge = n;
  for (int i = 0; i < n; ++i) {
    const int j = (i + 1) % n;
    const double ax = outer.x[i], ay = outer.y[i], bx = outer.x[j], by = outer.y[j];
    if ((ay > my) == (by > my)) continue;
    const double t = (my - ay) / (by - ay);
    const double x = ax + t * (bx - ax);
    if (x >= mx - 1e-12 && x < best_x) {
      best_x = x;
      best_edge = i;
      hx = x;
      hy = my;
    }
  }
  out.n = 0;
  if (best_edge == n) {  // degenerate: the hole is dropped (polygon.cpp:219-222)
    for (int i = 0; i < n; ++i)
      if (!push(out, outer.x[i], outer.y[i])) return false;
    return true;
  }
  const int eb = (best_edge + 1) % n;
  int cand = outer.x[best_edge] > outer.x[eb] ? best_edge : eb;
  double cx = outer.x[cand], cy = outer.y[cand];
  double best_metric = INFINITY;
  for (int i = 0; i < n; ++i) {
    if (i == cand) continue;
    const int ip = (i + n - 1) % n, in = (i + 1) % n;
    const bool reflex =
        cross2(outer.x[ip], outer.y[ip], outer.x[i], outer.y[i], outer.x[in], outer.y[in]) < 0.0;
    if (!reflex) continue;
    if (point_in_tri_strict(outer.x[i], outer.y[i], mx, my, hx, hy, cx, cy) ||
        point_in_tri_strict(outer.x[i], outer.y[i], mx, my, cx, cy, hx, hy)) {
      const double dx = outer.x[i] - mx, dy = outer.y[i] - my;
      const double metric = fabs(M::atan2(dy, dx));
      if (metric < best_metric) {
        best_metric = metric;
        cand = i;
        cx = outer.x[i];
        cy = outer.y[i];
      }
    }
  }
  for (int i = 0; i <= cand; ++i)
    if (!push(out, outer.x[i], outer.y[i])) return false;
  for (int k = 0; k <= hole.n; ++k)
    if (!push(out, hole.x[(mi + k) % hole.n], hole.y[(mi + k) % hole.n])) return false;
  if (!push(out, outer.x[cand], outer.y[cand])) return false;
  for (int i = cand + 1; i < n; ++i)
    if (!push(out, outer.x[i], outer.y[i])) return false;
  return true;
}

struct HoleScratch {
  Ring o, h, tmp;
  HoleRing mg, mg2;
};

// region_for(i) of a full annulus with a hole (theta = pi, min_r > 0;
// relationships.cpp:197-209): annulus_sector's full branch (polygon.cpp:157-167, outer
// circle + CW inner circle), the shim intersection (outer and hole each clipped to the
// rect; a hole that clips away is dropped), from_boost, then triangulate (orientation,
// bridge_hole) and ear_clip_ring into the sampler table. max_r must be finite.
template <class M>
SB_HD int hole_annulus_table(double cx, double cy, double min_r, double max_r,
                             const SupportClip& clip, double erode_r, HoleScratch& sc,
                             TableSink& sink) {
  const double step = 5.0 * kPi / 180.0;
  auto arc = [&](Ring& out, double radius, double a0, double a1) -> bool {
    int na = (int)ceil(fabs(a1 - a0) / step);
    if (na < 1) na = 1;
    for (int i = 0; i <= na; ++i) {
      const double a = a0 + (a1 - a0) * (double)i / (double)na;
      double sa, ca;
      M::sincos(a, &sa, &ca);
      if (!push(out, cx + radius * ca, cy + radius * sa)) return false;
    }
    out.n -= 1;  // closing vertex
    return true;
  };
  sc.o.n = 0;
  sc.h.n = 0;
  if (!arc(sc.o, max_r, 0.0, 2.0 * kPi) || !arc(sc.h, min_r, 2.0 * kPi, 0.0))
    return kRegionOverflow;
  const int so = intersect_support(sc.o, sc.tmp, clip, false);
  if (so == kRegionOverflow) return so;
  if (so != kRegionOk) return kRegionEmpty;
  const int sh = intersect_support(sc.h, sc.tmp, clip, true);
  if (sh == kRegionOverflow) return sh;
  if (erode_r > 0.0) {  // apply_ratio_on_support: the shim's buffer takes hole-free rings only
    if (sh == kRegionOk) return kRegionBadArg;
    const int se = erode_convex_ring(sc.o, sc.tmp, erode_r);
    if (se != kRegionOk) return se;
  }
  if (ring_area(sc.o) < 0.0) reverse_ring(sc.o);  // triangulate (polygon.cpp:348-354)
  if (sh == kRegionOk) {
    if (ring_area(sc.h) > 0.0) reverse_ring(sc.h);
    if (!bridge_hole<M>(sc.o, sc.h, sc.mg)) return kRegionOverflow;
  } else {
    sc.mg.n = 0;
    for (int i = 0; i < sc.o.n; ++i) push(sc.mg, sc.o.x[i], sc.o.y[i]);
  }
  if (!ear_clip_into(sc.mg, sink, false)) return kRegionOverflow;
  return kRegionOk;
}

// annulus_sector (polygon.cpp:136-176) for every shape but the holed annulus, into a big
// ring (wide annular sectors need up to 2 * 73 arc points). max_r must be finite.
template <class M>
SB_HD int sector_ring(double cx, double cy, double vx, double vy, double theta, double min_r,
                      double max_r, HoleRing& out) {
  out.n = 0;
  const bool full = theta >= kPi - 1e-12;
  const double step = 5.0 * kPi / 180.0;
  auto arc = [&](double radius, double a0, double a1) -> bool {
    int na = (int)ceil(fabs(a1 - a0) / step);
    if (na < 1) na = 1;
    for (int i = 0; i <= na; ++i) {
      const double a = a0 + (a1 - a0) * (double)i / (double)na;
      double sa, ca;
      M::sincos(a, &sa, &ca);
      if (!push(out, cx + radius * ca, cy + radius * sa)) return false;
    }
    return true;
  };
  if (full) {
    if (min_r > 0.0) return kRegionBadArg;  // holed annulus: hole_annulus_table
    if (!arc(max_r, 0.0, 2.0 * kPi)) return kRegionOverflow;
    out.n -= 1;  // closing vertex
    return kRegionOk;
  }
  const double base = M::atan2(vy, vx);
  if (!arc(max_r, base - theta, base + theta)) return kRegionOverflow;
  if (min_r > 0.0) {
    if (!arc(min_r, base + theta, base - theta)) return kRegionOverflow;
  } else if (!push(out, cx, cy)) {
    return kRegionOverflow;
  }
  return kRegionOk;
}

// region_for(i) on the serial path: shapes whose ring outgrows the group path's kCap, and
// every shape on a polygon support (sector_ring -> the shim intersection -> optional
// erosion -> triangulate -> the sampler table).
template <class M>
SB_HD int big_region_table(double cx, double cy, double vx, double vy, double theta,
                           double min_r, double max_r, const SupportClip& clip, double erode_r,
                           HoleScratch& sc, TableSink& sink) {
  int st = sector_ring<M>(cx, cy, vx, vy, theta, min_r, max_r, sc.mg);
  if (st != kRegionOk) return st;
  st = intersect_support(sc.mg, sc.mg2, clip, false);
  if (st == kRegionOverflow) return st;
  if (st != kRegionOk) return kRegionEmpty;
  if (erode_r > 0.0) {  // apply_ratio_on_support: convex rings only (the shim's buffer)
    st = erode_convex_ring(sc.mg, sc.mg2, erode_r);
    if (st != kRegionOk) return st;
  }
  if (!ear_clip_into(sc.mg, sink, true)) return kRegionOverflow;
  return kRegionOk;
}

// region_for(i) of a `middle` relation (relationships.cpp:192-196): middle_polygon ->
// the shim intersection with the support -> optional erosion (apply_ratio_on_support) ->
// triangulate -> the sampler table.
template <class M>
SB_HD int middle_region_table(const double* px, const double* py, int m, const SupportClip& clip,
                              double erode_r, Ring& r, Ring& tmp, TableSink& sink) {
  int st = middle_ring<M>(px, py, m, r, tmp);
  if (st != kRegionOk) return st;
  st = intersect_support(r, tmp, clip, false);
  if (st != kRegionOk) return st;
  if (erode_r > 0.0) {
    st = erode_convex_ring(r, tmp, erode_r);
    if (st != kRegionOk) return st;
  }
  if (!ear_clip_into(r, sink, true)) return kRegionOverflow;
  return kRegionOk;
}

// Normalise the cumulative table (polygon.cpp:381-387). Returns the triangle count
// (0 = invalid sampler, i.e. placeable == 0).
SB_HD int finish_table(TableSink& s) {
  if (s.total > 0.0) {
    for (int k = 0; k < s.n; ++k) s.cum[k] /= s.total;
    s.cum[s.n - 1] = 1.0;
    return s.n;
  }
  s.n = 0;
  return 0;
}

// PolygonSampler::draw (polygon.cpp:390-400) given the three uniforms.
SB_HD void draw_point(const SbRegionTri* tris, const double* cum, int n, double u, double r1,
                      double r2, double& px, double& py) {
  int lo = 0, hi = n;  // lower_bound: first k with !(cum[k] < u)
  while (lo < hi) {
    int mid = lo + ((hi - lo) >> 1);
    if (cum[mid] < u) lo = mid + 1;
    else hi = mid;
  }
  int idx = lo < n - 1 ? lo : n - 1;
  const SbRegionTri& t = tris[idx];
  double s = sqrt(r1);
  double wa = 1.0 - s;
  double wb = s * (1.0 - r2);
  double wc = s * r2;
  px = t.a[0] * wa + t.b[0] * wb + t.c[0] * wc;
  py = t.a[1] * wa + t.b[1] * wb + t.c[1] * wc;
}

}  // namespace sbp
