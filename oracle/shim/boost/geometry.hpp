// TEST INFRASTRUCTURE ONLY (oracle build of the reference; never linked into the product).
//
// Minimal stand-in for the Boost.Geometry calls made by /root/reference/proj/src/polygon.cpp
// (Boost is not vendored with the reference and is absent from this image).
//
// Implemented (the subset the hot path needs):
//   append, get, correct (close rings, outer CCW / holes CW), area (shoelace),
//   intersection(multi_polygon, multi_polygon) where the SECOND operand is a single
//     axis-aligned rectangle (a support rect, polygon.cpp:115-119 via
//     relationships.cpp:284,295). Each ring of the first operand is clipped with
//     Sutherland-Hodgman against x>=x0, x<=x1, y>=y0, y<=y1 in that order; consecutive
//     exact duplicates are dropped; rings with < 3 vertices or zero area are discarded.
//     This is a DEFINED stand-in: the product restates exactly this algorithm, and parity
//     against an upstream Boost build of the reference is unpinned.
//   When the second operand is not an axis-aligned rectangle it must be a convex polygon
//     (a convex support surface): each ring is clipped against the half planes left of
//     its corrected (counter-clockwise) edges v0->v1, v1->v2, ... in ring order; side(p) =
//     (b-a) x (p-a), inside iff side >= 0, crossing point prev + t (cur - prev) with
//     t = side(prev) / (side(prev) - side(cur)); then the same duplicate / area filter.
// buffer: erosion (negative distance) of convex hole-free polygons (see below).
// is_valid (polygon): >= 3 vertices after dropping consecutive exact duplicates, finite
//   coordinates, non-zero area, and no two non-adjacent edges that intersect or touch
//   (closed segments, exact orientation signs) -- a simple ring.
// convex_hull (multi_point): Andrew's monotone chain over the points sorted by (x, y);
//   collinear and duplicate points dropped; counter-clockwise from the lowest (x, y).
// union_: polygons that share an edge (exact vertex equality, opposite directions) are
//   spliced along it (the shared edge removed, every other vertex kept, the first
//   operand's ring order and start kept); parts sharing no edge stay separate.
//   This is the stand-in support-surface extraction (surface.cpp:103-109) runs on.
// distance throws (not on the hot path).
// Like the rect clipping, each of these is a DEFINED stand-in the product restates
// exactly; parity against upstream Boost is unpinned.
#pragma once

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <vector>

namespace boost {
namespace geometry {
namespace model {
namespace d2 {
template <class T>
struct point_xy {
  T v[2];
  point_xy(T x = 0, T y = 0) : v{x, y} {}
};
}  // namespace d2
template <class P, bool ClockWise = true, bool Closed = true>
struct polygon {
  using ring_type = std::vector<P>;
  ring_type outer_;
  std::vector<ring_type> inners_;
  ring_type& outer() { return outer_; }
  const ring_type& outer() const { return outer_; }
  std::vector<ring_type>& inners() { return inners_; }
  const std::vector<ring_type>& inners() const { return inners_; }
};
template <class P>
struct multi_polygon : std::vector<P> {};
template <class P>
struct multi_point : std::vector<P> {};
}  // namespace model

template <int I, class T>
T get(const model::d2::point_xy<T>& p) {
  return p.v[I];
}
template <class Container, class P>
void append(Container& c, const P& p) {
  c.push_back(p);
}

namespace shim_detail {
template <class Ring>
double signed_area(const Ring& r) {  // ring may be closed or open
  double s = 0.0;
  std::size_t n = r.size();
  for (std::size_t i = 0; i < n; ++i) {
    const auto& a = r[i];
    const auto& b = r[(i + 1) % n];
    s += a.v[0] * b.v[1] - b.v[0] * a.v[1];
  }
  return 0.5 * s;
}
template <class Ring>
void close_ring(Ring& r) {
  if (!r.empty() && (r.front().v[0] != r.back().v[0] || r.front().v[1] != r.back().v[1]))
    r.push_back(r.front());
}
template <class Ring>
Ring open_ring(const Ring& r) {
  Ring o = r;
  if (o.size() > 1 && o.front().v[0] == o.back().v[0] && o.front().v[1] == o.back().v[1])
    o.pop_back();
  return o;
}
// Sutherland-Hodgman against one axis-aligned half plane.
// axis 0: x, axis 1: y; keep_ge: keep coord >= bound, else keep coord <= bound.
template <class Ring>
Ring clip_half(const Ring& in, int axis, double bound, bool keep_ge) {
  Ring out;
  std::size_t n = in.size();
  if (n == 0) return out;
  auto inside = [&](const auto& p) { return keep_ge ? p.v[axis] >= bound : p.v[axis] <= bound; };
  auto cross = [&](const auto& p, const auto& q) {
    typename Ring::value_type r;
    int o = 1 - axis;
    double t = (bound - p.v[axis]) / (q.v[axis] - p.v[axis]);
    r.v[axis] = bound;
    r.v[o] = p.v[o] + t * (q.v[o] - p.v[o]);
    return r;
  };
  for (std::size_t i = 0; i < n; ++i) {
    const auto& cur = in[i];
    const auto& prev = in[(i + n - 1) % n];
    bool ci = inside(cur), pi = inside(prev);
    if (ci) {
      if (!pi) out.push_back(cross(prev, cur));
      out.push_back(cur);
    } else if (pi) {
      out.push_back(cross(prev, cur));
    }
  }
  return out;
}
// Sutherland-Hodgman against the half plane left of edge a->b (convex clip operand).
template <class Ring, class P>
Ring clip_edge(const Ring& in, const P& a, const P& b) {
  Ring out;
  std::size_t n = in.size();
  if (n == 0) return out;
  const double ex = b.v[0] - a.v[0], ey = b.v[1] - a.v[1];
  auto side = [&](const P& p) { return ex * (p.v[1] - a.v[1]) - ey * (p.v[0] - a.v[0]); };
  for (std::size_t i = 0; i < n; ++i) {
    const auto& cur = in[i];
    const auto& prev = in[(i + n - 1) % n];
    const double sc = side(cur), sp = side(prev);
    const bool ci = sc >= 0.0, pi = sp >= 0.0;
    if (ci != pi) {
      const double t = sp / (sp - sc);
      P r;
      r.v[0] = prev.v[0] + t * (cur.v[0] - prev.v[0]);
      r.v[1] = prev.v[1] + t * (cur.v[1] - prev.v[1]);
      out.push_back(r);
    }
    if (ci) out.push_back(cur);
  }
  return out;
}
template <class Ring>
Ring dedupe_ring(const Ring& r) {
  Ring o;
  for (const auto& p : r) {
    if (o.empty() || p.v[0] != o.back().v[0] || p.v[1] != o.back().v[1]) o.push_back(p);
  }
  while (o.size() > 1 && o.front().v[0] == o.back().v[0] && o.front().v[1] == o.back().v[1])
    o.pop_back();
  return o;
}
template <class Ring>
Ring clip_convex(const Ring& closed_in, const Ring& clip_open) {
  Ring r = open_ring(closed_in);
  for (std::size_t e = 0; e < clip_open.size(); ++e)
    r = clip_edge(r, clip_open[e], clip_open[(e + 1) % clip_open.size()]);
  return dedupe_ring(r);
}
template <class Ring>
Ring clip_rect(const Ring& closed_in, double x0, double y0, double x1, double y1) {
  Ring r = open_ring(closed_in);
  r = clip_half(r, 0, x0, true);
  r = clip_half(r, 0, x1, false);
  r = clip_half(r, 1, y0, true);
  r = clip_half(r, 1, y1, false);
  Ring o;
  for (const auto& p : r) {
    if (o.empty() || p.v[0] != o.back().v[0] || p.v[1] != o.back().v[1]) o.push_back(p);
  }
  while (o.size() > 1 && o.front().v[0] == o.back().v[0] && o.front().v[1] == o.back().v[1])
    o.pop_back();
  return o;
}
}  // namespace shim_detail

template <class P, bool CW, bool Cl>
void correct(model::polygon<P, CW, Cl>& poly) {
  shim_detail::close_ring(poly.outer());
  for (auto& h : poly.inners()) shim_detail::close_ring(h);
  // CW == false: outer counter-clockwise (positive area), holes clockwise.
  double sgn = CW ? -1.0 : 1.0;
  if (sgn * shim_detail::signed_area(poly.outer()) < 0.0)
    std::vector<P>(poly.outer().rbegin(), poly.outer().rend()).swap(poly.outer());
  for (auto& h : poly.inners())
    if (sgn * shim_detail::signed_area(h) > 0.0) std::vector<P>(h.rbegin(), h.rend()).swap(h);
}

template <class P, bool CW, bool Cl>
double area(const model::polygon<P, CW, Cl>& p) {
  double a = std::abs(shim_detail::signed_area(p.outer()));
  for (const auto& h : p.inners()) a -= std::abs(shim_detail::signed_area(h));
  return a;
}
template <class P>
double area(const model::multi_polygon<P>& m) {
  double a = 0.0;
  for (const auto& p : m) a += area(p);
  return a;
}

template <class Poly>
void intersection(const model::multi_polygon<Poly>& a, const model::multi_polygon<Poly>& b,
                  model::multi_polygon<Poly>& out) {
  if (b.size() != 1 || !b[0].inners().empty())
    throw std::runtime_error("boost shim: intersection needs a single rectangle clip operand");
  auto rect = shim_detail::open_ring(b[0].outer());
  if (rect.size() < 3) throw std::runtime_error("boost shim: clip operand has < 3 vertices");
  double x0 = rect[0].v[0], x1 = rect[0].v[0], y0 = rect[0].v[1], y1 = rect[0].v[1];
  for (const auto& p : rect) {
    x0 = std::fmin(x0, p.v[0]);
    x1 = std::fmax(x1, p.v[0]);
    y0 = std::fmin(y0, p.v[1]);
    y1 = std::fmax(y1, p.v[1]);
  }
  bool is_rect = rect.size() == 4;
  for (const auto& p : rect) {
    bool on_x = p.v[0] == x0 || p.v[0] == x1;
    bool on_y = p.v[1] == y0 || p.v[1] == y1;
    if (!on_x || !on_y) is_rect = false;
  }
  if (!is_rect) {
    const std::size_t k = rect.size();
    for (std::size_t i = 0; i < k; ++i) {
      const auto& o = rect[(i + k - 1) % k];
      const auto& p = rect[i];
      const auto& q = rect[(i + 1) % k];
      if ((p.v[0] - o.v[0]) * (q.v[1] - o.v[1]) - (p.v[1] - o.v[1]) * (q.v[0] - o.v[0]) < 0.0)
        throw std::runtime_error("boost shim: clip operand is neither a rectangle nor convex");
    }
  }
  auto clip = [&](const typename Poly::ring_type& ring) {
    return is_rect ? shim_detail::clip_rect(ring, x0, y0, x1, y1) : shim_detail::clip_convex(ring, rect);
  };
  for (const auto& poly : a) {
    Poly res;
    res.outer() = clip(poly.outer());
    if (res.outer().size() < 3 || shim_detail::signed_area(res.outer()) == 0.0) continue;
    for (const auto& h : poly.inners()) {
      auto hc = clip(h);
      if (hc.size() >= 3 && shim_detail::signed_area(hc) != 0.0) res.inners().push_back(hc);
    }
    shim_detail::close_ring(res.outer());
    for (auto& h : res.inners()) shim_detail::close_ring(h);
    out.push_back(res);
  }
}

namespace strategy {
namespace buffer {
template <class T>
struct distance_symmetric {
  T value;
  explicit distance_symmetric(T v) : value(v) {}
};
struct side_straight {};
struct join_round {
  explicit join_round(int) {}
};
struct end_round {
  explicit end_round(int) {}
};
struct point_circle {
  explicit point_circle(int) {}
};
}  // namespace buffer
}  // namespace strategy

// buffer with a negative distance on convex, hole-free polygons: the DEFINED stand-in for
// erode() (polygon.cpp:101-113) -- every edge moves inward by r along its unit normal and
// vertex i becomes the intersection of the offset edges i-1 and i (same order as the input
// ring); a polygon whose offset edges reverse (eroded away) is dropped. The product
// restates exactly this (sbh::erode_convex). Concave or holed input throws.
template <class Poly, class D, class... Rest>
void buffer(const model::multi_polygon<Poly>& in, model::multi_polygon<Poly>& out,
            const strategy::buffer::distance_symmetric<D>& dist, Rest&&...) {
  const double r = -static_cast<double>(dist.value);
  if (!(r > 0.0)) throw std::runtime_error("boost shim: buffer supports erosion only");
  for (const auto& poly : in) {
    if (!poly.inners().empty()) throw std::runtime_error("boost shim: erosion of a holed polygon");
    auto ring = shim_detail::open_ring(poly.outer());
    const std::size_t n = ring.size();
    if (n < 3) continue;
    std::vector<double> ax(n), ay(n), dx(n), dy(n);
    for (std::size_t i = 0; i < n; ++i) {
      const auto& p = ring[i];
      const auto& q = ring[(i + 1) % n];
      const auto& o = ring[(i + n - 1) % n];
      const double cr = (p.v[0] - o.v[0]) * (q.v[1] - o.v[1]) - (p.v[1] - o.v[1]) * (q.v[0] - o.v[0]);
      if (cr < 0.0) throw std::runtime_error("boost shim: erosion of a concave polygon");
      dx[i] = q.v[0] - p.v[0];
      dy[i] = q.v[1] - p.v[1];
      const double len = std::sqrt(dx[i] * dx[i] + dy[i] * dy[i]);
      ax[i] = p.v[0] + (-dy[i] / len) * r;
      ay[i] = p.v[1] + (dx[i] / len) * r;
    }
    Poly res;
    for (std::size_t i = 0; i < n; ++i) {
      const std::size_t h = (i + n - 1) % n;
      const double den = dx[h] * dy[i] - dy[h] * dx[i];
      const double t = ((ax[i] - ax[h]) * dy[i] - (ay[i] - ay[h]) * dx[i]) / den;
      res.outer().push_back(typename Poly::ring_type::value_type(ax[h] + t * dx[h], ay[h] + t * dy[h]));
    }
    bool alive = true;
    for (std::size_t i = 0; i < n; ++i) {
      const auto& p = res.outer()[i];
      const auto& q = res.outer()[(i + 1) % n];
      if (!((q.v[0] - p.v[0]) * dx[i] + (q.v[1] - p.v[1]) * dy[i] > 0.0)) alive = false;
    }
    if (!alive) continue;
    shim_detail::close_ring(res.outer());
    out.push_back(res);
  }
}
namespace shim_detail {
inline int orient_sign(double ax, double ay, double bx, double by, double cx, double cy) {
  const double c = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
  return c > 0.0 ? 1 : (c < 0.0 ? -1 : 0);
}
// closed segments pq and rs intersect or touch
inline bool segments_meet(double px, double py, double qx, double qy, double rx, double ry,
                          double sx, double sy) {
  const int o1 = orient_sign(px, py, qx, qy, rx, ry), o2 = orient_sign(px, py, qx, qy, sx, sy);
  const int o3 = orient_sign(rx, ry, sx, sy, px, py), o4 = orient_sign(rx, ry, sx, sy, qx, qy);
  if (o1 != o2 && o3 != o4) return true;  // crossing, or an endpoint on the other segment
  auto on = [](double ax, double ay, double bx, double by, double cx, double cy) {
    return std::fmin(ax, bx) <= cx && cx <= std::fmax(ax, bx) && std::fmin(ay, by) <= cy &&
           cy <= std::fmax(ay, by);
  };
  if (o1 == 0 && on(px, py, qx, qy, rx, ry)) return true;
  if (o2 == 0 && on(px, py, qx, qy, sx, sy)) return true;
  if (o3 == 0 && on(rx, ry, sx, sy, px, py)) return true;
  if (o4 == 0 && on(rx, ry, sx, sy, qx, qy)) return true;
  return false;
}
template <class Ring>
bool simple_ring(const Ring& closed) {
  const Ring r = dedupe_ring(open_ring(closed));
  const std::size_t n = r.size();
  if (n < 3) return false;
  for (const auto& p : r)
    if (!std::isfinite(p.v[0]) || !std::isfinite(p.v[1])) return false;
  if (signed_area(r) == 0.0) return false;
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = i + 1; j < n; ++j) {
      if (j == i + 1 || (i == 0 && j == n - 1)) continue;  // adjacent edges share a vertex
      const auto& p = r[i];
      const auto& q = r[(i + 1) % n];
      const auto& a = r[j];
      const auto& b = r[(j + 1) % n];
      if (segments_meet(p.v[0], p.v[1], q.v[0], q.v[1], a.v[0], a.v[1], b.v[0], b.v[1])) return false;
    }
  return true;
}
}  // namespace shim_detail

template <class P, bool CW, bool Cl>
bool is_valid(const model::polygon<P, CW, Cl>& poly) {
  if (!poly.inners().empty()) throw std::runtime_error("boost shim: is_valid of a holed polygon");
  return shim_detail::simple_ring(poly.outer());
}

template <class P, class Poly>
void convex_hull(const model::multi_point<P>& mp, Poly& hull) {
  std::vector<P> pts(mp.begin(), mp.end());
  std::sort(pts.begin(), pts.end(), [](const P& a, const P& b) {
    return a.v[0] < b.v[0] || (a.v[0] == b.v[0] && a.v[1] < b.v[1]);
  });
  std::vector<P> h;
  auto turn = [](const P& o, const P& a, const P& b) {
    return (a.v[0] - o.v[0]) * (b.v[1] - o.v[1]) - (a.v[1] - o.v[1]) * (b.v[0] - o.v[0]);
  };
  for (const P& p : pts) {  // lower hull
    while (h.size() >= 2 && turn(h[h.size() - 2], h[h.size() - 1], p) <= 0.0) h.pop_back();
    h.push_back(p);
  }
  const std::size_t lower = h.size() + 1;
  for (std::size_t i = pts.size(); i-- > 0;) {  // upper hull
    const P& p = pts[i];
    while (h.size() >= lower && turn(h[h.size() - 2], h[h.size() - 1], p) <= 0.0) h.pop_back();
    h.push_back(p);
  }
  if (h.size() > 1) h.pop_back();  // the start point again
  hull.outer() = h;
  hull.inners().clear();
  shim_detail::close_ring(hull.outer());
}

namespace shim_detail {
// splice ring `b` into ring `a` along one shared edge (a: u->v, b: v->u); false if none.
template <class Ring>
bool splice(Ring& a, const Ring& b) {
  const std::size_t na = a.size(), nb = b.size();
  for (std::size_t i = 0; i < na; ++i) {
    const auto& u = a[i];
    const auto& v = a[(i + 1) % na];
    for (std::size_t j = 0; j < nb; ++j) {
      const auto& p = b[j];
      const auto& q = b[(j + 1) % nb];
      if (p.v[0] == v.v[0] && p.v[1] == v.v[1] && q.v[0] == u.v[0] && q.v[1] == u.v[1]) {
        Ring out;
        for (std::size_t k = 0; k <= i; ++k) out.push_back(a[k]);  // ..., u
        // b from q (= u) onwards, skipping u itself, up to p (= v) exclusive
        for (std::size_t k = 2; k < nb; ++k) out.push_back(b[(j + k) % nb]);
        for (std::size_t k = i + 1; k < na; ++k) out.push_back(a[k]);  // v, ...
        a = dedupe_ring(out);
        return true;
      }
    }
  }
  return false;
}
}  // namespace shim_detail

template <class Poly>
void union_(const model::multi_polygon<Poly>& a, const model::multi_polygon<Poly>& b,
            model::multi_polygon<Poly>& out) {
  std::vector<typename Poly::ring_type> parts;
  for (const auto& p : a) {
    if (!p.inners().empty()) throw std::runtime_error("boost shim: union_ of a holed polygon");
    parts.push_back(shim_detail::open_ring(p.outer()));
  }
  for (const auto& p : b) {
    if (!p.inners().empty()) throw std::runtime_error("boost shim: union_ of a holed polygon");
    auto ring = shim_detail::open_ring(p.outer());
    // merge into the first part sharing an edge, then fold any other part that now
    // shares an edge with it
    std::size_t host = parts.size();
    for (std::size_t k = 0; k < parts.size() && host == parts.size(); ++k)
      if (shim_detail::splice(parts[k], ring)) host = k;
    if (host == parts.size()) {
      parts.push_back(ring);
      continue;
    }
    for (bool again = true; again;) {
      again = false;
      for (std::size_t k = 0; k < parts.size(); ++k) {
        if (k == host) continue;
        if (shim_detail::splice(parts[host], parts[k])) {
          parts.erase(parts.begin() + static_cast<std::ptrdiff_t>(k));
          if (k < host) --host;
          again = true;
          break;
        }
      }
    }
  }
  for (auto& r : parts) {
    Poly poly;
    poly.outer() = r;
    shim_detail::close_ring(poly.outer());
    out.push_back(poly);
  }
}
template <class... A>
double distance(A&&...) {
  throw std::runtime_error("boost shim: distance is out of scope");
}

}  // namespace geometry
}  // namespace boost
