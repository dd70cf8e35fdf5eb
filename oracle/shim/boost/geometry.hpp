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
// buffer: erosion (negative distance) of convex hole-free polygons (see below).
// Everything else (union_, distance, is_valid, convex_hull) throws: those paths
// (support-surface extraction, `middle`) are out of scope.
#pragma once

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
  if (rect.size() != 4) throw std::runtime_error("boost shim: clip operand is not a rectangle");
  double x0 = rect[0].v[0], x1 = rect[0].v[0], y0 = rect[0].v[1], y1 = rect[0].v[1];
  for (const auto& p : rect) {
    x0 = std::fmin(x0, p.v[0]);
    x1 = std::fmax(x1, p.v[0]);
    y0 = std::fmin(y0, p.v[1]);
    y1 = std::fmax(y1, p.v[1]);
  }
  for (const auto& p : rect) {
    bool on_x = p.v[0] == x0 || p.v[0] == x1;
    bool on_y = p.v[1] == y0 || p.v[1] == y1;
    if (!on_x || !on_y) throw std::runtime_error("boost shim: clip operand is not axis-aligned");
  }
  for (const auto& poly : a) {
    Poly res;
    res.outer() = shim_detail::clip_rect(poly.outer(), x0, y0, x1, y1);
    if (res.outer().size() < 3 || shim_detail::signed_area(res.outer()) == 0.0) continue;
    for (const auto& h : poly.inners()) {
      auto hc = shim_detail::clip_rect(h, x0, y0, x1, y1);
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
template <class... A>
void union_(A&&...) {
  throw std::runtime_error("boost shim: union_ is out of scope");
}
template <class... A>
double distance(A&&...) {
  throw std::runtime_error("boost shim: distance is out of scope");
}
template <class... A>
bool is_valid(A&&...) {
  throw std::runtime_error("boost shim: is_valid is out of scope");
}
template <class... A>
void convex_hull(A&&...) {
  throw std::runtime_error("boost shim: convex_hull is out of scope");
}

}  // namespace geometry
}  // namespace boost
