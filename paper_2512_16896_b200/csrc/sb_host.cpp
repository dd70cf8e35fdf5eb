// Host-side geometry preparation. See sb_host.hpp.
#include <fstream>
#include <sstream>
#include <cstdlib>
#include "sb_host.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <numeric>
#include <stdexcept>

#include "sb_poly.h"

namespace sbh {

uint64_t mix64(uint64_t x) {  // rng.hpp:9-14
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

Mesh make_box(double sx, double sy, double sz) {  // trimesh.cpp:40-53
  Mesh m;
  double x = sx / 2, y = sy / 2, z = sz / 2;
  m.v = {{-x, -y, -z}, {x, -y, -z}, {x, y, -z}, {-x, y, -z},
         {-x, -y, z},  {x, -y, z},  {x, y, z},  {-x, y, z}};
  m.t = {{0, 2, 1}, {0, 3, 2}, {4, 5, 6}, {4, 6, 7}, {0, 1, 5}, {0, 5, 4},
         {2, 3, 7}, {2, 7, 6}, {1, 2, 6}, {1, 6, 5}, {3, 0, 4}, {3, 4, 7}};
  return m;
}

// ---------------------------------------------------------------- Wavefront OBJ subset
Mesh parse_obj(const std::string& text, const std::string& name) {
  Mesh m;
  size_t pos = 0;
  int line_no = 0;
  auto fail = [&](const std::string& what) {
    throw std::runtime_error(name + ":" + std::to_string(line_no) + ": " + what);
  };
  while (pos <= text.size()) {
    size_t end = text.find('\n', pos);
    if (end == std::string::npos) end = text.size();
    std::string line = text.substr(pos, end - pos);
    pos = end + 1;
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    const size_t hash = line.find('#');
    if (hash != std::string::npos) line.resize(hash);
    std::istringstream in(line);
    std::string tag;
    if (!(in >> tag)) {
      if (end == text.size()) break;
      continue;
    }
    if (tag == "v") {
      V3 p{};
      for (int c = 0; c < 3; ++c) {
        std::string tok;
        if (!(in >> tok)) fail("vertex needs 3 coordinates");
        char* e = nullptr;
        p[c] = std::strtod(tok.c_str(), &e);
        if (e == tok.c_str() || *e != '\0' || !std::isfinite(p[c])) fail("bad coordinate '" + tok + "'");
      }
      m.v.push_back(p);
    } else if (tag == "f") {
      std::vector<uint32_t> idx;
      std::string tok;
      while (in >> tok) {
        const std::string head = tok.substr(0, tok.find('/'));
        char* e = nullptr;
        const long long k = std::strtoll(head.c_str(), &e, 10);
        if (head.empty() || *e != '\0' || k == 0) fail("bad face index '" + tok + "'");
        const long long nv = static_cast<long long>(m.v.size());
        const long long i = k > 0 ? k - 1 : nv + k;  // negative: relative to the end
        if (i < 0 || i >= nv) fail("face index " + std::to_string(k) + " out of range");
        idx.push_back(static_cast<uint32_t>(i));
      }
      if (idx.size() < 3) fail("face needs at least 3 vertices");
      for (size_t j = 1; j + 1 < idx.size(); ++j) m.t.push_back({idx[0], idx[j], idx[j + 1]});
    }
    if (end == text.size()) break;
  }
  if (m.t.empty()) throw std::runtime_error(name + ": no faces");
  return m;
}

Mesh load_obj(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error(path + ": cannot open");
  std::ostringstream ss;
  ss << f.rdbuf();
  return parse_obj(ss.str(), path);
}

Mesh make_cylinder(double radius, double height, int segments) {  // trimesh.cpp:55-76
  if (segments < 3) throw std::invalid_argument("make_cylinder: segments must be >= 3");
  Mesh m;
  double h = height / 2;
  for (int i = 0; i < segments; ++i) {
    double a = 2.0 * M_PI * i / segments;
    m.v.push_back({radius * std::cos(a), radius * std::sin(a), -h});
    m.v.push_back({radius * std::cos(a), radius * std::sin(a), h});
  }
  uint32_t bottom_c = static_cast<uint32_t>(m.v.size());
  m.v.push_back({0, 0, -h});
  uint32_t top_c = bottom_c + 1;
  m.v.push_back({0, 0, h});
  for (int i = 0; i < segments; ++i) {
    uint32_t b0 = 2 * i, t0 = 2 * i + 1;
    uint32_t b1 = 2 * ((i + 1) % segments), t1 = b1 + 1;
    m.t.push_back({b0, b1, t1});
    m.t.push_back({b0, t1, t0});
    m.t.push_back({bottom_c, b1, b0});
    m.t.push_back({top_c, t0, t1});
  }
  return m;
}

Mesh make_sphere(double radius, int stacks, int slices) {  // trimesh.cpp:78-104
  if (stacks < 2 || slices < 3) throw std::invalid_argument("make_sphere: stacks>=2, slices>=3");
  Mesh m;
  m.v.push_back({0, 0, radius});
  for (int s = 1; s < stacks; ++s) {
    double phi = M_PI * s / stacks;
    for (int k = 0; k < slices; ++k) {
      double lam = 2.0 * M_PI * k / slices;
      m.v.push_back({radius * std::sin(phi) * std::cos(lam), radius * std::sin(phi) * std::sin(lam),
                     radius * std::cos(phi)});
    }
  }
  uint32_t south = static_cast<uint32_t>(m.v.size());
  m.v.push_back({0, 0, -radius});
  auto ring = [&](int s, int k) -> uint32_t {
    return 1 + static_cast<uint32_t>((s - 1) * slices + (k % slices));
  };
  for (int k = 0; k < slices; ++k) m.t.push_back({0, ring(1, k), ring(1, k + 1)});
  for (int s = 1; s < stacks - 1; ++s)
    for (int k = 0; k < slices; ++k) {
      m.t.push_back({ring(s, k), ring(s + 1, k), ring(s + 1, k + 1)});
      m.t.push_back({ring(s, k), ring(s + 1, k + 1), ring(s, k + 1)});
    }
  for (int k = 0; k < slices; ++k) m.t.push_back({south, ring(stacks - 1, k + 1), ring(stacks - 1, k)});
  return m;
}

uint64_t mesh_fingerprint(const Mesh& m) {  // trimesh.cpp:120-135
  static_assert(sizeof(V3) == 24 && sizeof(std::array<uint32_t, 3>) == 12, "packed layout");
  uint64_t h = 0x6a09e667f3bcc908ULL;
  auto feed = [&h](const void* p, std::size_t bytes) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    for (std::size_t i = 0; i + 8 <= bytes; i += 8) {
      uint64_t w;
      std::memcpy(&w, c + i, 8);
      h = mix64(h ^ w);
    }
  };
  h = mix64(h ^ m.v.size());
  h = mix64(h ^ m.t.size());
  if (!m.v.empty()) feed(m.v.data(), m.v.size() * sizeof(V3));
  if (!m.t.empty()) feed(m.t.data(), m.t.size() * 12);
  return h;
}

namespace {
inline V3 sub(const V3& a, const V3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
inline V3 cross(const V3& a, const V3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
inline double sqnorm(const V3& a) { return a[0] * a[0] + a[1] * a[1] + a[2] * a[2]; }
// std::min / std::max semantics of Eigen's cwiseMin / cwiseMax.
inline void expand(double mn[3], double mx[3], const V3& p) {
  for (int k = 0; k < 3; ++k) {
    mn[k] = std::min(mn[k], p[k]);
    mx[k] = std::max(mx[k], p[k]);
  }
}
constexpr double kInf = std::numeric_limits<double>::infinity();
}  // namespace

std::size_t drop_degenerate(Mesh& m, double area_eps) {  // trimesh.cpp:16-29
  std::size_t before = m.t.size();
  std::vector<std::array<uint32_t, 3>> kept;
  kept.reserve(before);
  for (const auto& t : m.t) {
    if (t[0] >= m.v.size() || t[1] >= m.v.size() || t[2] >= m.v.size()) continue;
    V3 e1 = sub(m.v[t[1]], m.v[t[0]]);
    V3 e2 = sub(m.v[t[2]], m.v[t[0]]);
    if (0.5 * std::sqrt(sqnorm(cross(e1, e2))) <= area_eps) continue;
    kept.push_back(t);
  }
  m.t.swap(kept);
  return before - m.t.size();
}

void mesh_aabb(const Mesh& m, double box[6]) {
  double mn[3] = {kInf, kInf, kInf}, mx[3] = {-kInf, -kInf, -kInf};
  for (const auto& v : m.v) expand(mn, mx, v);
  for (int k = 0; k < 3; ++k) {
    box[k] = mn[k];
    box[3 + k] = mx[k];
  }
}

// ---------------------------------------------------------------------------- BVH
namespace {
struct RefNode {
  double mn[3], mx[3];
  int left = -1;
  uint32_t start = 0, count = 0;
};

struct Builder {
  const Mesh& mesh;
  const std::vector<V3>& centroids;
  std::vector<RefNode>& nodes;
  std::vector<uint32_t>& leaf_tris;  // mesh triangle ids in leaf order (tris_ order)
  int max_depth = 0;

  // collision.cpp:253-276 restated: median split on the longest centroid axis.
  int build(std::vector<uint32_t>& tris, uint32_t begin, uint32_t end, int depth) {
    max_depth = std::max(max_depth, depth);
    int idx = static_cast<int>(nodes.size());
    nodes.emplace_back();
    double mn[3] = {kInf, kInf, kInf}, mx[3] = {-kInf, -kInf, -kInf};
    for (uint32_t i = begin; i < end; ++i) {
      // tri_box then Aabb3::expand(Aabb3): cwiseMin/cwiseMax of the boxes
      double tmn[3] = {kInf, kInf, kInf}, tmx[3] = {-kInf, -kInf, -kInf};
      for (uint32_t vi : mesh.t[tris[i]]) expand(tmn, tmx, mesh.v[vi]);
      for (int k = 0; k < 3; ++k) {
        mn[k] = std::min(mn[k], tmn[k]);
        mx[k] = std::max(mx[k], tmx[k]);
      }
    }
    std::memcpy(nodes[idx].mn, mn, sizeof mn);
    std::memcpy(nodes[idx].mx, mx, sizeof mx);
    if (end - begin <= 4) {
      nodes[idx].start = static_cast<uint32_t>(leaf_tris.size());
      nodes[idx].count = end - begin;
      for (uint32_t i = begin; i < end; ++i) leaf_tris.push_back(tris[i]);
      return idx;
    }
    double cmn[3] = {kInf, kInf, kInf}, cmx[3] = {-kInf, -kInf, -kInf};
    for (uint32_t i = begin; i < end; ++i) expand(cmn, cmx, centroids[tris[i]]);
    double ext[3] = {cmx[0] - cmn[0], cmx[1] - cmn[1], cmx[2] - cmn[2]};
    int axis = 0;
    if (ext[1] > ext[0]) axis = 1;
    if (ext[2] > ext[axis]) axis = 2;
    uint32_t mid = (begin + end) / 2;
    // Same libstdc++ nth_element as the reference build -> same permutation.
    std::nth_element(tris.begin() + begin, tris.begin() + mid, tris.begin() + end,
                     [&](uint32_t a, uint32_t b) { return centroids[a][axis] < centroids[b][axis]; });
    int left = build(tris, begin, mid, depth + 1);
    nodes[idx].left = left;
    build(tris, mid, end, depth + 1);
    return idx;
  }
};
}  // namespace

EffectiveBvh build_effective_bvh(const Mesh& mesh) {
  if (mesh.t.empty()) throw std::invalid_argument("MeshBvh: empty mesh");
  const std::size_t n = mesh.t.size();
  std::vector<V3> centroids(n);
  std::vector<uint32_t> order(n);
  for (std::size_t t = 0; t < n; ++t) {
    const auto& tri = mesh.t[t];
    const V3& a = mesh.v[tri[0]];
    const V3& b = mesh.v[tri[1]];
    const V3& c = mesh.v[tri[2]];
    centroids[t] = {(a[0] + b[0] + c[0]) / 3.0, (a[1] + b[1] + c[1]) / 3.0,
                    (a[2] + b[2] + c[2]) / 3.0};
    order[t] = static_cast<uint32_t>(t);
  }
  std::vector<RefNode> nodes;
  nodes.reserve(2 * n);
  std::vector<uint32_t> leaf_tris;
  leaf_tris.reserve(n);
  Builder b{mesh, centroids, nodes, leaf_tris};
  b.build(order, 0, static_cast<uint32_t>(n), 1);

  // Reachable set under the reference's child indexing {left, left+1}.
  std::vector<char> reach(nodes.size(), 0);
  std::vector<int> stack{0};
  while (!stack.empty()) {
    int i = stack.back();
    stack.pop_back();
    if (reach[i]) continue;
    reach[i] = 1;
    if (nodes[i].left >= 0) {
      stack.push_back(nodes[i].left);
      stack.push_back(nodes[i].left + 1);
    }
  }
  std::vector<int> compact(nodes.size(), -1);
  EffectiveBvh out;
  out.full_nodes = static_cast<int>(nodes.size());
  out.full_depth = b.max_depth;
  for (std::size_t i = 0; i < nodes.size(); ++i)
    if (reach[i]) compact[i] = static_cast<int>(out.nodes.size()), out.nodes.emplace_back();
  for (std::size_t i = 0; i < nodes.size(); ++i) {
    if (!reach[i]) continue;
    const RefNode& r = nodes[i];
    SbNode& d = out.nodes[compact[i]];
    std::memset(&d, 0, sizeof d);
    for (int k = 0; k < 3; ++k) {
      d.bmin[k] = r.mn[k];
      d.bmax[k] = r.mx[k];
      d.c[k] = (r.mn[k] + r.mx[k]) * 0.5;  // Aabb3::center: 0.5 * (min + max)
      d.h[k] = (r.mx[k] - r.mn[k]) * 0.5;  // 0.5 * extent()
    }
    double e0 = r.mx[0] - r.mn[0], e1 = r.mx[1] - r.mn[1], e2 = r.mx[2] - r.mn[2];
    d.ext2 = e0 * e0 + e1 * e1 + e2 * e2;
    if (r.left >= 0) {
      d.child0 = compact[r.left];
      d.child1 = compact[r.left + 1];
      d.tri_start = d.tri_count = 0;
    } else {
      d.child0 = d.child1 = -1;
      d.tri_start = static_cast<int32_t>(out.tris.size());
      d.tri_count = static_cast<int32_t>(r.count);
      for (uint32_t k = 0; k < r.count; ++k) {
        const auto& tri = mesh.t[leaf_tris[r.start + k]];
        SbTri t;
        t.leaf = compact[i];
        t.pad = 0;
        for (int v = 0; v < 3; ++v)
          for (int c = 0; c < 3; ++c) t.v[3 * v + c] = mesh.v[tri[v]][c];
        out.tris.push_back(t);
      }
    }
  }
  // leaves_below: effective leaves under each node (children ids exceed their parent's)
  for (int i = static_cast<int>(out.nodes.size()) - 1; i >= 0; --i) {
    SbNode& d = out.nodes[i];
    d.leaves_below = d.child0 < 0 ? (1u << i)
                                  : (out.nodes[d.child0].leaves_below | out.nodes[d.child1].leaves_below);
  }
  out.reachable_tris = static_cast<int>(out.tris.size());
  return out;
}

// ----------------------------------------------------------------- triangulation
std::vector<std::array<V2, 3>> triangulate_ring(const std::vector<V2>& ring) {
  std::vector<std::array<V2, 3>> tris;
  if (ring.size() < 3 || ring.size() > static_cast<std::size_t>(sbp::kCap))
    throw std::invalid_argument("triangulate_ring: ring size outside [3, capacity]");
  static thread_local sbp::Ring r;
  r.n = static_cast<int>(ring.size());
  for (int i = 0; i < r.n; ++i) {
    r.x[i] = ring[i][0];
    r.y[i] = ring[i][1];
  }
  SbRegionTri buf[sbp::kCap];
  double cum[sbp::kCap];
  // Capture every emitted triangle (the sink drops zero-area ones, so use a raw copy).
  sbp::TableSink sink{buf, cum, 0, sbp::kCap, 0.0};
  // ear_clip_into filters zero-area triangles through the sink; triangulate() itself does
  // not, but PolygonSampler (its only hot-path consumer) does, so tables are identical.
  if (!sbp::ear_clip_into(r, sink)) throw std::runtime_error("triangulate_ring: overflow");
  for (int i = 0; i < sink.n; ++i)
    tris.push_back({V2{buf[i].a[0], buf[i].a[1]}, V2{buf[i].b[0], buf[i].b[1]},
                    V2{buf[i].c[0], buf[i].c[1]}});
  return tris;
}

SamplerTable sampler_table(const std::vector<std::vector<V2>>& part_rings) {
  SamplerTable out;
  std::vector<SbRegionTri> buf(sbp::kCap * part_rings.size() + 1);
  std::vector<double> cum(buf.size());
  sbp::TableSink sink{buf.data(), cum.data(), 0, static_cast<int>(buf.size()), 0.0};
  static thread_local sbp::Ring r;
  for (const auto& ring : part_rings) {
    if (ring.size() < 3) continue;
    if (ring.size() > static_cast<std::size_t>(sbp::kCap))
      throw std::invalid_argument("sampler_table: ring exceeds capacity");
    r.n = static_cast<int>(ring.size());
    for (int i = 0; i < r.n; ++i) {
      r.x[i] = ring[i][0];
      r.y[i] = ring[i][1];
    }
    if (!sbp::ear_clip_into(r, sink)) throw std::runtime_error("sampler_table: overflow");
  }
  int n = sbp::finish_table(sink);
  out.tris.assign(buf.begin(), buf.begin() + n);
  out.cum.assign(cum.begin(), cum.begin() + n);
  return out;
}

std::vector<V2> erode_convex(const std::vector<V2>& ring, double r) {
  const std::size_t n = ring.size();
  if (n < 3) return {};
  std::vector<double> ax(n), ay(n), dx(n), dy(n);
  for (std::size_t i = 0; i < n; ++i) {
    const V2& p = ring[i];
    const V2& q = ring[(i + 1) % n];
    const V2& o = ring[(i + n - 1) % n];
    const double cr = (p[0] - o[0]) * (q[1] - o[1]) - (p[1] - o[1]) * (q[0] - o[0]);
    if (cr < 0.0) throw std::invalid_argument("erode: concave support polygon");
    dx[i] = q[0] - p[0];
    dy[i] = q[1] - p[1];
    const double len = std::sqrt(dx[i] * dx[i] + dy[i] * dy[i]);
    ax[i] = p[0] + (-dy[i] / len) * r;
    ay[i] = p[1] + (dx[i] / len) * r;
  }
  std::vector<V2> out(n);
  for (std::size_t i = 0; i < n; ++i) {
    const std::size_t h = (i + n - 1) % n;
    const double den = dx[h] * dy[i] - dy[h] * dx[i];
    const double t = ((ax[i] - ax[h]) * dy[i] - (ay[i] - ay[h]) * dx[i]) / den;
    out[i] = {ax[h] + t * dx[h], ay[h] + t * dy[h]};
  }
  for (std::size_t i = 0; i < n; ++i) {
    const V2& p = out[i];
    const V2& q = out[(i + 1) % n];
    if (!((q[0] - p[0]) * dx[i] + (q[1] - p[1]) * dy[i] > 0.0)) return {};  // eroded away
  }
  return out;
}


// ------------------------------------------------------------ support-surface extraction
namespace {

struct Pcg32H {  // rng.hpp:24-60
  uint64_t state = 0, inc;
  explicit Pcg32H(uint64_t seed, uint64_t seq = 0xda3e39cb94b95bdbULL) : inc((seq << 1u) | 1u) {
    next_u32();
    state += seed;
    next_u32();
  }
  uint32_t next_u32() {
    const uint64_t old = state;
    state = old * 6364136223846793005ULL + inc;
    const uint32_t xs = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
    const uint32_t rot = static_cast<uint32_t>(old >> 59u);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
  }
  double next_double() {
    const uint64_t hi = next_u32();  // GCC evaluates the left operand first
    const uint64_t w = (hi << 32) | next_u32();
    return static_cast<double>(w >> 11) * 0x1.0p-53;
  }
};

// the shim's ring helpers (oracle/shim/boost/geometry.hpp): exact duplicates only
double shim_signed_area(const std::vector<V2>& r) {
  double s = 0.0;
  const std::size_t n = r.size();
  for (std::size_t i = 0; i < n; ++i) {
    const V2& a = r[i];
    const V2& b = r[(i + 1) % n];
    s += a[0] * b[1] - b[0] * a[1];
  }
  return 0.5 * s;
}
std::vector<V2> shim_dedupe(const std::vector<V2>& r) {
  std::vector<V2> o;
  for (const V2& p : r)
    if (o.empty() || p[0] != o.back()[0] || p[1] != o.back()[1]) o.push_back(p);
  while (o.size() > 1 && o.front()[0] == o.back()[0] && o.front()[1] == o.back()[1]) o.pop_back();
  return o;
}
// to_boost's bg::correct of an open exterior: counter-clockwise, vertex 0 first
std::vector<V2> shim_correct(std::vector<V2> r) {
  std::vector<V2> closed = r;
  if (!closed.empty()) closed.push_back(closed.front());
  if (shim_signed_area(closed) < 0.0) std::reverse(r.begin() + (r.empty() ? 0 : 1), r.end());
  return r;
}
// splice ring b into ring a along one shared edge (a: u->v, b: v->u)
bool shim_splice(std::vector<V2>& a, const std::vector<V2>& b) {
  const std::size_t na = a.size(), nb = b.size();
  for (std::size_t i = 0; i < na; ++i) {
    const V2& u = a[i];
    const V2& v = a[(i + 1) % na];
    for (std::size_t j = 0; j < nb; ++j) {
      const V2& p = b[j];
      const V2& q = b[(j + 1) % nb];
      if (p[0] == v[0] && p[1] == v[1] && q[0] == u[0] && q[1] == u[1]) {
        std::vector<V2> out;
        for (std::size_t k = 0; k <= i; ++k) out.push_back(a[k]);
        for (std::size_t k = 2; k < nb; ++k) out.push_back(b[(j + k) % nb]);
        for (std::size_t k = i + 1; k < na; ++k) out.push_back(a[k]);
        a = shim_dedupe(out);
        return true;
      }
    }
  }
  return false;
}
// union_of(a, b) (polygon.cpp:121-125): to_boost both, the shim's union_, from_boost
std::vector<std::vector<V2>> shim_union(const std::vector<std::vector<V2>>& a,
                                        const std::vector<std::vector<V2>>& b) {
  std::vector<std::vector<V2>> parts;
  for (const auto& p : a) parts.push_back(shim_correct(p));
  for (const auto& q : b) {
    std::vector<V2> ring = shim_correct(q);
    std::size_t host = parts.size();
    for (std::size_t k = 0; k < parts.size() && host == parts.size(); ++k)
      if (shim_splice(parts[k], ring)) host = k;
    if (host == parts.size()) {
      parts.push_back(ring);
      continue;
    }
    for (bool again = true; again;) {
      again = false;
      for (std::size_t k = 0; k < parts.size(); ++k) {
        if (k == host) continue;
        if (shim_splice(parts[host], parts[k])) {
          parts.erase(parts.begin() + static_cast<std::ptrdiff_t>(k));
          if (k < host) --host;
          again = true;
          break;
        }
      }
    }
  }
  std::vector<std::vector<V2>> out;  // from_boost: closed ring -> ring_to_vec, >= 3 points
  for (auto& r : parts) {
    std::vector<V2> v = r;
    if (!v.empty()) v.push_back(v.front());  // close_ring
    if (v.size() > 1) {
      const double dx = v.front()[0] - v.back()[0], dy = v.front()[1] - v.back()[1];
      if (std::sqrt(dx * dx + dy * dy) < 1e-15) v.pop_back();
    }
    if (v.size() >= 3) out.push_back(std::move(v));
  }
  return out;
}

// Moller-Trumbore with a +z ray (surface.cpp:20-37)
double ray_up_hit(const Mesh& m, std::size_t t, const V3& o) {
  const auto& tri = m.t[t];
  const V3& v0 = m.v[tri[0]];
  const V3 e1 = {m.v[tri[1]][0] - v0[0], m.v[tri[1]][1] - v0[1], m.v[tri[1]][2] - v0[2]};
  const V3 e2 = {m.v[tri[2]][0] - v0[0], m.v[tri[2]][1] - v0[1], m.v[tri[2]][2] - v0[2]};
  const V3 pvec = {-e2[1], e2[0], 0.0};
  const double det = e1[0] * pvec[0] + e1[1] * pvec[1] + e1[2] * pvec[2];
  if (std::abs(det) < 1e-14) return -1.0;
  const double inv = 1.0 / det;
  const V3 tv = {o[0] - v0[0], o[1] - v0[1], o[2] - v0[2]};
  const double u = (tv[0] * pvec[0] + tv[1] * pvec[1] + tv[2] * pvec[2]) * inv;
  if (u < -1e-12 || u > 1.0 + 1e-12) return -1.0;
  const V3 q = {tv[1] * e1[2] - tv[2] * e1[1], tv[2] * e1[0] - tv[0] * e1[2],
                tv[0] * e1[1] - tv[1] * e1[0]};
  const double v = q[2] * inv;
  if (v < -1e-12 || u + v > 1.0 + 1e-12) return -1.0;
  return (e2[0] * q[0] + e2[1] * q[1] + e2[2] * q[2]) * inv;
}

}  // namespace

std::vector<Surface> extract_all_support_surfaces(const Mesh& mesh) {
  std::vector<Surface> out;
  if (mesh.t.empty()) return out;
  const double cos_tol = std::cos(5.0 * M_PI / 180.0);
  std::vector<std::size_t> up;
  for (std::size_t t = 0; t < mesh.t.size(); ++t) {  // triangle_normal (trimesh.cpp:31-36)
    const auto& tri = mesh.t[t];
    const V3& a = mesh.v[tri[0]];
    const V3 b = {mesh.v[tri[1]][0] - a[0], mesh.v[tri[1]][1] - a[1], mesh.v[tri[1]][2] - a[2]};
    const V3 c = {mesh.v[tri[2]][0] - a[0], mesh.v[tri[2]][1] - a[1], mesh.v[tri[2]][2] - a[2]};
    const V3 n = {b[1] * c[2] - b[2] * c[1], b[2] * c[0] - b[0] * c[2], b[0] * c[1] - b[1] * c[0]};
    const double len = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    const double nz = len > 0.0 ? n[2] / len : 0.0;
    if (nz >= cos_tol) up.push_back(t);
  }
  if (up.empty()) return out;
  std::vector<int> parent(up.size());  // DisjointSet with path halving
  std::iota(parent.begin(), parent.end(), 0);
  auto find = [&](int x) {
    while (parent[x] != x) x = parent[x] = parent[parent[x]];
    return x;
  };
  using EdgeKey = std::array<int64_t, 6>;
  std::map<EdgeKey, int> edge_owner;
  auto quantize = [](double v) { return static_cast<int64_t>(std::llround(v * 1e9)); };
  for (std::size_t i = 0; i < up.size(); ++i) {
    const auto& tri = mesh.t[up[i]];
    for (int e = 0; e < 3; ++e) {
      const V3& a = mesh.v[tri[e]];
      const V3& b = mesh.v[tri[(e + 1) % 3]];
      const EdgeKey ka{quantize(a[0]), quantize(a[1]), quantize(a[2]),
                       quantize(b[0]), quantize(b[1]), quantize(b[2])};
      const EdgeKey kb{ka[3], ka[4], ka[5], ka[0], ka[1], ka[2]};
      auto [it, inserted] = edge_owner.try_emplace(std::min(ka, kb), static_cast<int>(i));
      if (!inserted) parent[find(it->second)] = find(static_cast<int>(i));
    }
  }
  std::map<int, std::vector<std::size_t>> clusters;
  for (std::size_t i = 0; i < up.size(); ++i) clusters[find(static_cast<int>(i))].push_back(up[i]);
  int cluster_index = 0;
  for (const auto& [root, tris] : clusters) {
    (void)root;
    double z_top = -std::numeric_limits<double>::infinity();
    for (std::size_t t : tris)
      for (uint32_t vi : mesh.t[t]) z_top = std::max(z_top, mesh.v[vi][2]);
    std::vector<std::vector<V2>> merged;
    for (std::size_t t : tris) {
      const auto& tri = mesh.t[t];
      std::vector<V2> p;
      for (int k = 0; k < 3; ++k) p.push_back({mesh.v[tri[k]][0], mesh.v[tri[k]][1]});
      const double a2 = (p[1][0] - p[0][0]) * (p[2][1] - p[0][1]) - (p[1][1] - p[0][1]) * (p[2][0] - p[0][0]);
      if (std::abs(a2) < 1e-14) continue;
      if (a2 < 0.0) std::reverse(p.begin(), p.end());
      merged = merged.empty() ? std::vector<std::vector<V2>>{p} : shim_union(merged, {p});
    }
    for (auto& part : merged) {
      std::vector<V2> closed = shim_correct(part);  // area(MultiPolygon) via to_boost
      closed.push_back(closed.front());
      const double a = std::abs(shim_signed_area(closed));
      if (a < 1e-4) continue;
      Surface s;
      s.z_top = z_top;
      s.area = a;
      const SamplerTable tab = sampler_table({part});  // PolygonSampler(one)
      Pcg32H rng(mix64(mix64(0x853c49e6748fea9bULL ^ 0x726f6f66ULL) ^ static_cast<uint64_t>(cluster_index)));
      int hits = 0, cast = 0;
      for (int i = 0; i < 16 && !tab.tris.empty(); ++i) {
        const double u = rng.next_double(), r1 = rng.next_double(), r2 = rng.next_double();
        double px, py;
        sbp::draw_point(tab.tris.data(), tab.cum.data(), static_cast<int>(tab.tris.size()), u, r1,
                        r2, px, py);
        const V3 origin = {px, py, z_top};
        ++cast;
        for (std::size_t t = 0; t < mesh.t.size(); ++t)
          if (ray_up_hit(mesh, t, origin) > 1e-4) {
            ++hits;
            break;
          }
      }
      s.roofed = cast > 0 && hits * 2 >= cast;
      s.polygon = part;
      out.push_back(std::move(s));
      ++cluster_index;
    }
  }
  std::stable_sort(out.begin(), out.end(), [](const Surface& a, const Surface& b) { return a.area > b.area; });
  return out;
}

}  // namespace sbh
