// TEST INFRASTRUCTURE ONLY -- the oracle. Never linked into the product.
//
// Builder-written driver around the UNMODIFIED reference sources (compiled in place from
// /root/reference/proj/src by oracle/Makefile against oracle/shim). The reference has no
// engine; this file is the rejection loop SPEC.md:516-542 describes,
// with the ordering choices frozen in DESIGN.md ("Appendix C contract"):
//   1. `active` ascending; attempt 0 = all valid instances, then the still-failing ones.
//   2. salt = placement index; run_seed as given.
//   3. pose = translation(p + z_off * z) * rotation_z(yaw)   (transform.hpp:40-54).
//   4. candidates are checked against every enabled object, fixed ones included.
//   5. accept = update_transform + set_enabled(inst); after K attempts the instance is
//      invalid and later placements skip it.
//   6. placeable == 0 (empty region) counts as a failed attempt (not checked).
//   7. margin 0.
//   8. reachability filter (optional, per placement; "and reachability, if
//      flagged"): placement_filter(map, robot_base, {candidate pose}) before collision;
//      an unreachable candidate is a failed attempt and is not checked.
// Exposes a C ABI (prefix ref_) for ctypes; data layouts come from include/scenebatch_b200.h.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "scenebatch/collision.hpp"
#include "scenebatch/parallel.hpp"
#include "scenebatch/polygon.hpp"
#include "scenebatch/reachability.hpp"
#include "scenebatch/relationships.hpp"
#include "scenebatch/rng.hpp"
#include "scenebatch/sampler.hpp"
#include "scenebatch/scene_graph.hpp"
#include "scenebatch/trimesh.hpp"
#include "scenebatch_b200.h"

using namespace scenebatch;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

#define REF_TRY(...)                                        \
  try {                                                      \
    __VA_ARGS__;                                                  \
    return 0;                                                \
  } catch (const std::invalid_argument& e) {                 \
    return fail(e, SB_ERR_INVALID_ARGUMENT);                 \
  } catch (const std::out_of_range& e) {                     \
    return fail(e, SB_ERR_OUT_OF_RANGE);                     \
  } catch (const std::logic_error& e) {                      \
    return fail(e, SB_ERR_LOGIC);                            \
  } catch (const std::exception& e) {                        \
    return fail(e, SB_ERR_RUNTIME);                          \
  }

Mat4 mat_from(const double* p) {
  Mat4 m;
  for (int k = 0; k < 16; ++k) m.data()[k] = p[k];
  return m;
}
void mat_to(const Mat4& m, double* p) {
  for (int k = 0; k < 16; ++k) p[k] = m.data()[k];
}

TriMesh mesh_from(const double* v, uint32_t nv, const uint32_t* t, uint32_t nt) {
  TriMesh m;
  m.vertices.reserve(nv);
  for (uint32_t i = 0; i < nv; ++i) m.vertices.emplace_back(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
  m.triangles.reserve(nt);
  for (uint32_t i = 0; i < nt; ++i) m.triangles.push_back({t[3 * i], t[3 * i + 1], t[3 * i + 2]});
  return m;
}

void mesh_out(const TriMesh& m, double* v, uint32_t* nv, uint32_t* t, uint32_t* nt) {
  if (nv) *nv = static_cast<uint32_t>(m.vertices.size());
  if (nt) *nt = static_cast<uint32_t>(m.triangles.size());
  if (v)
    for (std::size_t i = 0; i < m.vertices.size(); ++i)
      for (int c = 0; c < 3; ++c) v[3 * i + c] = m.vertices[i][c];
  if (t)
    for (std::size_t i = 0; i < m.triangles.size(); ++i)
      for (int c = 0; c < 3; ++c) t[3 * i + c] = m.triangles[i][c];
}

struct RefWorld {
  CollisionWorld world;
  std::unique_ptr<ThreadPool> pool;
  RefWorld(std::size_t n, double margin, int threads) : world(n, margin) {
    if (threads != 1) pool = std::make_unique<ThreadPool>(threads);
  }
};

// RelationshipSpec::anchors of an sb_relation: {anchor, extra_anchors...}
std::vector<int32_t> anchors_of(const sb_relation& r) {
  std::vector<int32_t> out;
  if (r.anchor < 0) return out;
  out.push_back(r.anchor);
  if (r.n_extra_anchors < 0 || r.n_extra_anchors > SB_MAX_ANCHORS - 1)
    throw std::invalid_argument("relationship: n_extra_anchors outside [0, 7]");
  for (int k = 0; k < r.n_extra_anchors; ++k) out.push_back(r.extra_anchors[k]);
  return out;
}

// the support polygon of an sb_support: the rect (make_rect order) or the given ring
MultiPolygon2D support_region_of(const sb_support& sup) {
  if (sup.n_polygon == 0)
    return MultiPolygon2D::from(make_rect(sup.rect[0], sup.rect[1], sup.rect[2], sup.rect[3]));
  if (sup.n_polygon < 3 || !sup.polygon_xy) throw std::invalid_argument("support polygon needs >= 3 vertices");
  Polygon2D p;
  for (uint32_t k = 0; k < sup.n_polygon; ++k)
    p.exterior.emplace_back(sup.polygon_xy[2 * k], sup.polygon_xy[2 * k + 1]);
  return MultiPolygon2D::from(p);
}

RelationshipSpec spec_from(const sb_relation& r) {
  RelationshipSpec s;
  s.kind = SurfaceMode::on;
  for (int32_t a : anchors_of(r)) s.anchors.push_back("p" + std::to_string(a));
  s.distance_type = static_cast<DistanceType>(r.distance_type);
  s.direction = static_cast<DirectionKind>(r.direction);
  s.frame = static_cast<DirectionFrame>(r.frame);
  s.direction_vector = Vec2(r.direction_vector[0], r.direction_vector[1]);
  s.distance = r.distance;
  if (r.angle_threshold > 0.0) s.angle_threshold = r.angle_threshold;
  return s;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- RNG / geometry KATs
uint64_t ref_mix64(uint64_t x) { return mix64(x); }
uint64_t ref_stream_key2(uint64_t a, uint64_t b) { return stream_key({a, b}); }
uint64_t ref_stream_key3(uint64_t a, uint64_t b, uint64_t c) { return stream_key({a, b, c}); }
uint64_t ref_pcg_next_u64(uint64_t seed) {
  Pcg32 r(seed);
  return r.next_u64();
}
void ref_pcg_u32s(uint64_t seed, uint32_t* out, uint32_t n) {
  Pcg32 r(seed);
  for (uint32_t i = 0; i < n; ++i) out[i] = r.next_u32();
}
// make_stream(seed, {c...}) then n next_double()
void ref_stream_doubles(uint64_t seed, const uint64_t* c, uint32_t nc, double* out, uint32_t n) {
  uint64_t h = mix64(seed);
  for (uint32_t i = 0; i < nc; ++i) h = mix64(h ^ c[i]);
  Pcg32 r(h);
  for (uint32_t i = 0; i < n; ++i) out[i] = r.next_double();
}

int ref_make_box(double sx, double sy, double sz, double* v, uint32_t* nv, uint32_t* t,
                 uint32_t* nt) {
  REF_TRY(mesh_out(make_box(sx, sy, sz), v, nv, t, nt));
}
int ref_make_cylinder(double r, double h, int seg, double* v, uint32_t* nv, uint32_t* t,
                      uint32_t* nt) {
  REF_TRY(mesh_out(make_cylinder(r, h, seg), v, nv, t, nt));
}
int ref_make_sphere(double r, int st, int sl, double* v, uint32_t* nv, uint32_t* t,
                    uint32_t* nt) {
  REF_TRY(mesh_out(make_sphere(r, st, sl), v, nv, t, nt));
}
uint64_t ref_mesh_fingerprint(const double* v, uint32_t nv, const uint32_t* t, uint32_t nt) {
  return mesh_fingerprint(mesh_from(v, nv, t, nt));
}
int ref_tri_tri(const double* p /*18*/) {
  Vec3 a(p[0], p[1], p[2]), b(p[3], p[4], p[5]), c(p[6], p[7], p[8]);
  Vec3 d(p[9], p[10], p[11]), e(p[12], p[13], p[14]), f(p[15], p[16], p[17]);
  return tri_tri_intersect(a, b, c, d, e, f) ? 1 : 0;
}
// Batched tri_tri_intersect over n sextuples (18 doubles each).
void ref_tri_tri_batch(const double* p, uint64_t n, uint8_t* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = static_cast<uint8_t>(ref_tri_tri(p + 18 * i));
}
// PolygonSampler over one region (rect or polygon ring), n draws from make_stream(seed,{c})
int ref_polygon_draws(const double* ring, uint32_t nring, uint64_t seed, const uint64_t* c,
                      uint32_t nc, double* out, uint32_t n) {
  REF_TRY({
    Polygon2D poly;
    for (uint32_t i = 0; i < nring; ++i) poly.exterior.emplace_back(ring[2 * i], ring[2 * i + 1]);
    PolygonSampler s(MultiPolygon2D::from(poly));
    uint64_t h = mix64(seed);
    for (uint32_t i = 0; i < nc; ++i) h = mix64(h ^ c[i]);
    Pcg32 r(h);
    for (uint32_t i = 0; i < n; ++i) {
      Vec2 q = s.draw(r);
      out[2 * i] = q.x();
      out[2 * i + 1] = q.y();
    }
  });
}
// triangulate(ring) -> up to max_tris triangles (6 doubles each); returns count via *nt.
int ref_triangulate(const double* ring, uint32_t nring, double* out, uint32_t max_tris,
                    uint32_t* nt) {
  REF_TRY({
    Polygon2D poly;
    for (uint32_t i = 0; i < nring; ++i) poly.exterior.emplace_back(ring[2 * i], ring[2 * i + 1]);
    auto tris = triangulate(poly);
    *nt = static_cast<uint32_t>(tris.size());
    for (std::size_t i = 0; i < tris.size() && i < max_tris; ++i)
      for (int k = 0; k < 3; ++k) {
        out[6 * i + 2 * k] = tris[i][k].x();
        out[6 * i + 2 * k + 1] = tris[i][k].y();
      }
  });
}
uint64_t ref_region_fingerprint_rect(double x0, double y0, double x1, double y1) {
  return region_fingerprint(MultiPolygon2D::from(make_rect(x0, y0, x1, y1)));
}
// region_for(0): build_constraint_region(spec, support, {anchor states}, 1) +
// apply_ratio_on_support(ratio, footprint fx x fy) (relationships.cpp:161-230), then n draws
// of PolygonSampler(region) from Pcg32(make_stream(seed, c)). states: (x, y, yaw) per
// anchor. *ntri = triangle count of the region's sampler (0: empty region).
int ref_region_draws(const sb_relation* rel, const sb_support* sup, const double* states,
                     double ratio, double fx, double fy, uint64_t seed, const uint64_t* c,
                     uint32_t nc, double* out, uint32_t n, int32_t* ntri) {
  REF_TRY({
    RelationshipSpec spec = spec_from(*rel);
    MultiPolygon2D support = support_region_of(*sup);
    std::vector<std::vector<AnchorState>> anchors;
    const std::size_t na = anchors_of(*rel).size();
    for (std::size_t a = 0; a < na; ++a) {
      AnchorState s;
      s.position = Vec2(states[3 * a], states[3 * a + 1]);
      s.yaw = states[3 * a + 2];
      anchors.push_back({s});
    }
    ConstraintRegion cr = build_constraint_region(spec, support, anchors, 1);
    if (ratio != 0.0) apply_ratio_on_support(cr, fx, fy, ratio);
    PolygonSampler ps(cr.region);
    *ntri = static_cast<int32_t>(ps.triangle_count());
    uint64_t h = mix64(seed);
    for (uint32_t i = 0; i < nc; ++i) h = mix64(h ^ c[i]);
    Pcg32 r(h);
    for (uint32_t i = 0; i < n && ps.valid(); ++i) {
      Vec2 q = ps.draw(r);
      out[2 * i] = q.x();
      out[2 * i + 1] = q.y();
    }
  });
}
// extract_support_surfaces / extract_all_support_surfaces (surface.cpp:53-153) into
// sb_surface records (mode: SB_SURFACE_*).
int ref_extract_support_surfaces(const double* v, uint32_t nv, const uint32_t* t, uint32_t nt,
                                 int32_t mode, sb_surface* out, uint32_t cap, uint32_t* n_out) {
  REF_TRY({
    TriMesh m = mesh_from(v, nv, t, nt);
    std::vector<SupportSurface> ss = mode == SB_SURFACE_ALL
                                         ? extract_all_support_surfaces(m)
                                         : extract_support_surfaces(m, static_cast<SurfaceMode>(mode));
    *n_out = static_cast<uint32_t>(ss.size());
    for (std::size_t k = 0; k < ss.size() && k < cap; ++k) {
      sb_surface& o = out[k];
      std::memset(&o, 0, sizeof o);
      for (int c = 0; c < 4; ++c)
        for (int r = 0; r < 4; ++r) o.frame[4 * c + r] = ss[k].frame(r, c);
      o.area = ss[k].area;
      o.roofed = ss[k].roofed ? 1 : 0;
      const auto& ext = ss[k].polygon.exterior;
      if (ext.size() > SB_MAX_SURFACE_VERTS) throw std::invalid_argument("surface polygon too large");
      o.n_polygon = static_cast<uint32_t>(ext.size());
      for (std::size_t i = 0; i < ext.size(); ++i) {
        o.polygon_xy[2 * i] = ext[i].x();
        o.polygon_xy[2 * i + 1] = ext[i].y();
      }
    }
  });
}
// middle_polygon (relationships.cpp:124-157) of n points -> exterior ring.
int ref_middle_polygon(const double* xy, uint32_t n, double* out, uint32_t cap, uint32_t* nout) {
  REF_TRY({
    std::vector<Vec2> pts;
    for (uint32_t i = 0; i < n; ++i) pts.emplace_back(xy[2 * i], xy[2 * i + 1]);
    Polygon2D p = middle_polygon(pts);
    *nout = static_cast<uint32_t>(p.exterior.size());
    for (std::size_t i = 0; i < p.exterior.size() && i < cap; ++i) {
      out[2 * i] = p.exterior[i].x();
      out[2 * i + 1] = p.exterior[i].y();
    }
  });
}
// build_constraint_region for one anchor state, return the region's exterior ring(s).
// out: flattened xy of part 0 exterior (max_pts), *npts, *nparts.
int ref_relation_region(const sb_relation* rel, const double* rect, double ax, double ay,
                        double ayaw, double* out, uint32_t max_pts, uint32_t* npts,
                        uint32_t* nparts) {
  REF_TRY({
    RelationshipSpec spec = spec_from(*rel);
    MultiPolygon2D support = MultiPolygon2D::from(make_rect(rect[0], rect[1], rect[2], rect[3]));
    std::vector<std::vector<AnchorState>> anchors;
    if (rel->anchor >= 0) {
      AnchorState s;
      s.position = Vec2(ax, ay);
      s.yaw = ayaw;
      anchors.push_back({s});
    }
    ConstraintRegion cr = build_constraint_region(spec, support, anchors, 1);
    *nparts = static_cast<uint32_t>(cr.region.parts.size());
    *npts = 0;
    if (!cr.region.parts.empty()) {
      const auto& ext = cr.region.parts[0].exterior;
      *npts = static_cast<uint32_t>(ext.size());
      for (std::size_t i = 0; i < ext.size() && i < max_pts; ++i) {
        out[2 * i] = ext[i].x();
        out[2 * i + 1] = ext[i].y();
      }
    }
  });
}


// ---------------------------------------------------------------- PositionSampler (sampler.hpp:71-96)
// Region input: n_rings outer rings (xy, ring_offsets[n_rings + 1] in points); canonical
// region = all rings; per_instance: instance i's region = rings [inst_rings[i], inst_rings[i+1]).
struct RefSampler {
  PositionSampler sampler;
  ConstraintRegion region;
  explicit RefSampler(uint64_t salt) : sampler(salt) {}
};
static MultiPolygon2D rings_to_region(const double* xy, const uint32_t* off, uint32_t r0, uint32_t r1) {
  MultiPolygon2D m;
  for (uint32_t r = r0; r < r1; ++r) {
    Polygon2D poly;
    for (uint32_t k = off[r]; k < off[r + 1]; ++k) poly.exterior.emplace_back(xy[2 * k], xy[2 * k + 1]);
    m.parts.push_back(std::move(poly));
  }
  return m;
}
void* ref_sampler_create(uint64_t salt) { return new RefSampler(salt); }
void ref_sampler_destroy(void* h) { delete static_cast<RefSampler*>(h); }
int ref_sampler_prepare(void* h, const double* xy, const uint32_t* ring_offsets, uint32_t n_rings,
                        const uint32_t* inst_rings, uint64_t n, uint64_t run_seed) {
  REF_TRY({
    RefSampler& s = *static_cast<RefSampler*>(h);
    s.region = ConstraintRegion();
    if (inst_rings) {
      s.region.per_instance = true;
      for (uint64_t i = 0; i < n; ++i)
        s.region.regions_by_instance.push_back(rings_to_region(xy, ring_offsets, inst_rings[i], inst_rings[i + 1]));
      s.region.region = s.region.regions_by_instance.empty() ? MultiPolygon2D() : s.region.regions_by_instance[0];
    } else {
      s.region.region = rings_to_region(xy, ring_offsets, 0, n_rings);
    }
    s.sampler.prepare(&s.region, n, run_seed);
  });
}
// build_constraint_region(spec, rect, {states}, n) (relationships.cpp:161-218) + prepare;
// states: n x (x, y, yaw); rel->anchor < 0: no anchors (region = the support rect).
int ref_sampler_prepare_relation(void* h, const sb_relation* rel, const double* rect,
                                 const double* states, uint64_t n, uint64_t run_seed) {
  REF_TRY({
    RefSampler& s = *static_cast<RefSampler*>(h);
    RelationshipSpec spec = spec_from(*rel);
    MultiPolygon2D support = MultiPolygon2D::from(make_rect(rect[0], rect[1], rect[2], rect[3]));
    std::vector<std::vector<AnchorState>> anchors;
    if (rel->anchor >= 0) {
      std::vector<AnchorState> a(n);
      for (uint64_t i = 0; i < n; ++i) {
        a[i].position = Vec2(states[3 * i], states[3 * i + 1]);
        a[i].yaw = states[3 * i + 2];
      }
      anchors.push_back(std::move(a));
    }
    s.region = build_constraint_region(spec, support, anchors, n);
    s.sampler.prepare(&s.region, n, run_seed);
  });
}
// support16: N column-major Mat4; positions: 3 per active entry
int ref_sampler_sample(void* h, const double* support16, uint64_t n, const uint32_t* active,
                       uint64_t m, uint64_t attempt, double* positions, uint8_t* placeable,
                       uint64_t* refill_count) {
  REF_TRY({
    RefSampler& s = *static_cast<RefSampler*>(h);
    TransformBatch sw(n);
    for (uint64_t i = 0; i < n; ++i)
      for (int c = 0; c < 4; ++c)
        for (int r = 0; r < 4; ++r) sw[i](r, c) = support16[16 * i + 4 * c + r];
    std::vector<Vec3> pos;
    std::vector<uint8_t> pl;
    s.sampler.sample(sw, std::span<const uint32_t>(active, m), attempt, pos, pl);
    for (uint64_t j = 0; j < m; ++j) {
      positions[3 * j] = pos[j].x();
      positions[3 * j + 1] = pos[j].y();
      positions[3 * j + 2] = pos[j].z();
      placeable[j] = pl[j];
    }
    if (refill_count) *refill_count = s.sampler.cache().refill_count;
  });
}
// sample_orientations (sampler.cpp:129-156); kind 0 fixed, 1 uniform_yaw, 2 face_to;
// face_xy: N targets (face_to only)
int ref_sample_orientations(int kind, const uint32_t* active, uint64_t m, const double* positions,
                            const double* face_xy, uint64_t n, uint64_t run_seed, uint64_t salt,
                            uint64_t attempt, double* yaws) {
  REF_TRY({
    OrientationRule rule;
    rule.kind = kind == 1 ? OrientationRule::Kind::uniform_yaw
                          : (kind == 2 ? OrientationRule::Kind::face_to : OrientationRule::Kind::fixed);
    std::vector<Vec3> pos(m);
    for (uint64_t j = 0; j < m; ++j) pos[j] = Vec3(positions[3 * j], positions[3 * j + 1], positions[3 * j + 2]);
    std::vector<Vec2> targets;
    if (face_xy)
      for (uint64_t i = 0; i < n; ++i) targets.emplace_back(face_xy[2 * i], face_xy[2 * i + 1]);
    auto y = sample_orientations(rule, std::span<const uint32_t>(active, m), pos,
                                 face_xy ? &targets : nullptr, run_seed, salt, attempt);
    for (uint64_t j = 0; j < m; ++j) yaws[j] = y[j];
  });
}

// ---------------------------------------------------------------- BatchedSceneGraph
// scene_graph.hpp:33-94 over column-major double[16] batches.
static Mat4 mat_from16(const double* c) {
  Mat4 m;
  for (int col = 0; col < 4; ++col)
    for (int r = 0; r < 4; ++r) m(r, col) = c[4 * col + r];
  return m;
}
static void mat_to16(const Mat4& m, double* c) {
  for (int col = 0; col < 4; ++col)
    for (int r = 0; r < 4; ++r) c[4 * col + r] = m(r, col);
}
void* ref_graph_create(uint64_t n) {
  try {
    return new BatchedSceneGraph(n);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_graph_destroy(void* h) { delete static_cast<BatchedSceneGraph*>(h); }
int ref_graph_add_node(void* h, uint32_t parent, const char* name, int64_t geom, int has_joint,
                       int kind, const double* axis, double lo, double hi, uint32_t* id) {
  REF_TRY({
    std::optional<JointSpec> j;
    if (has_joint)
      j = JointSpec(kind == 1 ? JointSpec::Kind::prismatic : JointSpec::Kind::revolute,
                    Vec3(axis[0], axis[1], axis[2]), lo, hi);
    *id = static_cast<BatchedSceneGraph*>(h)->add_node(NodeId{parent}, name, geom, j).index;
  });
}
int ref_graph_set_edge_batch(void* h, uint32_t parent, uint32_t child, const double* t16) {
  REF_TRY({
    auto& g = *static_cast<BatchedSceneGraph*>(h);
    TransformBatch t(g.batch_size());
    for (std::size_t i = 0; i < g.batch_size(); ++i) t[i] = mat_from16(t16 + 16 * i);
    g.set_edge_batch(NodeId{parent}, NodeId{child}, t);
  });
}
int ref_graph_set_edge(void* h, uint32_t child, uint64_t i, const double* m16) {
  REF_TRY(static_cast<BatchedSceneGraph*>(h)->set_edge(NodeId{child}, i, mat_from16(m16)));
}
int ref_graph_edge_batch(void* h, uint32_t child, double* out16) {
  REF_TRY({
    const auto& t = static_cast<BatchedSceneGraph*>(h)->edge_batch(NodeId{child});
    for (std::size_t i = 0; i < t.size(); ++i) mat_to16(t[i], out16 + 16 * i);
  });
}
int ref_graph_set_joint_states(void* h, uint32_t node, const double* v, uint64_t n) {
  REF_TRY(static_cast<BatchedSceneGraph*>(h)->set_joint_states(NodeId{node}, std::span<const double>(v, n)));
}
int ref_graph_joint_states(void* h, uint32_t node, double* out) {
  REF_TRY({
    const auto& v = static_cast<BatchedSceneGraph*>(h)->joint_states(NodeId{node});
    for (std::size_t i = 0; i < v.size(); ++i) out[i] = v[i];
  });
}
int ref_graph_world_poses(void* h, uint32_t node, double* out16) {
  REF_TRY({
    TransformBatch t = static_cast<BatchedSceneGraph*>(h)->world_poses(NodeId{node});
    for (std::size_t i = 0; i < t.size(); ++i) mat_to16(t[i], out16 + 16 * i);
  });
}
int ref_graph_world_pose(void* h, uint32_t node, uint64_t i, double* out16) {
  REF_TRY(mat_to16(static_cast<BatchedSceneGraph*>(h)->world_pose(NodeId{node}, i), out16));
}
int ref_graph_is_tree(void* h) { return static_cast<BatchedSceneGraph*>(h)->is_tree() ? 1 : 0; }
void ref_graph_mark_invalid(void* h, uint64_t i) { static_cast<BatchedSceneGraph*>(h)->mark_invalid(i); }
uint64_t ref_graph_valid_count(void* h) { return static_cast<BatchedSceneGraph*>(h)->valid_count(); }

// ---------------------------------------------------------------- ReachMap4D
// reachability.hpp:14-94; joints: n x (kind, ax, ay, az, lo, hi)
void* ref_reach_build(uint32_t n_links, const double* origins16, const double* joints,
                      const double* ee16, uint64_t samples, double res, double psi_res,
                      uint64_t seed, int threads) {
  try {
    KinematicChain chain;
    for (uint32_t l = 0; l < n_links; ++l) {
      ChainLink link;
      link.origin = mat_from16(origins16 + 16 * l);
      const double* j = joints + 6 * l;
      link.joint = JointSpec(j[0] == 1.0 ? JointSpec::Kind::prismatic : JointSpec::Kind::revolute,
                             Vec3(j[1], j[2], j[3]), j[4], j[5]);
      chain.links.push_back(link);
    }
    if (ee16) chain.ee_offset = mat_from16(ee16);
    std::unique_ptr<ThreadPool> pool;
    if (threads != 1) pool = std::make_unique<ThreadPool>(threads);
    return new ReachMap4D(ReachMap4D::build(chain, samples, res, psi_res, seed, pool.get()));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_reach_destroy(void* h) { delete static_cast<ReachMap4D*>(h); }
int ref_reach_save(void* h, const char* path) { REF_TRY(static_cast<ReachMap4D*>(h)->save(path)); }
void* ref_reach_load(const char* path) {
  try {
    return new ReachMap4D(ReachMap4D::load(path));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
// out: samples, resolution, psi_resolution, max_radius, cell_count, occupied_cells
void ref_reach_info(void* h, double* out) {
  const ReachMap4D& m = *static_cast<ReachMap4D*>(h);
  out[0] = static_cast<double>(m.sample_count());
  out[1] = m.resolution();
  out[2] = m.psi_resolution();
  out[3] = m.max_radius();
  out[4] = static_cast<double>(m.cell_count());
  out[5] = static_cast<double>(m.occupied_cells());
}
uint32_t ref_reach_cell_samples(void* h, uint64_t ir, uint64_t iz, uint64_t ip) {
  return static_cast<ReachMap4D*>(h)->cell_samples(ir, iz, ip);
}
int ref_reach_query_batch(void* h, const double* base16, const double* targets, uint64_t n,
                          int has_incl, double incl, uint8_t* out) {
  REF_TRY({
    TransformBatch b(n);
    std::vector<Vec3> t(n);
    for (uint64_t i = 0; i < n; ++i) {
      b[i] = mat_from16(base16 + 16 * i);
      t[i] = Vec3(targets[3 * i], targets[3 * i + 1], targets[3 * i + 2]);
    }
    std::optional<double> inc;
    if (has_incl) inc = incl;
    auto r = static_cast<ReachMap4D*>(h)->query_batch(b, t, inc);
    for (uint64_t i = 0; i < n; ++i) out[i] = r[i];
  });
}
// frames16: n_frames x N x 16 (contiguous); present[f] = 0 -> a null frame
int ref_reach_placement_filter(void* h, const double* base16, uint64_t n, const double* frames16,
                               const uint8_t* present, uint32_t n_frames, const uint32_t* active,
                               uint64_t m, uint8_t* out) {
  REF_TRY({
    TransformBatch b(n);
    for (uint64_t i = 0; i < n; ++i) b[i] = mat_from16(base16 + 16 * i);
    std::vector<TransformBatch> fr(n_frames, TransformBatch(n));
    std::vector<const TransformBatch*> ptr(n_frames, nullptr);
    for (uint32_t f = 0; f < n_frames; ++f) {
      if (!present[f]) continue;
      for (uint64_t i = 0; i < n; ++i) fr[f][i] = mat_from16(frames16 + 16 * (f * n + i));
      ptr[f] = &fr[f];
    }
    auto r = placement_filter(*static_cast<ReachMap4D*>(h), b, ptr, std::span<const uint32_t>(active, m));
    for (uint64_t j = 0; j < m; ++j) out[j] = r[j];
  });
}

// ---------------------------------------------------------------- CollisionWorld
void* ref_world_create(uint64_t n, double margin, int threads) {
  try {
    return new RefWorld(n, margin, threads);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_world_destroy(void* h) { delete static_cast<RefWorld*>(h); }
int ref_register_geometry(void* h, const double* v, uint32_t nv, const uint32_t* t, uint32_t nt,
                          int32_t* id) {
  REF_TRY(*id = static_cast<RefWorld*>(h)->world.register_geometry(mesh_from(v, nv, t, nt)));
}
int ref_add_object(void* h, int32_t geom, int32_t* id) {
  REF_TRY(*id = static_cast<RefWorld*>(h)->world.add_object("o", geom));
}
int ref_set_enabled(void* h, int32_t obj, const uint32_t* inst, uint64_t n, int flag) {
  REF_TRY(static_cast<RefWorld*>(h)->world.set_enabled(obj, std::span<const uint32_t>(inst, n),
                                                       flag != 0));
}
int ref_set_enabled_all(void* h, int32_t obj, int flag) {
  REF_TRY(static_cast<RefWorld*>(h)->world.set_enabled_all(obj, flag != 0));
}
int ref_update_transforms(void* h, int32_t obj, const double* poses) {
  REF_TRY({
    RefWorld* w = static_cast<RefWorld*>(h);
    TransformBatch b(w->world.batch_size());
    for (std::size_t i = 0; i < b.size(); ++i) b[i] = mat_from(poses + 16 * i);
    w->world.update_transforms(obj, b);
  });
}
int ref_update_transform(void* h, int32_t obj, uint64_t inst, const double* pose) {
  REF_TRY(static_cast<RefWorld*>(h)->world.update_transform(obj, inst, mat_from(pose)));
}
int ref_check_batch(void* h, int32_t geom, const double* poses, const uint32_t* active,
                    uint64_t m, uint8_t* free_out, int32_t* contact_out) {
  REF_TRY({
    RefWorld* w = static_cast<RefWorld*>(h);
    std::vector<Mat4> p(m);
    for (uint64_t j = 0; j < m; ++j) p[j] = mat_from(poses + 16 * j);
    CollisionMask mask = w->world.check_batch(geom, p, std::span<const uint32_t>(active, m),
                                              w->pool.get());
    std::memcpy(free_out, mask.free.data(), mask.free.size());
    std::memcpy(contact_out, mask.contact_object.data(), mask.contact_object.size() * 4);
  });
}
void ref_get_stats(void* h, uint64_t* out) {
  const CollisionStats& s = static_cast<RefWorld*>(h)->world.stats();
  out[0] = s.geometry_registrations;
  out[1] = s.bvh_builds;
  out[2] = s.check_calls;
  out[3] = s.checked_instances;
  out[4] = s.narrow_phase_tests;
  out[5] = s.triangle_pair_tests;
}

// ---------------------------------------------------------------- generation driver
// Optional per-round trace (debugging parity): global instance ids, candidate poses,
// placeable flags, free flags per active slot.
// ---------------------------------------------------------------- fused reachability filter
// Appendix C item 8 (driver contract): placement -> (map, robot base per GLOBAL instance).
struct RefReach {
  const ReachMap4D* map;
  std::vector<Mat4> base;
};
static std::map<uint32_t, RefReach> g_reach;
extern "C" int ref_set_reach_filter(uint32_t placement, void* map, const double* base16,
                                    uint64_t n_total) {
  REF_TRY({
    if (!map) {
      g_reach.erase(placement);
      return 0;
    }
    RefReach r{static_cast<ReachMap4D*>(map), std::vector<Mat4>(n_total)};
    for (uint64_t i = 0; i < n_total; ++i) r.base[i] = mat_from16(base16 + 16 * i);
    g_reach[placement] = std::move(r);
  });
}
extern "C" void ref_clear_reach_filters() { g_reach.clear(); }

typedef void (*ref_trace_fn)(void* ctx, int32_t placement, int32_t attempt, uint64_t m,
                             const uint32_t* active_global, const double* poses16,
                             const uint8_t* placeable, const uint8_t* free_by_slot);

// The rejection loop, split as the reference's SPEC splits it:
// RefEngine's constructor is the cold part (RefWorld + ThreadPool, geometry registration
// with its BVH builds, object creation); generate() is one warm run -- the only part
// bench.py times. shard may be NULL (whole batch). threads: ThreadPool size (0 = hardware
// concurrency, 1 = serial). Outputs follow sb_result (local instances).
struct RefEngine {
  uint64_t n_total = 0, begin = 0, end = 0;
  int rank = 0, world_size = 1;
  sb_allgather_fn ag = nullptr;
  void* ag_ctx = nullptr;
  std::size_t n_local = 0;
  int K = 0;
  std::vector<sb_fixed_object> fixed;
  std::vector<sb_support> supports;
  std::vector<sb_placement> placements;
  RefWorld w;
  std::vector<TriMesh> meshes;
  std::vector<int> geom_of_mesh;
  std::vector<int> obj_of_placement;
  std::vector<std::vector<double>> support_batches;

  static std::size_t local_size(const sb_scene* sc, const sb_shard* shard) {
    if (!sc) throw std::invalid_argument("scene is NULL");
    const uint64_t b = shard ? shard->begin : 0, e = shard ? shard->end : sc->n_instances;
    if (b > e || e > sc->n_instances) throw std::invalid_argument("bad shard range");
    if (e == b) throw std::invalid_argument("empty shard");
    return e - b;
  }

  RefEngine(const sb_scene* sc, const sb_shard* shard, int threads)
      : w(local_size(sc, shard), 0.0, threads) {
    n_total = sc->n_instances;
    begin = 0;
    end = n_total;
    if (shard) {
      begin = shard->begin;
      end = shard->end;
      rank = shard->rank;
      world_size = shard->world_size;
      ag = shard->allgather;
      ag_ctx = shard->ctx;
    }
    n_local = end - begin;
    if (world_size > 1 && !ag) throw std::invalid_argument("sharded run needs an allgather callback");
    K = sc->attempts;
    fixed.assign(sc->fixed, sc->fixed + sc->n_fixed);
    supports.assign(sc->supports, sc->supports + sc->n_supports);
    placements.assign(sc->placements, sc->placements + sc->n_placements);
    for (uint32_t i = 0; i < sc->n_meshes; ++i) {
      const sb_mesh& m = sc->meshes[i];
      meshes.push_back(mesh_from(m.vertices, m.n_vertices, m.triangles, m.n_triangles));
      geom_of_mesh.push_back(w.world.register_geometry(meshes.back()));
    }
    for (const sb_fixed_object& f : fixed) {
      int obj = w.world.add_object("fixed", geom_of_mesh.at(f.mesh));
      if (f.poses16) {  // per-instance TransformBatch (GLOBAL order; this shard's range)
        TransformBatch b(n_local);
        for (std::size_t i = 0; i < n_local; ++i) b[i] = mat_from(f.poses16 + 16 * (begin + i));
        w.world.update_transforms(obj, b);
      } else {
        w.world.update_transforms(obj, TransformBatch(n_local, mat_from(f.pose)));
      }
      w.world.set_enabled_all(obj, true);
    }
    support_batches.resize(supports.size());
    for (std::size_t k = 0; k < supports.size(); ++k)
      if (supports[k].poses16) {  // keep the caller's support_world batch (global order)
        support_batches[k].assign(supports[k].poses16, supports[k].poses16 + 16 * n_total);
        supports[k].poses16 = support_batches[k].data();
      }
    for (uint32_t p = 0; p < placements.size(); ++p)
      obj_of_placement.push_back(
          w.world.add_object("p" + std::to_string(p), geom_of_mesh.at(placements[p].mesh)));
  }

  std::vector<uint64_t> allgather(std::vector<uint64_t> send) {
    if (world_size == 1) return send;
    std::vector<uint64_t> recv(send.size() * world_size);
    if (ag(ag_ctx, send.data(), static_cast<uint32_t>(send.size()), recv.data()) != 0)
      throw std::runtime_error("allgather callback failed");
    return recv;
  }

  void generate(uint64_t run_seed, sb_result* out, sb_run_stats* st, ref_trace_fn trace,
                void* trace_ctx);
};

void RefEngine::generate(uint64_t run_seed, sb_result* out, sb_run_stats* st,
                         ref_trace_fn trace, void* trace_ctx) {
    // warm reset: every placed object leaves the world, counters restart
    for (int obj : obj_of_placement) w.world.set_enabled_all(obj, false);
    w.world.reset_stats();
    struct {
      uint32_t n_placements;
      const sb_placement* placements;
      const sb_support* supports;
    } scv{static_cast<uint32_t>(placements.size()), placements.data(), supports.data()};
    const auto* sc = &scv;
    std::vector<uint8_t> valid(n_local, 1);
    // K: attempts per placement (member)
    uint64_t rounds = 0, sampled = 0, per_inst = 0;
    if (out && out->accepted)
      for (std::size_t k = 0; k < sc->n_placements * n_local; ++k) out->accepted[k] = -1;

    for (uint32_t p = 0; p < sc->n_placements; ++p) {
      const sb_placement& pl = sc->placements[p];
      const sb_support& sup = sc->supports[pl.support];
      const int obj = obj_of_placement[p];
      const int geom = geom_of_mesh.at(pl.mesh);
      const double z_off = rest_pose(meshes.at(pl.mesh)).z_offset;
      Mat4 sup_pose = mat_from(sup.pose);
      MultiPolygon2D support_region = support_region_of(sup);
      RelationshipSpec spec = spec_from(pl.relation);

      // support_world (sampler.hpp:78-80), GLOBAL instance order: the surface of an earlier
      // placed object (its accepted pose * the surface frame), a given batch (e.g. FK world
      // poses of a drawer times the surface frame), or one pose for all
      TransformBatch support_world(n_total, sup_pose);
      if (sup.on_placement >= 0) {
        const int sobj = obj_of_placement.at(sup.on_placement);
        for (std::size_t i = 0; i < n_local; ++i)
          support_world[begin + i] = w.world.object_pose(sobj, i) * sup_pose;
      } else if (sup.poses16) {
        for (std::size_t i = 0; i < n_total; ++i) support_world[i] = mat_from(sup.poses16 + 16 * i);
      }
      // Anchor states in the support frame, indexed by GLOBAL instance id.
      std::vector<std::vector<AnchorState>> anchors;
      const std::vector<int32_t> anchor_ids = anchors_of(pl.relation);
      if (!anchor_ids.empty()) {
        const std::size_t na = anchor_ids.size();
        std::vector<std::vector<AnchorState>> local(na, std::vector<AnchorState>(n_local));
        for (std::size_t a = 0; a < na; ++a) {
          const int aobj = obj_of_placement.at(anchor_ids[a]);
          for (std::size_t i = 0; i < n_local; ++i) {
            Mat4 rel = inverse_rigid(support_world[begin + i]) * w.world.object_pose(aobj, i);
            local[a][i].position = Vec2(rel(0, 3), rel(1, 3));
            local[a][i].yaw = yaw_of(rel);
          }
        }
        std::vector<std::vector<AnchorState>> all(na, std::vector<AnchorState>(n_total));
        if (world_size == 1) {
          all = local;
        } else {
          // instance 0 lives on rank 0; exchange its anchor states and each rank's vary
          // flag (relationships.cpp:178-186 compares every instance against instance 0).
          std::vector<uint64_t> send(3 * na, 0);
          if (begin == 0)
            for (std::size_t a = 0; a < na; ++a) {
              std::memcpy(&send[3 * a + 0], &local[a][0].position.x(), 8);
              std::memcpy(&send[3 * a + 1], &local[a][0].position.y(), 8);
              std::memcpy(&send[3 * a + 2], &local[a][0].yaw, 8);
            }
          std::vector<uint64_t> recv = allgather(send);  // rank 0's slots first
          std::vector<AnchorState> s0(na);
          bool local_vary = false;
          for (std::size_t a = 0; a < na; ++a) {
            double tmp[3];
            std::memcpy(tmp, &recv[3 * a], 24);
            s0[a].position = Vec2(tmp[0], tmp[1]);
            s0[a].yaw = tmp[2];
            for (std::size_t i = 0; i < n_local; ++i)
              if ((local[a][i].position - s0[a].position).norm() > 1e-12 ||
                  std::abs(local[a][i].yaw - s0[a].yaw) > 1e-12)
                local_vary = true;
          }
          std::vector<uint64_t> flags = allgather({local_vary ? 1ull : 0ull});
          bool global_vary = false;
          for (uint64_t f : flags) global_vary = global_vary || f != 0;
          for (std::size_t a = 0; a < na; ++a) {
            for (std::size_t i = 0; i < n_total; ++i) all[a][i] = s0[a];
            for (std::size_t i = 0; i < n_local; ++i) all[a][begin + i] = local[a][i];
          }
          if (global_vary && !local_vary) {
            // force the per-instance path through a non-local slot (never sampled here)
            std::size_t slot = begin == 0 ? n_total - 1 : 0;
            all[0][slot].position = s0[0].position + Vec2(1.0, 0.0);
          }
        }
        for (auto& a : all) anchors.push_back(std::move(a));
      }
      ConstraintRegion cr = build_constraint_region(spec, support_region, anchors, n_total);
      if (pl.ratio_on_support != 0.0) {  // footprint = the mesh AABB's x / y extents
        const Aabb3 fb = meshes.at(pl.mesh).aabb();
        apply_ratio_on_support(cr, fb.max.x() - fb.min.x(), fb.max.y() - fb.min.y(),
                               pl.ratio_on_support);
      }
      if (cr.per_instance) ++per_inst;
      PositionSampler sampler(p);
      sampler.prepare(&cr, n_total, run_seed);
      OrientationRule rule;
      rule.kind = static_cast<OrientationRule::Kind>(pl.orientation);
      std::vector<Vec2> face_targets;
      if (pl.orientation == SB_ORIENT_FACE_TO) {
        const int tobj = obj_of_placement.at(pl.face_target);
        face_targets.assign(n_total, Vec2(0, 0));
        for (std::size_t i = 0; i < n_local; ++i) {
          const Mat4& tp = w.world.object_pose(tobj, i);
          face_targets[begin + i] = Vec2(tp(0, 3), tp(1, 3));
        }
      }

      std::vector<uint32_t> active;  // GLOBAL ids, ascending
      for (std::size_t i = 0; i < n_local; ++i)
        if (valid[i]) active.push_back(static_cast<uint32_t>(begin + i));

      for (int a = 0; a < K; ++a) {
        // Fast-path stream: this rank's draws start after the lower ranks' draws.
        std::vector<uint64_t> counts = allgather({static_cast<uint64_t>(active.size())});
        uint64_t total = 0, before = 0;
        for (int r = 0; r < world_size; ++r) {
          if (r < rank) before += counts[r];
          total += counts[r];
        }
        if (total == 0) break;
        ++rounds;
        std::vector<Vec3> pos;
        std::vector<uint8_t> placeable;
        const bool fast = sampler.fast_path();
        auto skip = [&](uint64_t k) {
          if (k == 0 || !fast) return;
          std::vector<uint32_t> dummy(k, 0);
          std::vector<Vec3> dp;
          std::vector<uint8_t> dpl;
          sampler.sample(support_world, dummy, a, dp, dpl, nullptr);
        };
        skip(before);
        if (!active.empty()) {
          sampler.sample(support_world, active, a, pos, placeable, w.pool.get());
          sampled += active.size();
        }
        skip(total - before - active.size());
        if (active.empty()) continue;
        std::vector<double> yaws =
            sample_orientations(rule, active, pos, face_targets.empty() ? nullptr : &face_targets,
                                run_seed, p, a);
        std::vector<Mat4> poses(active.size());
        std::vector<Mat4> chk_poses;
        std::vector<uint32_t> chk_local;
        for (std::size_t j = 0; j < active.size(); ++j)
          poses[j] = translation(pos[j] + Vec3(0, 0, z_off)) * rotation_z(yaws[j]);
        // 8. reachability (if set for this placement): placement_filter on the candidate
        //    frame before collision; unreachable = failed attempt, not checked.
        auto rit = g_reach.find(p);
        if (rit != g_reach.end()) {
          TransformBatch rb(active.size()), fr(active.size());
          std::vector<uint32_t> idx(active.size());
          for (std::size_t j = 0; j < active.size(); ++j) {
            rb[j] = rit->second.base[active[j]];
            fr[j] = poses[j];
            idx[j] = static_cast<uint32_t>(j);
          }
          std::vector<const TransformBatch*> frames{&fr};
          auto ok = placement_filter(*rit->second.map, rb, frames, idx);
          for (std::size_t j = 0; j < active.size(); ++j)
            if (!ok[j]) placeable[j] = 0;
        }
        for (std::size_t j = 0; j < active.size(); ++j) {
          if (placeable[j]) {
            chk_poses.push_back(poses[j]);
            chk_local.push_back(static_cast<uint32_t>(active[j] - begin));
          }
        }
        CollisionMask mask;
        if (!chk_local.empty()) mask = w.world.check_batch(geom, chk_poses, chk_local, w.pool.get());
        std::vector<uint32_t> next;
        std::vector<uint8_t> free_by_slot(active.size(), 0);
        for (std::size_t j = 0; j < active.size(); ++j) {
          uint32_t li = static_cast<uint32_t>(active[j] - begin);
          bool ok = placeable[j] && mask.free[li];
          free_by_slot[j] = ok ? 1 : 0;
          if (ok) {
            w.world.update_transform(obj, li, poses[j]);
            uint32_t one[1] = {li};
            w.world.set_enabled(obj, std::span<const uint32_t>(one, 1), true);
            if (out && out->accepted) out->accepted[p * n_local + li] = static_cast<int16_t>(a);
          } else {
            next.push_back(active[j]);
          }
        }
        if (trace) {
          std::vector<double> flat(16 * active.size());
          for (std::size_t j = 0; j < active.size(); ++j) mat_to(poses[j], flat.data() + 16 * j);
          trace(trace_ctx, static_cast<int32_t>(p), a, active.size(), active.data(), flat.data(),
                placeable.data(), free_by_slot.data());
        }
        active.swap(next);
      }
      for (uint32_t g : active) valid[g - begin] = 0;
    }

    if (out) {
      if (out->valid) std::memcpy(out->valid, valid.data(), n_local);
      if (out->poses)
        for (uint32_t p = 0; p < sc->n_placements; ++p)
          for (std::size_t i = 0; i < n_local; ++i)
            mat_to(w.world.object_pose(obj_of_placement[p], i), out->poses + 16 * (p * n_local + i));
    }
    if (st) {
      const CollisionStats& cs = w.world.stats();
      uint64_t nv = 0;
      for (uint8_t v : valid) nv += v;
      st->valid_instances = nv;
      st->candidates_sampled = sampled;
      st->candidate_checks = cs.checked_instances;
      st->narrow_phase_tests = cs.narrow_phase_tests;
      st->triangle_pair_tests = cs.triangle_pair_tests;
      st->rounds = rounds;
      st->per_instance_placements = per_inst;
    }
}

int ref_generate(const sb_scene* sc, const sb_shard* shard, uint64_t run_seed, int threads,
                 sb_result* out, sb_run_stats* st, ref_trace_fn trace, void* trace_ctx) {
  REF_TRY({
    RefEngine e(sc, shard, threads);
    e.generate(run_seed, out, st, trace, trace_ctx);
  });
}

extern "C" void* ref_engine_create(const sb_scene* sc, const sb_shard* shard, int threads) {
  try {
    return new RefEngine(sc, shard, threads);
  } catch (const std::exception& e) {
    fail(e, SB_ERR_INVALID_ARGUMENT);
    return nullptr;
  }
}
extern "C" void ref_engine_destroy(void* h) { delete static_cast<RefEngine*>(h); }
extern "C" int ref_engine_generate(void* h, uint64_t run_seed, sb_result* out, sb_run_stats* st) {
  REF_TRY(static_cast<RefEngine*>(h)->generate(run_seed, out, st, nullptr, nullptr));
}

}  // extern "C"
