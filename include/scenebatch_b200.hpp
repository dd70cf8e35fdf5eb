// scenebatch_b200.hpp -- the reference's C++ class API on top of the C ABI.
//
// Drop-in shape of /root/reference/proj/include/scenebatch/{collision,trimesh,sampler,
// scene_graph,reachability}.hpp plus
// the generation engine the reference specifies but does not ship.
// Header-only; link libscenebatch_b200.so. Errors are rethrown as the reference's
// exception types (std::invalid_argument, std::out_of_range, std::logic_error,
// std::runtime_error; CUDA failures as scenebatch_b200::cuda_error).
//
// Poses are column-major double[16] (Eigen::Matrix4d memory), so a reference
// TransformBatch's data can be passed as `const double*` directly.
#pragma once

#include <array>
#include <optional>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "scenebatch_b200.h"

namespace scenebatch_b200 {

struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(sb_status s) {
  if (s == SB_OK) return;
  std::string msg = sb_last_error();
  switch (s) {
    case SB_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case SB_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case SB_ERR_LOGIC: throw std::logic_error(msg);
    case SB_ERR_CUDA: throw cuda_error(msg);
    default: throw std::runtime_error(msg);
  }
}

using Pose = std::array<double, 16>;  // column-major, like Eigen::Matrix4d::data()

// TriMesh (trimesh.hpp:12-22), flat storage.
struct TriMesh {
  std::vector<double> vertices;    // xyz triples
  std::vector<uint32_t> triangles; // index triples
  uint32_t n_vertices() const { return static_cast<uint32_t>(vertices.size() / 3); }
  uint32_t n_triangles() const { return static_cast<uint32_t>(triangles.size() / 3); }
};

namespace detail {
template <class F, class... A>
TriMesh make(F f, A... a) {
  uint32_t nv = 0, nt = 0;
  check(f(a..., nullptr, &nv, nullptr, &nt));
  TriMesh m;
  m.vertices.resize(3 * nv);
  m.triangles.resize(3 * nt);
  check(f(a..., m.vertices.data(), &nv, m.triangles.data(), &nt));
  return m;
}
}  // namespace detail

// trimesh.hpp:27-32
inline TriMesh make_box(double sx, double sy, double sz) {
  return detail::make(sb_make_box, sx, sy, sz);
}
inline TriMesh make_cylinder(double radius, double height, int segments = 32) {
  return detail::make(sb_make_cylinder, radius, height, segments);
}
inline TriMesh make_sphere(double radius, int stacks = 12, int slices = 16) {
  return detail::make(sb_make_sphere, radius, stacks, slices);
}
// trimesh.hpp:35
inline TriMesh transformed(const TriMesh& m, const Pose& pose) {
  TriMesh out = m;
  check(sb_transform_vertices(pose.data(), out.vertices.data(), out.n_vertices()));
  return out;
}
// trimesh.hpp:38
inline uint64_t mesh_fingerprint(const TriMesh& m) {
  uint64_t fp = 0;
  check(sb_mesh_fingerprint(m.vertices.data(), m.n_vertices(), m.triangles.data(),
                            m.n_triangles(), &fp));
  return fp;
}

// CollisionMask / CollisionStats (collision.hpp:60-72)
struct CollisionMask {
  std::vector<uint8_t> free;
  std::vector<int32_t> contact_object;
};
using CollisionStats = sb_stats;

// CollisionWorld (collision.hpp:76-127), state resident on one B200.
class CollisionWorld {
 public:
  explicit CollisionWorld(std::size_t batch_size, double margin = 0.0, int device = 0)
      : n_(batch_size) {
    check(sb_world_create(batch_size, margin, device, &w_));
  }
  ~CollisionWorld() {
    if (owned_) sb_world_destroy(w_);
  }
  CollisionWorld(const CollisionWorld&) = delete;
  CollisionWorld& operator=(const CollisionWorld&) = delete;

  std::size_t batch_size() const { return n_; }
  int register_geometry(const TriMesh& mesh) {
    int32_t id = -1;
    check(sb_register_geometry(w_, mesh.vertices.data(), mesh.n_vertices(),
                               mesh.triangles.data(), mesh.n_triangles(), &id));
    return id;
  }
  int add_object(const std::string& name, int geom_id) {
    int32_t id = -1;
    check(sb_add_object(w_, name.c_str(), geom_id, &id));
    return id;
  }
  bool enabled(int object, std::size_t instance) const {
    int e = 0;
    check(sb_enabled(w_, object, instance, &e));
    return e != 0;
  }
  void set_enabled(int object, std::span<const uint32_t> instances, bool enabled) {
    check(sb_set_enabled(w_, object, instances.data(), instances.size(), enabled ? 1 : 0));
  }
  void set_enabled_all(int object, bool enabled) {
    check(sb_set_enabled_all(w_, object, enabled ? 1 : 0));
  }
  // poses: N column-major Mat4 (TransformBatch::data memory)
  void update_transforms(int object, const double* poses_colmajor16xN) {
    check(sb_update_transforms(w_, object, poses_colmajor16xN));
  }
  void update_transform(int object, std::size_t instance, const Pose& pose) {
    check(sb_update_transform(w_, object, instance, pose.data()));
  }
  Pose object_pose(int object, std::size_t instance) const {
    Pose p{};
    check(sb_object_pose(w_, object, instance, p.data()));
    return p;
  }
  CollisionMask check_batch(int geom_id, std::span<const Pose> poses,
                            std::span<const uint32_t> active) {
    if (poses.size() != active.size())
      throw std::invalid_argument("check_batch: poses/active size mismatch");
    CollisionMask m;
    m.free.assign(n_, 1);
    m.contact_object.assign(n_, -1);
    check(sb_check_batch(w_, geom_id, poses.empty() ? nullptr : poses[0].data(), active.data(),
                         active.size(), m.free.data(), m.contact_object.data()));
    return m;
  }
  CollisionStats stats() const {
    sb_stats s{};
    check(sb_get_stats(w_, &s));
    return s;
  }
  void reset_stats() { check(sb_reset_stats(w_)); }
  sb_world* handle() const { return w_; }

 private:
  friend class Engine;
  CollisionWorld(sb_world* w, std::size_t n) : w_(w), n_(n), owned_(false) {}
  sb_world* w_ = nullptr;
  std::size_t n_ = 0;
  bool owned_ = true;
};

// The reference's engine (initialize / generate) for one shard.
class Engine {
 public:
  Engine(const sb_scene& scene, const sb_shard* shard = nullptr, int device = 0) {
    check(sb_engine_create(&scene, shard, device, &e_));
  }
  ~Engine() { sb_engine_destroy(e_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  std::size_t local_instances() const { return sb_engine_local_instances(e_); }
  // One full generation; fills `out` (any member may be null) and returns the stats.
  sb_run_stats generate(uint64_t run_seed, sb_result* out = nullptr) {
    sb_run_stats st{};
    check(sb_engine_generate(e_, run_seed, out, &st));
    return st;
  }
  // Placement-stepped run (sb_engine_place): placements [first, first + count) of the run
  // with run_seed; `out` only on the call that completes it. Stats cumulative.
  sb_run_stats place(uint64_t run_seed, uint32_t first, uint32_t count = 1,
                     sb_result* out = nullptr) {
    sb_run_stats st{};
    check(sb_engine_place(e_, run_seed, first, count, out, &st));
    return st;
  }
  void download(sb_result& out) { check(sb_engine_download(e_, &out)); }
  CollisionWorld world() { return CollisionWorld(sb_engine_world(e_), local_instances()); }

 private:
  sb_engine* e_ = nullptr;
};

// Polygon2D / MultiPolygon2D (polygon.hpp:12-24), hole-free parts as xy rings.
using Ring = std::vector<std::array<double, 2>>;
using MultiPolygon2D = std::vector<Ring>;

// PositionSampler (sampler.hpp:66-96) on one B200. prepare() takes the canonical region
// (ConstraintRegion::region) or, via prepare_per_instance, regions_by_instance.
class PositionSampler {
 public:
  explicit PositionSampler(uint64_t placement_salt, int device = 0) {
    check(sb_sampler_create(placement_salt, device, &s_));
  }
  ~PositionSampler() { sb_sampler_destroy(s_); }
  PositionSampler(const PositionSampler&) = delete;
  PositionSampler& operator=(const PositionSampler&) = delete;

  void prepare(const MultiPolygon2D& region, std::size_t batch_size, uint64_t run_seed) {
    std::vector<double> xy;
    std::vector<uint32_t> off;
    flatten(region, xy, off);
    n_ = batch_size;
    check(sb_sampler_prepare(s_, xy.data(), off.data(), static_cast<uint32_t>(region.size()),
                             nullptr, batch_size, run_seed));
  }
  void prepare_per_instance(const std::vector<MultiPolygon2D>& regions, uint64_t run_seed) {
    MultiPolygon2D all;
    std::vector<uint32_t> inst{0};
    for (const auto& r : regions) {
      all.insert(all.end(), r.begin(), r.end());
      inst.push_back(static_cast<uint32_t>(all.size()));
    }
    std::vector<double> xy;
    std::vector<uint32_t> off;
    flatten(all, xy, off);
    n_ = regions.size();
    check(sb_sampler_prepare(s_, xy.data(), off.data(), static_cast<uint32_t>(all.size()),
                             inst.data(), regions.size(), run_seed));
  }
  // build_constraint_region(spec, support rect, {anchor states}, N) + prepare, on the device;
  // anchor_states: N x (x, y, yaw) in the support frame.
  void prepare_relation(const sb_relation& rel, const std::array<double, 4>& support_rect,
                        std::span<const std::array<double, 3>> anchor_states, uint64_t run_seed) {
    n_ = anchor_states.size();
    check(sb_sampler_prepare_relation(s_, &rel, support_rect.data(),
                                      anchor_states.empty() ? nullptr : anchor_states[0].data(),
                                      anchor_states.size(), run_seed));
  }
  // support_world: batch_size column-major Mat4 (TransformBatch::data memory)
  void sample(const double* support_world, std::span<const uint32_t> active, uint64_t attempt,
              std::vector<std::array<double, 3>>& positions, std::vector<uint8_t>& placeable) {
    positions.assign(active.size(), {0.0, 0.0, 0.0});
    placeable.assign(active.size(), 1);
    check(sb_sampler_sample(s_, support_world, active.data(), active.size(), attempt,
                            positions.empty() ? nullptr : positions[0].data(), placeable.data()));
  }
  uint64_t refill_count() const {
    uint64_t q = 0, r = 0;
    check(sb_sampler_cache_info(s_, &q, &r));
    return r;
  }

 private:
  static void flatten(const MultiPolygon2D& region, std::vector<double>& xy,
                      std::vector<uint32_t>& off) {
    off.assign(1, 0);
    for (const auto& ring : region) {
      for (const auto& p : ring) {
        xy.push_back(p[0]);
        xy.push_back(p[1]);
      }
      off.push_back(static_cast<uint32_t>(xy.size() / 2));
    }
  }
  sb_sampler* s_ = nullptr;
  std::size_t n_ = 0;
};

// sample_orientations (sampler.hpp:98-104); kind = SB_ORIENT_*.
inline std::vector<double> sample_orientations(int kind, std::span<const uint32_t> active,
                                               std::span<const std::array<double, 3>> positions,
                                               const std::vector<std::array<double, 2>>* face_targets,
                                               uint64_t run_seed, uint64_t placement_salt,
                                               uint64_t attempt, int device = 0) {
  std::vector<double> yaws(active.size(), 0.0);
  check(sb_sample_orientations(kind, active.data(), active.size(),
                               positions.empty() ? nullptr : positions[0].data(),
                               face_targets ? (*face_targets)[0].data() : nullptr,
                               face_targets ? face_targets->size() : 0, run_seed, placement_salt,
                               attempt, yaws.data(), device));
  return yaws;
}

// JointSpec / BatchedSceneGraph (scene_graph.hpp:19-94), edge batches resident on one B200.
using JointSpec = sb_joint;  // {kind 0 revolute / 1 prismatic, axis, lo, hi}

class BatchedSceneGraph {
 public:
  explicit BatchedSceneGraph(std::size_t batch_size, int device = 0) : n_(batch_size) {
    check(sb_graph_create(batch_size, device, &g_));
  }
  ~BatchedSceneGraph() { sb_graph_destroy(g_); }
  BatchedSceneGraph(const BatchedSceneGraph&) = delete;
  BatchedSceneGraph& operator=(const BatchedSceneGraph&) = delete;

  std::size_t batch_size() const { return n_; }
  uint32_t root() const { return 0; }
  uint32_t add_node(uint32_t parent, const std::string& name, int64_t geometry_id = -1,
                    const JointSpec* joint = nullptr) {
    uint32_t id = 0;
    check(sb_graph_add_node(g_, parent, name.c_str(), geometry_id, joint, &id));
    return id;
  }
  // transforms: batch_size column-major Mat4 (TransformBatch::data memory)
  void set_edge_batch(uint32_t parent, uint32_t child, const double* transforms) {
    check(sb_graph_set_edge_batch(g_, parent, child, transforms));
  }
  void set_edge(uint32_t child, std::size_t instance, const Pose& m) {
    check(sb_graph_set_edge(g_, child, instance, m.data()));
  }
  std::vector<Pose> edge_batch(uint32_t child) const { return batch(sb_graph_edge_batch, child); }
  void set_joint_states(uint32_t node, std::span<const double> values) {
    if (values.size() != n_) throw std::invalid_argument("joint value batch size mismatch");
    check(sb_graph_set_joint_states(g_, node, values.data()));
  }
  std::vector<double> joint_states(uint32_t node) const {
    std::vector<double> v(n_);
    check(sb_graph_joint_states(g_, node, v.data()));
    return v;
  }
  std::vector<Pose> world_poses(uint32_t node) const { return batch(sb_graph_world_poses, node); }
  Pose world_pose(uint32_t node, std::size_t instance) const {
    Pose p{};
    check(sb_graph_world_pose(g_, node, instance, p.data()));
    return p;
  }
  std::optional<uint32_t> find(const std::string& name) const {
    int64_t id = -1;
    check(sb_graph_find(g_, name.c_str(), &id));
    if (id < 0) return std::nullopt;
    return static_cast<uint32_t>(id);
  }
  std::size_t node_count() const { return sb_graph_node_count(g_); }
  bool is_tree() const {
    int t = 0;
    check(sb_graph_is_tree(g_, &t));
    return t != 0;
  }
  std::vector<uint8_t> valid_mask() const {
    std::vector<uint8_t> m(n_);
    check(sb_graph_valid_mask(g_, m.data()));
    return m;
  }
  void mark_invalid(std::size_t instance) { check(sb_graph_mark_invalid(g_, instance)); }
  void reset_validity() { check(sb_graph_reset_validity(g_)); }
  std::size_t valid_count() const {
    uint64_t c = 0;
    check(sb_graph_valid_count(g_, &c));
    return c;
  }
  sb_graph* handle() const { return g_; }

 private:
  template <class F>
  std::vector<Pose> batch(F f, uint32_t node) const {
    std::vector<Pose> out(n_);
    check(f(g_, node, out[0].data()));
    return out;
  }
  sb_graph* g_ = nullptr;
  std::size_t n_ = 0;
};

// ReachMap4D (reachability.hpp:34-94) built and queried on one B200; SBRM v1 files.
class ReachMap4D {
 public:
  static ReachMap4D build(std::span<const sb_chain_link> chain, const Pose& ee_offset,
                          std::size_t samples, double resolution, double psi_resolution,
                          uint64_t seed, int device = 0) {
    ReachMap4D m;
    check(sb_reach_build(chain.data(), static_cast<uint32_t>(chain.size()), ee_offset.data(),
                         samples, resolution, psi_resolution, seed, device, &m.m_));
    return m;
  }
  static ReachMap4D load(const std::string& path, int device = 0) {
    ReachMap4D m;
    check(sb_reach_load(path.c_str(), device, &m.m_));
    return m;
  }
  ReachMap4D(ReachMap4D&& o) noexcept : m_(o.m_) { o.m_ = nullptr; }
  ReachMap4D& operator=(ReachMap4D&& o) noexcept {
    std::swap(m_, o.m_);
    return *this;
  }
  ~ReachMap4D() {
    if (m_) sb_reach_destroy(m_);
  }
  void save(const std::string& path) const { check(sb_reach_save(m_, path.c_str())); }
  sb_reach_info info() const {
    sb_reach_info i{};
    check(sb_reach_get_info(m_, &i));
    return i;
  }
  // targets[i] is a world point checked against base_poses[i]
  std::vector<uint8_t> query_batch(std::span<const Pose> base_poses,
                                   std::span<const std::array<double, 3>> targets,
                                   std::optional<double> inclination = std::nullopt) const {
    if (base_poses.size() != targets.size()) throw std::invalid_argument("query_batch: size mismatch");
    std::vector<uint8_t> out(targets.size());
    if (targets.empty()) return out;
    check(sb_reach_query_batch(m_, base_poses[0].data(), targets[0].data(), targets.size(),
                               inclination ? 1 : 0, inclination.value_or(0.0), out.data()));
    return out;
  }
  sb_reach_map* handle() const { return m_; }

 private:
  ReachMap4D() = default;
  sb_reach_map* m_ = nullptr;
};

// placement_filter(map, robot_base, frames, active) (reachability.cpp:164-190); frames:
// column-major pose batches of robot_base's size, nullptr entries skipped.
inline std::vector<uint8_t> placement_filter(const ReachMap4D& map, std::span<const Pose> robot_base,
                                             std::span<const double* const> frames,
                                             std::span<const uint32_t> active) {
  std::vector<uint8_t> out(active.size());
  if (active.empty()) return out;
  check(sb_reach_placement_filter(map.handle(), robot_base[0].data(), robot_base.size(),
                                  frames.data(), static_cast<uint32_t>(frames.size()),
                                  active.data(), active.size(), out.data()));
  return out;
}

}  // namespace scenebatch_b200
