// Host runtime + C ABI (include/scenebatch_b200.h). C++17, CUDA runtime API only.
//
// World  = CollisionWorld (collision.hpp:76-127) with all per-instance state in HBM.
// Engine = the reference's absent rejection loop (contract frozen in
//          DESIGN.md) driving the fused per-round kernel; one engine per GPU / shard.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/scenebatch_b200.h"
#include "sb_graph.h"
#include "sb_host.hpp"
#include "sb_reach.h"
#include "sb_kernels.h"
#include "sb_place.h"
#include "sb_poly.h"
#include "sb_region.h"
#include "sb_layout.h"

namespace {

thread_local std::string g_error;

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error(std::string("CUDA: ") + what + ": " + cudaGetErrorString(e));
  }
}

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class T>
struct DevArray {
  T* p = nullptr;
  size_t count = 0;
  DevArray() = default;
  DevArray(const DevArray&) = delete;
  DevArray& operator=(const DevArray&) = delete;
  ~DevArray() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    count = 0;
  }
  void alloc(size_t n) {
    release();
    if (n == 0) return;
    cuda_check(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
    count = n;
  }
  void ensure(size_t n) {
    if (n > count) alloc(n);
  }
};

template <class T>
struct PinnedArray {
  T* p = nullptr;
  size_t count = 0;
  ~PinnedArray() {
    if (p) cudaFreeHost(p);
  }
  void ensure(size_t n) {
    if (n <= count) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cuda_check(cudaMallocHost(&p, n * sizeof(T)), "cudaMallocHost");
    count = n;
  }
};

void require_homogeneous(const double* p) {
  if (p[3] != 0.0 || p[7] != 0.0 || p[11] != 0.0 || p[15] != 1.0)
    throw std::invalid_argument("pose bottom row must be exactly (0,0,0,1)");
  for (int k = 0; k < 16; ++k)
    if (!std::isfinite(p[k])) throw std::invalid_argument("pose must be finite");
}

// inverse_rigid (transform.hpp:63-69) on the host, same operation order as the device.
void inverse_rigid34(const double* colmajor16, double out[12]) {
  double R[3][3], t[3];
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) R[i][j] = colmajor16[4 * j + i];
    t[i] = colmajor16[12 + i];
  }
  for (int i = 0; i < 3; ++i) {
    for (int k = 0; k < 3; ++k) out[4 * i + k] = R[k][i];
    double s = (-R[0][i]) * t[0];
    s = s + (-R[1][i]) * t[1];
    s = s + (-R[2][i]) * t[2];
    out[4 * i + 3] = s;
  }
}

void colmajor_to_34(const double* c, double out[12]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 4; ++j) out[4 * i + j] = c[4 * j + i];
}

int current_device_checked(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw CudaError("no CUDA device available (this build has no CPU fallback)");
  }
  if (device < 0 || device >= count) throw std::out_of_range("device index out of range");
  cudaDeviceProp prop;
  cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10)
    throw CudaError("device " + std::to_string(device) + " is sm_" + std::to_string(prop.major) +
                    std::to_string(prop.minor) + "; this build targets sm_100a only");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  return device;
}

// RelationshipSpec::validate (relationships.cpp:59-76) for the single-anchor subset, then
// the relation fields of the device record. Returns whether region_for() needs the serial
// big-ring region path: a full annulus with a hole (theta = pi, min_r > 0, bridged hole) or
// an annular sector wide enough to outgrow the group path's ring (SB_REGION_MAX_VERTS).
bool relation_to_dev(const sb_relation& r, SbPlacementDev& d) {
  if (r.distance < 0.0) throw std::invalid_argument("relationship: distance must be >= 0");
  if (r.angle_threshold > M_PI) throw std::invalid_argument("relationship: angle_threshold outside (0, pi]");
  const bool dist = r.distance_type == SB_DIST_GREATER || r.distance_type == SB_DIST_LESS ||
                    r.distance_type == SB_DIST_EQUAL;
  if (r.distance_type < SB_DIST_NONE || r.distance_type > SB_DIST_EQUAL)
    throw std::invalid_argument("relationship: distance_type (middle is out of scope)");
  if (dist && r.anchor < 0) throw std::invalid_argument("relationship: greater/less/equal require exactly 1 anchor");
  if (r.direction != SB_DIR_NONE && r.anchor < 0) throw std::invalid_argument("relationship: direction requires exactly 1 anchor");
  if (r.direction < SB_DIR_NONE || r.direction > SB_DIR_VECTOR) throw std::invalid_argument("relationship: direction");
  if (r.direction == SB_DIR_VECTOR &&
      std::sqrt(r.direction_vector[0] * r.direction_vector[0] + r.direction_vector[1] * r.direction_vector[1]) < 1e-12)
    throw std::invalid_argument("relationship: zero-length direction vector");
  if (r.distance_type == SB_DIST_LESS && !(0.0 < r.distance))
    throw std::invalid_argument("annulus_sector: min_r >= max_r");
  d.distance_type = r.distance_type;
  d.direction = r.direction;
  d.frame = r.frame;
  d.direction_vector[0] = r.direction_vector[0];
  d.direction_vector[1] = r.direction_vector[1];
  d.distance = r.distance;
  d.angle_threshold = r.angle_threshold;
  if (r.anchor < 0) return false;
  const double theta = r.angle_threshold > 0 ? r.angle_threshold : (r.direction == SB_DIR_NONE ? M_PI : M_PI / 4);
  double min_r = 0.0;  // distance_band (relationships.cpp:101-122)
  if (r.distance_type == SB_DIST_GREATER) min_r = r.distance;
  if (r.distance_type == SB_DIST_EQUAL) min_r = std::max(0.0, r.distance - std::max(0.05 * r.distance, 0.01));
  const bool full = theta >= M_PI - 1e-12;
  if (full && min_r > 0.0) return true;  // annulus with a hole
  // ring size of annulus_sector + up to 8 clip vertices (+1 arc point of rounding slack)
  const double step = 5.0 * M_PI / 180.0;
  const int arc = full ? 73 : static_cast<int>(std::ceil(2.0 * theta / step)) + 2;
  const int ring = arc + (!full && min_r > 0.0 ? arc : 1) + 8;
  return ring > SB_REGION_MAX_VERTS;  // the serial big-ring path
}

}  // namespace

// annulus_sector's arc points (polygon.cpp:136-176) with the host libm, shared by every
// instance when the direction is not in the anchor's local frame (sb_region.h).
bool sbk::arc_table_host(const SbPlacementDev& pl, SbArcTable& t) {
  std::memset(&t, 0, sizeof t);
  if (pl.direction != SB_DIR_NONE && pl.frame == SB_FRAME_LOCAL) return false;
  const double pi = M_PI;
  const double theta = pl.angle_threshold > 0.0 ? pl.angle_threshold
                                                : (pl.direction == SB_DIR_NONE ? pi : pi / 4.0);
  double min_r = 0.0;  // distance_band (relationships.cpp:101-122)
  if (pl.distance_type == SB_DIST_GREATER) min_r = pl.distance;
  if (pl.distance_type == SB_DIST_EQUAL)
    min_r = std::max(0.0, pl.distance - std::max(0.05 * pl.distance, 0.01));
  double vx = 1.0, vy = 0.0;  // resolve_direction (relationships.cpp:78-99), global frame
  switch (pl.direction) {
    case SB_DIR_LEFT: vx = -1; vy = 0; break;
    case SB_DIR_RIGHT: vx = 1; vy = 0; break;
    case SB_DIR_FRONT: vx = 0; vy = -1; break;
    case SB_DIR_BACK: vx = 0; vy = 1; break;
    case SB_DIR_VECTOR: {
      const double nrm = std::sqrt(pl.direction_vector[0] * pl.direction_vector[0] +
                                   pl.direction_vector[1] * pl.direction_vector[1]);
      vx = pl.direction_vector[0] / nrm;
      vy = pl.direction_vector[1] / nrm;
      break;
    }
    default: break;
  }
  const double step = 5.0 * pi / 180.0;
  const bool full = theta >= pi - 1e-12;
  double ends[2][2];
  int narcs = 1;
  if (full) {
    ends[0][0] = 0.0;
    ends[0][1] = 2.0 * pi;
  } else {
    const double base = std::atan2(vy, vx);
    ends[0][0] = base - theta;
    ends[0][1] = base + theta;
    ends[1][0] = base + theta;
    ends[1][1] = base - theta;
    if (min_r > 0.0) narcs = 2;
  }
  for (int k = 0; k < narcs; ++k) {
    const double a0 = ends[k][0], a1 = ends[k][1];
    const int na = std::max(1, static_cast<int>(std::ceil(std::abs(a1 - a0) / step)));
    if (na + 1 > kArcCap) return false;
    t.na[k] = na;
    for (int i = 0; i <= na; ++i) {
      const double a = a0 + (a1 - a0) * static_cast<double>(i) / na;
      t.c[k][i] = std::cos(a);
      t.s[k][i] = std::sin(a);
    }
  }
  return true;
}

// ===================================================================== World
struct sb_world {
  uint64_t n;
  int device;
  cudaStream_t stream = nullptr;
  sb_stats stats{};

  struct Geom {
    sbh::Mesh mesh;  // after drop_degenerate
    uint64_t fingerprint;
    SbGeom g;
  };
  std::vector<Geom> geoms;
  std::vector<SbNode> nodes;
  std::vector<SbTri> tris;
  std::vector<int32_t> obj_geom;
  std::vector<std::string> obj_name;

  DevArray<SbGeom> d_geoms;
  DevArray<SbNode> d_nodes;
  DevArray<SbTri> d_tris;
  DevArray<int32_t> d_grec;      // per geometry: record offset / length (16 B units), nN, nT
  DevArray<uint8_t> d_brec;      // compact narrow-phase records (sb_layout.h)
  DevArray<int32_t> d_obj_geom;
  DevArray<double> d_pose;
  DevArray<double> d_box;
  DevArray<uint32_t> d_enabled;
  int cap_objects = 0;
  int cap_words = 0;

  DevArray<double> d_scratch_poses;
  DevArray<uint32_t> d_scratch_idx;
  DevArray<uint8_t> d_free;
  DevArray<int32_t> d_contact;
  DevArray<unsigned long long> d_counters;

  double margin = 0.0;
  sb_world(uint64_t batch, double margin_, int dev) : n(batch), device(dev), margin(margin_) {
    if (batch == 0) throw std::invalid_argument("CollisionWorld: batch_size must be >= 1");
    if (!std::isfinite(margin)) throw std::invalid_argument("CollisionWorld: margin must be finite");
    if (batch > 0xffffffffull) throw std::invalid_argument("CollisionWorld: batch_size > 2^32-1");
    current_device_checked(dev);
    cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
    d_counters.alloc(8);
  }
  ~sb_world() {
    if (stream) {
      cudaSetDevice(device);
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
  }

  void activate() const { cuda_check(cudaSetDevice(device), "cudaSetDevice"); }
  sb_stream_t s() const { return reinterpret_cast<sb_stream_t>(stream); }

  SbWorldView view() const {
    SbWorldView v;
    v.n = n;
    v.n_objects = static_cast<int32_t>(obj_geom.size());
    v.n_words = (v.n_objects + 31) / 32;
    v.obj_stride = cap_objects;
    v.word_stride = cap_words;
    v.margin = margin;
    v.obj_geom = d_obj_geom.p;
    v.pose = d_pose.p;
    v.box = d_box.p;
    v.enabled = d_enabled.p;
    v.geoms = d_geoms.p;
    v.nodes = d_nodes.p;
    v.tris = d_tris.p;
    v.grec = d_grec.p;
    v.brec = d_brec.p;
    return v;
  }

  const Geom& geom_at(int id) const {
    if (id < 0 || static_cast<size_t>(id) >= geoms.size())
      throw std::out_of_range("unknown geometry id " + std::to_string(id));
    return geoms[id];
  }
  void object_check(int obj) const {
    if (obj < 0 || static_cast<size_t>(obj) >= obj_geom.size())
      throw std::out_of_range("unknown object id " + std::to_string(obj));
  }
  void instance_check(uint64_t inst) const {
    if (inst >= n) throw std::out_of_range("instance index out of range");
  }

  // register_geometry (collision.cpp:339-355)
  int register_geometry(sbh::Mesh mesh) {
    if (mesh.t.empty()) throw std::invalid_argument("register_geometry: empty mesh");
    uint64_t fp = sbh::mesh_fingerprint(mesh);
    for (size_t i = 0; i < geoms.size(); ++i)
      if (geoms[i].fingerprint == fp) return static_cast<int>(i);
    sbh::drop_degenerate(mesh);
    sbh::EffectiveBvh bvh = sbh::build_effective_bvh(mesh);
    if (bvh.nodes.size() > SB_MAX_NODES_PER_GEOM)
      throw std::invalid_argument("register_geometry: effective BVH has " +
                                  std::to_string(bvh.nodes.size()) + " nodes (> " +
                                  std::to_string(SB_MAX_NODES_PER_GEOM) + " supported)");
    if (bvh.tris.size() > SB_MAX_EFF_TRIS)
      throw std::invalid_argument("register_geometry: " + std::to_string(bvh.tris.size()) +
                                  " reachable triangles (> " + std::to_string(SB_MAX_EFF_TRIS) +
                                  " supported by the pooled narrow phase)");
    Geom g;
    g.fingerprint = fp;
    double box[6];
    sbh::mesh_aabb(mesh, box);  // local_box = mesh.aabb() after drop_degenerate
    std::memset(&g.g, 0, sizeof g.g);
    for (int k = 0; k < 3; ++k) {
      g.g.box_min[k] = box[k];
      g.g.box_max[k] = box[3 + k];
      g.g.box_c[k] = (box[k] + box[3 + k]) * 0.5;
      g.g.box_h[k] = (box[3 + k] - box[k]) * 0.5;
    }
    g.g.node_offset = static_cast<int32_t>(nodes.size());
    g.g.n_nodes = static_cast<int32_t>(bvh.nodes.size());
    g.g.tri_offset = static_cast<int32_t>(tris.size());
    g.g.n_tris = static_cast<int32_t>(bvh.tris.size());
    nodes.insert(nodes.end(), bvh.nodes.begin(), bvh.nodes.end());
    tris.insert(tris.end(), bvh.tris.begin(), bvh.tris.end());
    g.mesh = std::move(mesh);
    geoms.push_back(std::move(g));
    activate();
    cuda_check(cudaStreamSynchronize(stream), "sync");
    std::vector<SbGeom> gs;
    for (auto& x : geoms) gs.push_back(x.g);
    d_geoms.alloc(gs.size());
    d_nodes.alloc(nodes.size());
    d_tris.alloc(tris.size());
    cuda_check(cudaMemcpy(d_geoms.p, gs.data(), gs.size() * sizeof(SbGeom), cudaMemcpyHostToDevice), "H2D geoms");
    cuda_check(cudaMemcpy(d_nodes.p, nodes.data(), nodes.size() * sizeof(SbNode), cudaMemcpyHostToDevice), "H2D nodes");
    cuda_check(cudaMemcpy(d_tris.p, tris.data(), tris.size() * sizeof(SbTri), cudaMemcpyHostToDevice), "H2D tris");
    upload_narrow_records();
    ++stats.geometry_registrations;
    ++stats.bvh_builds;
    return static_cast<int>(geoms.size() - 1);
  }

  // Compact B-side narrow-phase records (layout in sb_layout.h), rebuilt per registration.
  void upload_narrow_records() {
    std::vector<int32_t> grec;
    std::vector<uint8_t> brec;
    for (const auto& g : geoms) {
      const int nN = g.g.n_nodes, nT = g.g.n_tris;
      const size_t off = brec.size(), len = static_cast<size_t>(sb_brec_bytes(nN, nT));
      brec.resize(off + len, 0);
      uint8_t* r = brec.data() + off;
      for (int k = 0; k < nN; ++k) {
        const SbNode& nd = nodes[g.g.node_offset + k];
        double box[6] = {nd.c[0], nd.c[1], nd.c[2], nd.h[0], nd.h[1], nd.h[2]};
        std::memcpy(r + 48 * k, box, sizeof box);
        uint32_t info[2];
        info[0] = static_cast<uint32_t>(nd.child0 < 0 ? 0xff : nd.child0) |
                  (static_cast<uint32_t>(nd.child1 < 0 ? 0xff : nd.child1) << 8);
        info[1] = nd.leaves_below;
        std::memcpy(r + 48 * nN + 8 * k, info, sizeof info);
      }
      for (int k = 0; k < nT; ++k) {
        const SbTri& t = tris[g.g.tri_offset + k];
        std::memcpy(r + 56 * nN + 72 * k, t.v, 72);
        r[56 * nN + 72 * nT + k] = static_cast<uint8_t>(t.leaf - 0);
      }
      grec.push_back(static_cast<int32_t>(off / 16));
      grec.push_back(static_cast<int32_t>(len / 16));
      grec.push_back(nN);
      grec.push_back(nT);
    }
    d_grec.alloc(grec.size());
    d_brec.alloc(brec.size());
    cuda_check(cudaMemcpy(d_grec.p, grec.data(), grec.size() * 4, cudaMemcpyHostToDevice), "H2D grec");
    cuda_check(cudaMemcpy(d_brec.p, brec.data(), brec.size(), cudaMemcpyHostToDevice), "H2D brec");
  }

  void grow_objects(int need) {
    if (need <= cap_objects) return;
    int cap = std::max(need, std::max(8, cap_objects * 2));
    int words = (cap + 31) / 32;
    activate();
    cuda_check(cudaStreamSynchronize(stream), "sync");
    DevArray<double> np, nb;
    DevArray<uint32_t> ne;
    np.alloc(static_cast<size_t>(cap) * n * 12);
    nb.alloc(static_cast<size_t>(cap) * n * 6);
    ne.alloc(static_cast<size_t>(words) * n);
    cuda_check(cudaMemset(ne.p, 0, ne.count * sizeof(uint32_t)), "memset enabled");
    if (cap_objects > 0) {  // instance-major records: re-pitch every instance row
      cuda_check(cudaMemcpy2D(np.p, sizeof(double) * 12 * cap, d_pose.p, sizeof(double) * 12 * cap_objects,
                              sizeof(double) * 12 * cap_objects, n, cudaMemcpyDeviceToDevice), "D2D pose");
      cuda_check(cudaMemcpy2D(nb.p, sizeof(double) * 6 * cap, d_box.p, sizeof(double) * 6 * cap_objects,
                              sizeof(double) * 6 * cap_objects, n, cudaMemcpyDeviceToDevice), "D2D box");
      cuda_check(cudaMemcpy2D(ne.p, sizeof(uint32_t) * words, d_enabled.p, sizeof(uint32_t) * cap_words,
                              sizeof(uint32_t) * cap_words, n, cudaMemcpyDeviceToDevice), "D2D enabled");
    }
    std::swap(d_pose.p, np.p);
    std::swap(d_pose.count, np.count);
    std::swap(d_box.p, nb.p);
    std::swap(d_box.count, nb.count);
    std::swap(d_enabled.p, ne.p);
    std::swap(d_enabled.count, ne.count);
    cap_objects = cap;
    cap_words = words;
  }

  // add_object (collision.cpp:365-376)
  int add_object(const std::string& name, int geom) {
    geom_at(geom);
    int id = static_cast<int>(obj_geom.size());
    grow_objects(id + 1);
    obj_geom.push_back(geom);
    obj_name.push_back(name);
    d_obj_geom.alloc(obj_geom.size());
    cuda_check(cudaMemcpy(d_obj_geom.p, obj_geom.data(), obj_geom.size() * 4, cudaMemcpyHostToDevice), "H2D obj_geom");
    sbk::init_object(view(), id, s());
    return id;
  }

  void set_enabled(int obj, const uint32_t* inst, uint64_t m, bool en) {
    object_check(obj);
    for (uint64_t j = 0; j < m; ++j) instance_check(inst[j]);
    if (m == 0) return;
    activate();
    d_scratch_idx.ensure(m);
    cuda_check(cudaMemcpyAsync(d_scratch_idx.p, inst, m * 4, cudaMemcpyHostToDevice, stream), "H2D");
    sbk::set_enabled_list(view(), obj, d_scratch_idx.p, m, en ? 1 : 0, s());
    cuda_check(cudaStreamSynchronize(stream), "sync");
  }
  void set_enabled_all(int obj, bool en) {
    object_check(obj);
    activate();
    sbk::set_enabled_all(view(), obj, en ? 1 : 0, s());
  }
  void upload_poses(const double* poses16, uint64_t m) {
    for (uint64_t j = 0; j < m; ++j) require_homogeneous(poses16 + 16 * j);
    d_scratch_poses.ensure(m * 16);
    cuda_check(cudaMemcpyAsync(d_scratch_poses.p, poses16, m * 16 * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D poses");
  }
  void update_transforms(int obj, const double* poses16) {
    object_check(obj);
    activate();
    upload_poses(poses16, n);
    sbk::update_transforms(view(), obj, d_scratch_poses.p, nullptr, n, 16, s());
    cuda_check(cudaStreamSynchronize(stream), "sync");
  }
  void update_transform(int obj, uint64_t inst, const double* pose16) {
    object_check(obj);
    instance_check(inst);
    activate();
    upload_poses(pose16, 1);
    d_scratch_idx.ensure(1);
    uint32_t i32 = static_cast<uint32_t>(inst);
    cuda_check(cudaMemcpyAsync(d_scratch_idx.p, &i32, 4, cudaMemcpyHostToDevice, stream), "H2D");
    sbk::update_transforms(view(), obj, d_scratch_poses.p, d_scratch_idx.p, 1, 16, s());
    cuda_check(cudaStreamSynchronize(stream), "sync");
  }
  void object_pose(int obj, uint64_t inst, double* out16) {
    object_check(obj);
    instance_check(inst);
    activate();
    double rec[12];
    cuda_check(cudaMemcpyAsync(rec, d_pose.p + sb_pose_off(view(), obj, inst), sizeof rec, cudaMemcpyDeviceToHost, stream), "D2H");
    cuda_check(cudaStreamSynchronize(stream), "sync");
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 4; ++j) out16[4 * j + i] = rec[4 * i + j];
    out16[3] = out16[7] = out16[11] = 0.0;
    out16[15] = 1.0;
  }
  bool enabled(int obj, uint64_t inst) {
    object_check(obj);
    instance_check(inst);
    activate();
    uint32_t w = 0;
    cuda_check(cudaMemcpyAsync(&w, d_enabled.p + sb_word_off(view(), obj >> 5, inst), 4, cudaMemcpyDeviceToHost, stream), "D2H");
    cuda_check(cudaStreamSynchronize(stream), "sync");
    return (w >> (obj & 31)) & 1u;
  }

  // check_batch (collision.cpp:418-461)
  void check_batch(int geom, const double* poses16, const uint32_t* active, uint64_t m,
                   uint8_t* free_out, int32_t* contact_out) {
    geom_at(geom);
    for (uint64_t j = 0; j < m; ++j) instance_check(active[j]);
    activate();
    d_free.ensure(n);
    d_contact.ensure(n);
    cuda_check(cudaMemsetAsync(d_free.p, 1, n, stream), "memset");
    cuda_check(cudaMemsetAsync(d_contact.p, 0xff, n * 4, stream), "memset");
    cuda_check(cudaMemsetAsync(d_counters.p, 0, 8 * sizeof(unsigned long long), stream), "memset");
    if (m > 0) {
      upload_poses(poses16, m);
      d_scratch_idx.ensure(m);
      cuda_check(cudaMemcpyAsync(d_scratch_idx.p, active, m * 4, cudaMemcpyHostToDevice, stream), "H2D");
      sbk::check_batch(view(), geom, d_scratch_poses.p, d_scratch_idx.p, m, d_free.p, d_contact.p,
                       d_counters.p, s());
    }
    unsigned long long c[8];
    cuda_check(cudaMemcpyAsync(free_out, d_free.p, n, cudaMemcpyDeviceToHost, stream), "D2H");
    cuda_check(cudaMemcpyAsync(contact_out, d_contact.p, n * 4, cudaMemcpyDeviceToHost, stream), "D2H");
    cuda_check(cudaMemcpyAsync(c, d_counters.p, sizeof c, cudaMemcpyDeviceToHost, stream), "D2H");
    cuda_check(cudaStreamSynchronize(stream), "sync");
    ++stats.check_calls;
    stats.checked_instances += m;
    stats.narrow_phase_tests += c[1];
    stats.triangle_pair_tests += c[2];
  }
};

// ===================================================================== Engine
struct sb_engine {
  std::unique_ptr<sb_world> world;
  void write_back(uint32_t placement, sb_graph& g, uint32_t node);  // defined after sb_graph
  struct ReachFilter {  // fused reachability filter of one placement (sb_engine_set_reach_filter)
    const unsigned long long* any = nullptr;
    sbk::ReachGrid grid{};
    std::unique_ptr<DevArray<double>> base;
  };
  std::vector<ReachFilter> reach;
  uint64_t n_total = 0, begin = 0, end = 0, n = 0;
  int rank = 0, world_size = 1;
  sb_allgather_fn allgather = nullptr;
  void* allgather_ctx = nullptr;
  sb_allgather_dev_fn allgather_dev = nullptr;  // device-side count exchange (optional)
  void* allgather_dev_ctx = nullptr;
  DevArray<unsigned long long> d_xcount, d_xrecv, d_xdraws;
  PinnedArray<unsigned long long> h_xrecv;
  int attempts = 0;

  struct Placement {
    SbPlacementDev dev;
    double support16[16];
    double inv_support[12];
    int canon_n = 0;  // host-built canonical table size (no anchor)
    bool hole = false;  // full annulus with a hole (theta = pi, min_r > 0)
    bool shared_arcs = false;  // arc table in d_arcs[p] (no local-frame direction)
    double ratio = 0.0;        // ratio_on_support (no-relation placements)
    int mesh = 0;
  };
  std::vector<Placement> places;
  int32_t first_place_obj = 0;
  int inst_cap = 0;  // region table stride (canonical and per instance)

  DevArray<uint8_t> d_valid;
  DevArray<int16_t> d_accepted;
  DevArray<uint32_t> d_tile_list;   // [ntiles * tile_inst] survivors per tile
  DevArray<uint32_t> d_tile_cnt;    // [2][ntiles]
  DevArray<double> d_cpose;         // [grid][kPlaceBlock][12] candidate poses
  DevArray<double> d_cinv;          // [grid][kPlaceBlock][12] their inverses
  DevArray<uint32_t> d_cells;       // broad-phase occupancy grid [n][g * g][words]
  SbCellGrid cell_grid{};
  DevArray<uint32_t> d_ctrl;
  DevArray<uint64_t> d_prof;
  DevArray<unsigned> d_dbg;        // SB_ROUND_DEBUG=1: per-round CTA maxima (fast path)
  bool round_debug = false;
  double last_dbg[3] = {0, 0, 0};
  DevArray<int32_t> d_rflags;
  std::vector<cudaEvent_t> ev_place;
  double last_prof[16] = {};
  bool place_times = false;  // SB_PLACE_TIMES=1: per-placement event times to stderr
  bool timing_pending = false;
  std::vector<char> pending_per_inst;
  std::vector<uint32_t> pending_rounds;
  double pending_sharded_ms = 0.0;
  int num_sms = 0;
  // tile decomposition of the shard (sb_place.h) and launch shape of the placement kernel
  uint32_t ntiles = 0;
  int tile_inst = 0, tile_inst_pi = 0, max_tris = 1, max_nodes = 1, ws_bytes = 0;
  int spec_target = 64;
  int solo_max = 16;
  int solo_spec = 0;  // SB_SOLO_SPEC: speculative slots per solo round (0/1: one round at a time)
  unsigned grid = 0;
  size_t smem = 0;
  DevArray<unsigned long long> d_counters;
  DevArray<double> d_anchor;
  DevArray<double> d_s0;
  DevArray<int32_t> d_flags;  // [0] vary, [1] region status
  DevArray<SbRegionTri> d_canon_tris;
  DevArray<double> d_canon_cum;
  DevArray<int32_t> d_canon_n;
  DevArray<sbk::SbArcTable> d_arcs;  // per placement: shared annulus arc points
  DevArray<SbRegionTri> d_inst_tris;
  DevArray<double> d_inst_cum;
  DevArray<int32_t> d_inst_n;
  DevArray<double> d_pose16;
  DevArray<double> d_out16;
  PinnedArray<uint8_t> h_stat;
  DevArray<unsigned long long> d_nvalid;
  bool host_times = std::getenv("SB_HOST_TIMES") != nullptr;  // end-of-run counters / ctrl words / region flags / timers  // [P][n][16] result poses written at accept (pipelined download)
  PinnedArray<uint64_t> h_count;
  cudaStream_t copy_stream = nullptr;  // pipelined result download
  std::vector<cudaEvent_t> ev_pose;
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr, ev_r0 = nullptr, ev_r1 = nullptr;

  uint64_t last_launches = 0;
  double last_total_ms = 0.0, last_check_ms = 0.0;
  uint64_t last_check_launches = 0;

  std::vector<uint64_t> exchange(const std::vector<uint64_t>& send) {
    if (world_size == 1) return send;
    std::vector<uint64_t> recv(send.size() * world_size);
    if (allgather(allgather_ctx, send.data(), static_cast<uint32_t>(send.size()), recv.data()) != 0)
      throw std::runtime_error("allgather callback failed");
    return recv;
  }

  sb_engine(const sb_scene* sc, const sb_shard* shard, int device) {
    if (!sc) throw std::invalid_argument("scene is NULL");
    n_total = sc->n_instances;
    begin = 0;
    end = n_total;
    if (shard) {
      begin = shard->begin;
      end = shard->end;
      rank = shard->rank;
      world_size = shard->world_size;
      allgather = shard->allgather;
      allgather_ctx = shard->ctx;
      allgather_dev = shard->allgather_dev;
      allgather_dev_ctx = shard->ctx_dev;
      if (world_size < 1 || rank < 0 || rank >= world_size) throw std::invalid_argument("bad shard rank");
      if (world_size > 1 && !allgather) throw std::invalid_argument("sharded engine needs an allgather callback");
    }
    if (begin >= end || end > n_total) throw std::invalid_argument("bad shard range");
    n = end - begin;
    attempts = sc->attempts;
    if (attempts < 1 || attempts > 32767) throw std::invalid_argument("attempts must be in [1, 32767]");
    world = std::make_unique<sb_world>(n, 0.0, device);

    std::vector<int> geom_of_mesh;
    std::vector<double> z_off;
    std::vector<std::array<double, 2>> footprint;  // mesh AABB x / y extents
    for (uint32_t i = 0; i < sc->n_meshes; ++i) {
      const sb_mesh& m = sc->meshes[i];
      if (!m.vertices || !m.triangles) throw std::invalid_argument("mesh arrays are NULL");
      sbh::Mesh h;
      h.v.resize(m.n_vertices);
      h.t.resize(m.n_triangles);
      for (uint32_t k = 0; k < m.n_vertices; ++k)
        h.v[k] = {m.vertices[3 * k], m.vertices[3 * k + 1], m.vertices[3 * k + 2]};
      for (uint32_t k = 0; k < m.n_triangles; ++k)
        h.t[k] = {m.triangles[3 * k], m.triangles[3 * k + 1], m.triangles[3 * k + 2]};
      double box[6];
      sbh::mesh_aabb(h, box);  // rest_pose uses the mesh as given (sampler.cpp:45-52)
      footprint.push_back({box[3] - box[0], box[4] - box[1]});
      if (!(box[2] <= box[5]) || !std::isfinite(box[2]) || !std::isfinite(box[5]))
        throw std::invalid_argument("rest_pose: degenerate bounding box");
      z_off.push_back(-box[2] + 1e-3);
      geom_of_mesh.push_back(world->register_geometry(std::move(h)));
    }
    auto mesh_geom = [&](int32_t m) {
      if (m < 0 || static_cast<uint32_t>(m) >= sc->n_meshes) throw std::out_of_range("mesh index");
      return geom_of_mesh[m];
    };
    for (uint32_t f = 0; f < sc->n_fixed; ++f) {
      int obj = world->add_object("fixed" + std::to_string(f), mesh_geom(sc->fixed[f].mesh));
      require_homogeneous(sc->fixed[f].pose);
      world->upload_poses(sc->fixed[f].pose, 1);
      // broadcast one pose to every instance (stride 0)
      sbk::update_transforms(world->view(), obj, world->d_scratch_poses.p, nullptr, n, 0, world->s());
      cuda_check(cudaStreamSynchronize(world->stream), "sync");
      world->set_enabled_all(obj, true);
    }
    first_place_obj = static_cast<int32_t>(sc->n_fixed);
    bool any_anchor = false, any_hole = false;
    for (uint32_t p = 0; p < sc->n_placements; ++p) {
      const sb_placement& sp = sc->placements[p];
      int obj = world->add_object("p" + std::to_string(p), mesh_geom(sp.mesh));
      if (sp.support < 0 || static_cast<uint32_t>(sp.support) >= sc->n_supports)
        throw std::out_of_range("support index");
      const sb_support& sup = sc->supports[sp.support];
      require_homogeneous(sup.pose);
      Placement pl;
      std::memset(&pl.dev, 0, sizeof pl.dev);
      pl.dev.geom = mesh_geom(sp.mesh);
      pl.dev.object = obj;
      pl.dev.orientation = sp.orientation;
      if (sp.orientation < SB_ORIENT_FIXED || sp.orientation > SB_ORIENT_FACE_TO)
        throw std::invalid_argument("orientation rule");
      pl.dev.face_object = -1;
      if (sp.orientation == SB_ORIENT_FACE_TO) {
        if (sp.face_target < 0 || static_cast<uint32_t>(sp.face_target) >= p)
          throw std::invalid_argument("sample_orientations: face_to target must be an earlier placement");
        pl.dev.face_object = first_place_obj + sp.face_target;
      }
      pl.dev.z_off = z_off[sp.mesh];
      std::memcpy(pl.support16, sup.pose, sizeof pl.support16);
      colmajor_to_34(sup.pose, pl.dev.support);
      inverse_rigid34(sup.pose, pl.inv_support);
      for (int k = 0; k < 4; ++k) pl.dev.rect[k] = sup.rect[k];
      const sb_relation& r = sp.relation;
      pl.hole = relation_to_dev(r, pl.dev);
      if (sp.ratio_on_support != 0.0) {  // apply_ratio_on_support's checks (relationships.cpp:222-227)
        if (sp.ratio_on_support < 0.0 || sp.ratio_on_support > 1.0)
          throw std::invalid_argument("apply_ratio_on_support: ratio outside [0,1]");
        if (!(footprint[sp.mesh][0] > 0.0) || !(footprint[sp.mesh][1] > 0.0))
          throw std::invalid_argument("apply_ratio_on_support: footprint edges must be positive");
        if (pl.hole)
          throw std::invalid_argument("ratio_on_support on an annulus with a hole or a wide annular sector (not convex) is out of scope");
      }
      pl.ratio = sp.ratio_on_support;
      pl.mesh = sp.mesh;
      if (r.anchor >= 0 && sp.ratio_on_support > 0.0)  // relation regions erode on the device
        pl.dev.erode_r = sp.ratio_on_support * std::min(footprint[sp.mesh][0], footprint[sp.mesh][1]) / 2.0;
      if (r.anchor >= 0 && static_cast<uint32_t>(r.anchor) >= p)
        throw std::invalid_argument("relationship: anchor must be an earlier placement");
      pl.dev.anchor_object = r.anchor >= 0 ? first_place_obj + r.anchor : -1;
      pl.dev.salt = p;
      if (r.anchor >= 0) any_anchor = true;
      any_hole = any_hole || pl.hole;
      places.push_back(pl);
    }
    attempts = sc->attempts;

    // canonical sampler tables (no-anchor placements: the support rect itself)
    const size_t P = places.size();
    {  // annulus arc points shared by all instances (host libm, sb_region.h)
      std::vector<sbk::SbArcTable> arcs(std::max<size_t>(1, P));
      for (size_t p = 0; p < P; ++p)
        places[p].shared_arcs = places[p].dev.anchor_object >= 0 && !places[p].hole &&
                                sbk::arc_table_host(places[p].dev, arcs[p]);
      d_arcs.alloc(arcs.size());
      cuda_check(cudaMemcpy(d_arcs.p, arcs.data(), arcs.size() * sizeof(sbk::SbArcTable), cudaMemcpyHostToDevice), "H2D arcs");
    }
    inst_cap = any_hole ? sbp::kHoleCap : SB_REGION_MAX_VERTS;
    d_canon_tris.alloc(std::max<size_t>(1, P) * inst_cap);
    d_canon_cum.alloc(std::max<size_t>(1, P) * inst_cap);
    d_canon_n.alloc(std::max<size_t>(1, P));
    for (size_t p = 0; p < P; ++p) {
      if (places[p].dev.anchor_object >= 0) continue;
      const double* rc = places[p].dev.rect;
      std::vector<sbh::V2> ring = {{rc[0], rc[1]}, {rc[2], rc[1]}, {rc[2], rc[3]}, {rc[0], rc[3]}};
      if (places[p].ratio > 0.0) {  // apply_ratio_on_support (relationships.cpp:220-230)
        const auto& fp = footprint[places[p].mesh];
        const double r = places[p].ratio * std::min(fp[0], fp[1]) / 2.0;
        if (r > 0.0) ring = sbh::erode_convex(ring, r);
      }
      sbh::SamplerTable t = sbh::sampler_table({ring});
      places[p].canon_n = static_cast<int>(t.tris.size());
      if (!t.tris.empty()) {
        cuda_check(cudaMemcpy(d_canon_tris.p + p * inst_cap, t.tris.data(), t.tris.size() * sizeof(SbRegionTri), cudaMemcpyHostToDevice), "H2D canon");
        cuda_check(cudaMemcpy(d_canon_cum.p + p * inst_cap, t.cum.data(), t.cum.size() * sizeof(double), cudaMemcpyHostToDevice), "H2D canon");
      }
    }
    if (any_anchor) {
      d_inst_tris.alloc(n * inst_cap);
      d_inst_cum.alloc(n * inst_cap);
      d_inst_n.alloc(n);
      d_anchor.alloc(3 * n);
    }
    d_s0.alloc(3);
    d_flags.alloc(2);
    d_valid.alloc(n);
    d_accepted.alloc(std::max<size_t>(1, P) * n);
    cuda_check(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, world->device), "attr");
    for (const auto& g : world->geoms) {
      max_tris = std::max(max_tris, static_cast<int>(g.g.n_tris));
      max_nodes = std::max(max_nodes, static_cast<int>(g.g.n_nodes));
    }
    if (max_tris > 16 || max_nodes > 16)
      throw std::invalid_argument("engine: a geometry's effective BVH exceeds 16 nodes / 16 triangles");
    ws_bytes = sbk::place_ws_bytes(max_tris, max_nodes);
    smem = sbk::place_smem_bytes(world->view().n_words, ws_bytes, world->view().n_objects);
    grid = static_cast<unsigned>(sbk::place_grid(num_sms, smem));
    if (grid == 0) throw CudaError("placement kernel does not fit on the device (shared memory)");
    {  // tiles: a multiple of the grid, at most kPlaceBlock instances each
      const uint64_t per_wave = static_cast<uint64_t>(grid) * sbk::kPlaceBlock;
      const uint64_t waves = (n + per_wave - 1) / per_wave;
      const uint64_t want = static_cast<uint64_t>(grid) * waves;
      tile_inst = static_cast<int>((n + want - 1) / want);
      // per-instance placements: smaller tiles, taken dynamically, so a dense tile's heavy
      // narrow phase does not hold the whole placement (SB_PI_SPLIT; measured best: 1)
      int split = 1;
      if (const char* e = std::getenv("SB_PI_SPLIT")) split = std::max(1, std::atoi(e));
      tile_inst_pi = std::max(1, (tile_inst + split - 1) / split);
      ntiles = static_cast<uint32_t>((n + tile_inst - 1) / tile_inst);
      if ((ntiles + grid - 1) / grid > static_cast<uint32_t>(sbk::kPlaceMaxOwnedTiles))
        throw std::invalid_argument("shard too large for one device: " + std::to_string(n) + " instances");
    }
    d_tile_list.alloc(static_cast<size_t>(ntiles) * tile_inst);
    d_tile_cnt.alloc(2 * static_cast<size_t>(ntiles));
    d_cpose.alloc(static_cast<size_t>(grid) * sbk::kPlaceBlock * 12);
    d_cinv.alloc(static_cast<size_t>(grid) * sbk::kPlaceBlock * 12);
    {  // occupancy grid over the supports' XY extent, widened by the largest object radius
      double bx0 = HUGE_VAL, by0 = HUGE_VAL, bx1 = -HUGE_VAL, by1 = -HUGE_VAL, rad = 0.0;
      for (uint32_t k = 0; k < sc->n_supports; ++k) {
        const sb_support& su = sc->supports[k];
        const double xs[2] = {su.rect[0], su.rect[2]}, ys[2] = {su.rect[1], su.rect[3]};
        for (double x : xs)
          for (double y : ys) {
            const double wx = su.pose[0] * x + su.pose[4] * y + su.pose[12];
            const double wy = su.pose[1] * x + su.pose[5] * y + su.pose[13];
            bx0 = std::min(bx0, wx);
            bx1 = std::max(bx1, wx);
            by0 = std::min(by0, wy);
            by1 = std::max(by1, wy);
          }
      }
      for (const Placement& pl : places) {  // candidates only: fixed objects just clamp
        const SbGeom& g = world->geom_at(pl.dev.geom).g;
        const double ex = std::max(std::fabs(g.box_min[0]), std::fabs(g.box_max[0]));
        const double ey = std::max(std::fabs(g.box_min[1]), std::fabs(g.box_max[1]));
        rad = std::max(rad, std::sqrt(ex * ex + ey * ey));
      }
      const int words = world->view().n_words;
      if (words > 8) throw std::invalid_argument("engine: more than 256 objects per scene");
      // Few objects: the broad phase reads every enabled object's box (one round trip);
      // many: the grid narrows the candidates first (SB_CELL_GRID=0/1 forces either).
      int g = world->view().n_objects > 32 ? 16 : 0;
      if (const char* e = std::getenv("SB_CELL_GRID")) g = std::atoi(e) ? 16 : 0;
      while (g > 1 && static_cast<double>(n) * g * g * words * 4.0 > 8.0e9) g /= 2;
      if (g == 1) g = 0;
      if (!(bx0 <= bx1) || !(by0 <= by1)) {
        bx0 = by0 = -1.0;
        bx1 = by1 = 1.0;
      }
      bx0 -= rad;
      by0 -= rad;
      bx1 += rad;
      by1 += rad;
      cell_grid.x0 = bx0;
      cell_grid.y0 = by0;
      cell_grid.inv_x = g / std::max(bx1 - bx0, 1e-9);
      cell_grid.inv_y = g / std::max(by1 - by0, 1e-9);
      cell_grid.g = g;
      cell_grid.words = words;
      if (g) d_cells.alloc(static_cast<size_t>(n) * g * g * words);
      cell_grid.cells = d_cells.p;
    }
    d_ctrl.alloc(8 * std::max<size_t>(1, places.size()));
    d_rflags.alloc(2 * std::max<size_t>(1, places.size()));
    d_prof.alloc(8);
    round_debug = std::getenv("SB_ROUND_DEBUG") != nullptr;
    place_times = std::getenv("SB_PLACE_TIMES") != nullptr;
    if (const char* st = std::getenv("SB_SPEC_TARGET")) spec_target = std::max(1, std::atoi(st));
    if (const char* so = std::getenv("SB_SOLO")) solo_max = std::max(0, std::min(sbk::kPlaceBlock, std::atoi(so)));
    if (const char* ss = std::getenv("SB_SOLO_SPEC")) solo_spec = std::max(0, std::min(sbk::kPlaceBlock, std::atoi(ss)));
    if (round_debug) d_dbg.alloc(3 * static_cast<size_t>(attempts) * std::max<size_t>(1, places.size()) + 16);
    d_counters.alloc(8);
    cuda_check(cudaEventCreate(&ev_start), "event");
    cuda_check(cudaEventCreate(&ev_stop), "event");
    cuda_check(cudaEventCreate(&ev_r0), "event");
    cuda_check(cudaEventCreate(&ev_r1), "event");
    cuda_check(cudaDeviceSynchronize(), "sync");
  }

  ~sb_engine() {
    if (world) cudaSetDevice(world->device);
    for (cudaEvent_t e : {ev_start, ev_stop, ev_r0, ev_r1})
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_place) cudaEventDestroy(e);
    for (cudaEvent_t e : ev_pose) cudaEventDestroy(e);
    if (copy_stream) {
      cudaStreamSynchronize(copy_stream);
      cudaStreamDestroy(copy_stream);
    }
  }


  // One placement's relation region (single GPU: decided on the device, no host sync).
  void relation_prep_device(size_t p, Placement& pl, const SbWorldView& wv, uint64_t& launches) {
    sbk::RelationRegionParams rp;
    std::memset(&rp, 0, sizeof rp);
    rp.w = wv;
    rp.pl = pl.dev;
    rp.anchor_object = pl.dev.anchor_object;
    rp.owns_instance0 = 1;
    std::memcpy(rp.inv_support, pl.inv_support, sizeof rp.inv_support);
    rp.cap = inst_cap;
    rp.hole = pl.hole ? 1 : 0;
    rp.arcs = pl.shared_arcs ? d_arcs.p + p : nullptr;
    rp.tris = d_inst_tris.p;
    rp.cum = d_inst_cum.p;
    rp.ntri = d_inst_n.p;
    rp.flags = d_rflags.p + 2 * p;
    sbk::relation_regions(rp, num_sms, world->s());
    ++launches;
  }

  // Sharded runs: instance 0's anchor state and the variation flag are exchanged.
  // Returns true if the anchors vary (per-instance path); else fills the canonical slot.
  bool relation_prep_sharded(size_t p, Placement& pl, const SbWorldView& wv, uint64_t& launches,
                             int& canon_n) {
    cudaStream_t stream = world->stream;
    sb_stream_t s = world->s();
    double s0[3] = {0, 0, 0};
    if (begin == 0) {
      sbk::anchor_states(wv, pl.dev.anchor_object, pl.inv_support, d_anchor.p, s);
      ++launches;
      cuda_check(cudaMemcpyAsync(s0, d_anchor.p, sizeof s0, cudaMemcpyDeviceToHost, stream), "D2H s0");
      cuda_check(cudaStreamSynchronize(stream), "sync");
    }
    std::vector<uint64_t> send(4, 0);
    std::memcpy(send.data(), s0, sizeof s0);
    send[3] = begin == 0 ? 1 : 0;
    std::vector<uint64_t> recv = exchange(send);
    for (int r = 0; r < world_size; ++r)
      if (recv[4 * r + 3]) std::memcpy(s0, &recv[4 * r], sizeof s0);
    cuda_check(cudaMemcpyAsync(d_s0.p, s0, sizeof s0, cudaMemcpyHostToDevice, stream), "H2D s0");
    sbk::RelationRegionParams rp;
    std::memset(&rp, 0, sizeof rp);
    rp.w = wv;
    rp.pl = pl.dev;
    rp.anchor_object = pl.dev.anchor_object;
    rp.owns_instance0 = 0;
    std::memcpy(rp.inv_support, pl.inv_support, sizeof rp.inv_support);
    rp.s0 = d_s0.p;
    rp.cap = inst_cap;
    rp.hole = pl.hole ? 1 : 0;
    rp.arcs = pl.shared_arcs ? d_arcs.p + p : nullptr;
    rp.tris = d_inst_tris.p;
    rp.cum = d_inst_cum.p;
    rp.ntri = d_inst_n.p;
    rp.flags = d_rflags.p + 2 * p;
    sbk::relation_regions(rp, num_sms, s);
    ++launches;
    int32_t flags[2];
    cuda_check(cudaMemcpyAsync(flags, rp.flags, sizeof flags, cudaMemcpyDeviceToHost, stream), "D2H flags");
    cuda_check(cudaStreamSynchronize(stream), "sync");
    bool vary = flags[0] != 0;
    std::vector<uint64_t> f = exchange({vary ? 1ull : 0ull});
    vary = false;
    for (uint64_t x : f) vary = vary || x != 0;
    if (!vary) {
      rp.from_s0 = 1;
      rp.tris = d_canon_tris.p + p * inst_cap;
      rp.cum = d_canon_cum.p + p * inst_cap;
      rp.ntri = d_canon_n.p + p;
      sbk::relation_regions(rp, num_sms, s);
      ++launches;
      cuda_check(cudaMemcpyAsync(&canon_n, d_canon_n.p + p, 4, cudaMemcpyDeviceToHost, stream), "D2H n");
      cuda_check(cudaStreamSynchronize(stream), "sync");
    }
    return vary;
  }

  // Results requested with the call (sb_engine_generate with an sb_result) are downloaded
  // while later placements compute: placement p's poses are final once its kernel ends, so
  // a copy stream converts them (k_pose_colmajor) and copies them to the host behind an event.
  void generate(uint64_t run_seed, sb_run_stats* st, sb_result* out = nullptr) {
    const auto th0 = std::chrono::steady_clock::now();
    world->activate();
    const bool pipe = out && out->poses && !places.empty();
    if (pipe) {
      if (!copy_stream)
        cuda_check(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
      while (ev_pose.size() < places.size()) {
        cudaEvent_t e;
        cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
        ev_pose.push_back(e);
      }
      d_out16.ensure(16 * n * places.size());
    }
    cudaStream_t stream = world->stream;
    sb_stream_t s = world->s();
    const SbWorldView wv = world->view();
    const size_t P = places.size();
    uint64_t launches = 0, rounds_host = 0, per_inst_host = 0, round_launches = 0;
    double sharded_check_ms = 0.0;
    std::vector<char> device_rounds(places.size(), world_size == 1 ? 1 : 0);
    while (ev_place.size() < 2 * P + 2) {
      cudaEvent_t e;
      cuda_check(cudaEventCreate(&e), "event");
      ev_place.push_back(e);
    }
    cuda_check(cudaEventRecord(ev_start, stream), "event");
    cuda_check(cudaMemsetAsync(d_counters.p, 0, 8 * sizeof(unsigned long long), stream), "memset");
    cuda_check(cudaMemsetAsync(d_prof.p, 0, 8 * sizeof(uint64_t), stream), "memset");
    if (round_debug) cuda_check(cudaMemsetAsync(d_dbg.p, 0, d_dbg.count * sizeof(unsigned), stream), "memset");
    cuda_check(cudaMemsetAsync(d_ctrl.p, 0, d_ctrl.count * sizeof(uint32_t), stream), "memset");
    cuda_check(cudaMemsetAsync(d_rflags.p, 0, d_rflags.count * sizeof(int32_t), stream), "memset");
    sbk::engine_reset(wv, first_place_obj, static_cast<int32_t>(P), d_valid.p, d_accepted.p,
                      static_cast<int32_t>(P), pipe ? d_out16.p : nullptr, s);
    launches += 1;
    if (cell_grid.g) {
      sbk::cells_reset(wv, cell_grid, first_place_obj, s);
      ++launches;
    }
    for (size_t p = 0; p < P; ++p) {
      Placement& pl = places[p];
      bool fast = true;
      int canon_n = pl.canon_n;
      const SbRegionTri* canon_tris = d_canon_tris.p + p * inst_cap;
      const double* canon_cum = d_canon_cum.p + p * inst_cap;
      const bool relation = pl.dev.anchor_object >= 0;
      cuda_check(cudaEventRecord(ev_place[2 * p], stream), "event");
      if (relation) {
        if (world_size == 1) {
          relation_prep_device(p, pl, wv, launches);
        } else {
          fast = !relation_prep_sharded(p, pl, wv, launches, canon_n);
          if (!fast) ++per_inst_host;
        }
      }
      cuda_check(cudaEventRecord(ev_place[2 * p + 1], stream), "event");
      uint64_t fast_state0 = 0;
      {  // Pcg32(make_stream(run_seed, {salt, "cach"})) state after the constructor
        uint64_t h = sbh::mix64(sbh::mix64(sbh::mix64(run_seed) ^ pl.dev.salt) ^ 0x63616368ULL);
        const uint64_t mult = 6364136223846793005ULL, inc = (0xda3e39cb94b95bdbULL << 1u) | 1u;
        uint64_t st0 = inc;
        st0 += h;
        st0 = st0 * mult + inc;
        fast_state0 = st0;
      }
      sbk::PlaceParams pp;
      std::memset(&pp, 0, sizeof pp);
      pp.w = wv;
      pp.pl = pl.dev;
      pp.attempts = attempts;
      pp.fast = fast ? 1 : 0;
      pp.run_seed = run_seed;
      pp.global_begin = begin;
      pp.fast_state0 = fast_state0;
      pp.canon_tris = canon_tris;
      pp.canon_cum = canon_cum;
      pp.canon_n = canon_n;
      pp.inst_cap = inst_cap;
      pp.inst_tris = d_inst_tris.p;
      pp.inst_cum = d_inst_cum.p;
      pp.inst_n = d_inst_n.p;
      pp.valid = d_valid.p;
      pp.accepted = d_accepted.p + p * n;
      pp.out16 = pipe ? d_out16.p + p * 16 * n : nullptr;
      pp.tile_list = d_tile_list.p;
      pp.tile_cnt = d_tile_cnt.p;
      pp.cpose = d_cpose.p;
      pp.cinv = d_cinv.p;
      pp.grid = cell_grid;
      pp.cnt_stride = ntiles;
      pp.ntiles = ntiles;
      pp.tile_inst = tile_inst;
      pp.tile_inst_pi = tile_inst_pi;
      pp.ntiles_pi = static_cast<uint32_t>((n + tile_inst_pi - 1) / tile_inst_pi);
      pp.spec_target = spec_target;
      pp.solo_max = world_size == 1 ? solo_max : 0;
      pp.solo_spec = solo_spec;
      pp.ws_bytes = ws_bytes;
      pp.max_tris = max_tris;
      pp.max_nodes = max_nodes;
      pp.ctrl = d_ctrl.p + 8 * p;
      pp.counters = d_counters.p;
      pp.prof = d_prof.p;
      pp.dbg = round_debug ? d_dbg.p + 3 * static_cast<size_t>(attempts) * p : nullptr;
      pp.dbg_inst = round_debug ? d_dbg.p + d_dbg.count - 16 : nullptr;
      pp.vary_flag = (relation && world_size == 1) ? d_rflags.p + 2 * p : nullptr;
      if (p < reach.size() && reach[p].any) {
        pp.reach_any = reach[p].any;
        pp.reach_grid = reach[p].grid;
        pp.reach_base = reach[p].base->p;
      }
      if (world_size == 1) {
        if (!sbk::place_persistent(pp, grid, smem, s))
          throw CudaError("cooperative launch of the placement kernel is not possible");
        ++launches;
        ++round_launches;
      } else if (!fast) {
        // per-instance regions: tiles are independent, no exchange
        device_rounds[p] = 1;
        cuda_check(cudaEventRecord(ev_r0, stream), "event");
        sbk::place_instances(pp, grid, smem, s);
        cuda_check(cudaEventRecord(ev_r1, stream), "event");
        ++launches;
        ++round_launches;
        cuda_check(cudaEventSynchronize(ev_r1), "sync");
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, ev_r0, ev_r1), "elapsed");
        sharded_check_ms += ms;
      } else if (allgather_dev) {
        // FIFO fast path, device-side exchange: round a's kernel reads the gathered counts
        // and the draws before it from device memory, the all-gather of its survivors is
        // enqueued behind it; the host only checks for completion every kChunk rounds.
        constexpr int kChunk = 4;
        const size_t K1 = static_cast<size_t>(attempts) + 1, W = static_cast<size_t>(world_size);
        d_xcount.ensure(K1);
        d_xrecv.ensure(K1 * W);
        d_xdraws.ensure(K1);
        h_xrecv.ensure(K1 * W);
        cuda_check(cudaMemsetAsync(d_xcount.p, 0, K1 * 8, stream), "memset");
        cuda_check(cudaMemsetAsync(d_xdraws.p, 0, K1 * 8, stream), "memset");
        pp.xcount = d_xcount.p;
        pp.xrecv = d_xrecv.p;
        pp.xdraws = d_xdraws.p;
        pp.xrank = rank;
        pp.xworld = world_size;
        auto gather = [&](int32_t a) {
          if (allgather_dev(allgather_dev_ctx, reinterpret_cast<const uint64_t*>(d_xcount.p + a), 1,
                            reinterpret_cast<uint64_t*>(d_xrecv.p + a * W), stream) != 0)
            throw std::runtime_error("sb_shard.allgather_dev failed");
        };
        cuda_check(cudaEventRecord(ev_r0, stream), "event");
        sbk::place_fast_init(pp, grid, smem, s);
        ++launches;
        gather(0);
        int32_t a = 0;
        uint64_t last_total = 1;
        while (a < attempts && last_total > 0) {
          const int32_t stop = std::min<int32_t>(attempts, a + kChunk);
          for (; a < stop; ++a) {
            sbk::place_fast_round(pp, a, grid, smem, s);
            launches += 1;
            round_launches += 1;
            gather(a + 1);
          }
          cuda_check(cudaMemcpyAsync(h_xrecv.p + a * W, d_xrecv.p + a * W, W * 8, cudaMemcpyDeviceToHost, stream), "D2H counts");
          cuda_check(cudaStreamSynchronize(stream), "sync");
          last_total = 0;
          for (size_t r = 0; r < W; ++r) last_total += h_xrecv.p[a * W + r];
        }
        cuda_check(cudaEventRecord(ev_r1, stream), "event");
        cuda_check(cudaMemcpyAsync(h_xrecv.p, d_xrecv.p, K1 * W * 8, cudaMemcpyDeviceToHost, stream), "D2H counts");
        cuda_check(cudaStreamSynchronize(stream), "sync");
        for (int32_t r = 0; r < a; ++r) {  // rounds the reference runs: total > 0
          uint64_t t = 0;
          for (size_t k = 0; k < W; ++k) t += h_xrecv.p[r * W + k];
          if (t > 0) ++rounds_host;
        }
        if (a == attempts && last_total > 0) {
          pp.xrecv = nullptr;  // mark the K-attempt survivors invalid
          sbk::place_fast_finish(pp, a, grid, s);
          ++launches;
        }
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, ev_r0, ev_r1), "elapsed");
        sharded_check_ms += ms;
      } else {
        // FIFO fast path: one launch per round, per-rank survivor counts exchanged between
        uint32_t* tot = pp.ctrl;
        auto read_total = [&](int32_t a) {
          uint32_t v = 0;
          cuda_check(cudaMemcpyAsync(&v, tot + sbk::place_total_word(a), 4, cudaMemcpyDeviceToHost, stream), "D2H total");
          cuda_check(cudaStreamSynchronize(stream), "sync");
          return static_cast<uint64_t>(v);
        };
        sbk::place_fast_init(pp, grid, smem, s);
        ++launches;
        uint64_t m = read_total(0), draws = 0;
        int32_t a = 0;
        for (; a < attempts; ++a) {
          std::vector<uint64_t> counts = exchange({m});
          uint64_t total = 0, before = 0;
          for (int r = 0; r < world_size; ++r) {
            if (r < rank) before += counts[r];
            total += counts[r];
          }
          if (total == 0) break;
          ++rounds_host;
          cuda_check(cudaMemsetAsync(tot + sbk::place_total_word(a + 1), 0, 4, stream), "memset");
          if (m > 0) {
            pp.draw_base = draws + before;
            cuda_check(cudaEventRecord(ev_r0, stream), "event");
            sbk::place_fast_round(pp, a, grid, smem, s);
            cuda_check(cudaEventRecord(ev_r1, stream), "event");
            launches += 1;
            round_launches += 1;
            m = read_total(a + 1);
            float ms = 0.f;
            cuda_check(cudaEventElapsedTime(&ms, ev_r0, ev_r1), "elapsed");
            sharded_check_ms += ms;
          } else {
            m = 0;
          }
          if (canon_n > 0) draws += total;
        }
        if (a == attempts && m > 0) {
          sbk::place_fast_finish(pp, a, grid, s);
          ++launches;
        }
      }
      if (pipe) {  // placement p is final: convert + copy its poses behind an event
        // (k_place wrote them at accept: a DMA only, no SM work beside the next placement)
        cuda_check(cudaEventRecord(ev_pose[p], stream), "event");
        cuda_check(cudaStreamWaitEvent(copy_stream, ev_pose[p], 0), "wait");
        cuda_check(cudaMemcpyAsync(out->poses + 16 * n * p, d_out16.p + 16 * n * p,
                                   16 * n * sizeof(double), cudaMemcpyDeviceToHost, copy_stream),
                   "D2H poses");
      }
    }
    if (out) {
      if (out->accepted && P)
        cuda_check(cudaMemcpyAsync(out->accepted, d_accepted.p, P * n * sizeof(int16_t), cudaMemcpyDeviceToHost, stream), "D2H accepted");
      if (out->valid)
        cuda_check(cudaMemcpyAsync(out->valid, d_valid.p, n, cudaMemcpyDeviceToHost, stream), "D2H valid");
    }
    cuda_check(cudaEventRecord(ev_place[2 * P], stream), "event");
    cuda_check(cudaEventRecord(ev_stop, stream), "event");
    // run statistics: small async copies into one pinned block, one synchronisation
    const size_t P1 = std::max<size_t>(1, P);
    h_stat.ensure(136 + 40 * P1);
    unsigned long long* c = reinterpret_cast<unsigned long long*>(h_stat.p);
    uint64_t* prof = reinterpret_cast<uint64_t*>(h_stat.p + 64);
    uint32_t* ctrl_all = reinterpret_cast<uint32_t*>(h_stat.p + 128);
    int32_t* rflags = reinterpret_cast<int32_t*>(h_stat.p + 128 + 32 * P1);
    cuda_check(cudaMemcpyAsync(c, d_counters.p, 64, cudaMemcpyDeviceToHost, stream), "D2H counters");
    cuda_check(cudaMemcpyAsync(prof, d_prof.p, 64, cudaMemcpyDeviceToHost, stream), "D2H prof");
    cuda_check(cudaMemcpyAsync(ctrl_all, d_ctrl.p, 32 * P1, cudaMemcpyDeviceToHost, stream), "D2H ctrl");
    cuda_check(cudaMemcpyAsync(rflags, d_rflags.p, 8 * P1, cudaMemcpyDeviceToHost, stream), "D2H flags");
    unsigned long long* nvalid = reinterpret_cast<unsigned long long*>(h_stat.p + 128 + 40 * P1);
    if (st) {  // valid instances counted on the device (no N-byte readback)
      d_nvalid.ensure(1);
      cuda_check(cudaMemsetAsync(d_nvalid.p, 0, 8, stream), "memset");
      sbk::graph_count_valid(d_valid.p, n, d_nvalid.p, s);
      cuda_check(cudaMemcpyAsync(nvalid, d_nvalid.p, 8, cudaMemcpyDeviceToHost, stream), "D2H nvalid");
    }
    const auto th1 = std::chrono::steady_clock::now();
    cuda_check(cudaStreamSynchronize(stream), "sync");
    const auto th2 = std::chrono::steady_clock::now();
    for (size_t p = 0; p < P; ++p) {
      if (rflags[2 * p + 1] != 0)
        throw std::runtime_error("constraint region build failed for placement " + std::to_string(p) +
                                 " (status " + std::to_string(rflags[2 * p + 1]) +
                                 ": capacity overflow or unsupported annulus)");
    }
    // CUDA-event timings are resolved lazily (resolve_timing: ~2.5 us per
    // cudaEventElapsedTime, 2 per placement) -- only phase_profile / last_timing need them.
    pending_per_inst.assign(P, 0);
    for (size_t p = 0; p < P; ++p)
      pending_per_inst[p] = places[p].dev.anchor_object >= 0 && rflags[2 * p] != 0;
    pending_rounds.assign(P, 0);
    for (size_t p = 0; p < P; ++p) pending_rounds[p] = device_rounds[p] ? ctrl_all[8 * p + 2] : 0u;
    pending_sharded_ms = sharded_check_ms;
    timing_pending = true;
    const auto th2a = std::chrono::steady_clock::now();
    uint64_t rounds = rounds_host;
    for (size_t p = 0; p < P; ++p)
      if (device_rounds[p]) rounds += ctrl_all[8 * p + 2];
    last_check_launches = round_launches;
    last_launches = launches;
    for (int k = 0; k < 7; ++k) last_prof[k] = prof[k] * 1e-6;
    last_prof[7] = static_cast<double>(prof[7]);
    if (round_debug) {
      std::vector<unsigned> dbg(d_dbg.count);
      cuda_check(cudaMemcpy(dbg.data(), d_dbg.p, dbg.size() * sizeof(unsigned), cudaMemcpyDeviceToHost), "D2H dbg");
      for (int k = 0; k < 3; ++k) last_prof[12 + k] = 0;
      for (size_t i = 0; i + 16 < dbg.size(); ++i) last_prof[12 + i % 3] += dbg[i] * 1e-6;
      const unsigned* di = dbg.data() + dbg.size() - 16;
      std::fprintf(stderr, "[round debug] per-instance tiles: %u, max %.1f us, mean %.1f us, max rounds %u, mean rounds %.2f; "
                   "per tile-round: A1 %.1f us, A2+B %.1f us, C %.1f us, max A2+B %.1f us, slots %.1f, "
                   "pairs queued %.1f (max %u) tested %.1f (max %u)\n",
                   di[4], di[0] * 1e-3, di[4] ? double(di[1]) / di[4] : 0.0, di[2], di[4] ? double(di[3]) / di[4] : 0.0,
                   di[3] ? double(di[5]) / di[3] : 0.0, di[3] ? double(di[6]) / di[3] : 0.0,
                   di[3] ? double(di[7]) / di[3] : 0.0, di[8] * 1e-3, di[3] ? double(di[9]) / di[3] : 0.0,
                   di[3] ? double(di[10]) / di[3] : 0.0, di[12], di[3] ? double(di[11]) / di[3] : 0.0, di[13]);
      std::fprintf(stderr, "[round debug] fast path: sum over rounds of max CTA work %.3f ms (A1 %.3f, A2+B %.3f); "
                   "mean CTA work %.3f ms, mean A2+B %.3f ms (grid %u)\n", last_prof[12], last_prof[13], last_prof[14],
                   di[14] * 1e-3 / grid, di[15] * 1e-3 / grid, grid);
    }
    if (place_times) resolve_timing();
    const auto th2b = std::chrono::steady_clock::now();
    world->stats.check_calls += round_launches;
    world->stats.checked_instances += c[0];
    world->stats.narrow_phase_tests += c[1];
    world->stats.triangle_pair_tests += c[2];
    if (st) {
      std::memset(st, 0, sizeof *st);
      st->candidate_checks = c[0];
      st->narrow_phase_tests = c[1];
      st->triangle_pair_tests = c[2];
      st->candidates_sampled = c[3];
      st->rounds = rounds;
      st->per_instance_placements = c[7] + per_inst_host;
      st->broad_phase_tests = c[4];
      st->node_pair_tests = c[5];
      st->accepted_candidates = c[6];
      st->valid_instances = *nvalid;
    }
    if (pipe) cuda_check(cudaStreamSynchronize(copy_stream), "sync copy stream");
    if (host_times) {
      const auto th3 = std::chrono::steady_clock::now();
      auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
      resolve_timing();
      std::fprintf(stderr, "[host] enqueue %.1f us, wait %.1f us, after %.1f us (%.1f / %.1f / %.1f) (device %.1f us) t0 %.1f t3 %.1f\n",
                   us(th0, th1), us(th1, th2), us(th2, th3), us(th2, th2a), us(th2a, th2b), us(th2b, th3),
                   last_total_ms * 1e3,
                   std::chrono::duration<double, std::micro>(th0.time_since_epoch()).count(),
                   std::chrono::duration<double, std::micro>(th3.time_since_epoch()).count());
    }
  }

  void resolve_timing() {
    if (!timing_pending) return;
    timing_pending = false;
    const size_t P = pending_per_inst.size();
    float total_ms = 0.f;
    cuda_check(cudaEventElapsedTime(&total_ms, ev_start, ev_stop), "elapsed");
    double regions_ms = 0.0, place_ms = 0.0, inst_ms = 0.0, fast_ms = 0.0;
    for (size_t p = 0; p < P; ++p) {
      float a = 0.f, b = 0.f;
      cuda_check(cudaEventElapsedTime(&a, ev_place[2 * p], ev_place[2 * p + 1]), "elapsed");
      cuda_check(cudaEventElapsedTime(&b, ev_place[2 * p + 1], ev_place[2 * p + 2]), "elapsed");
      regions_ms += a;
      place_ms += b;
      (pending_per_inst[p] ? inst_ms : fast_ms) += b;
      if (place_times)
        std::fprintf(stderr, "[place %2zu] %s regions %.1f us, placement %.1f us, rounds %u\n", p,
                     pending_per_inst[p] ? "per-instance" : "fifo        ", a * 1e3, b * 1e3,
                     pending_rounds[p]);
    }
    last_prof[8] = regions_ms;
    last_prof[9] = total_ms;
    last_prof[10] = inst_ms;
    last_prof[11] = fast_ms;
    last_total_ms = total_ms;
    last_check_ms = world_size == 1 ? place_ms : pending_sharded_ms;
  }

  void download(sb_result* out) {
    if (!out) return;
    world->activate();
    cudaStream_t stream = world->stream;
    const size_t P = places.size();
    if (out->accepted && P)
      cuda_check(cudaMemcpyAsync(out->accepted, d_accepted.p, P * n * sizeof(int16_t), cudaMemcpyDeviceToHost, stream), "D2H accepted");
    if (out->valid)
      cuda_check(cudaMemcpyAsync(out->valid, d_valid.p, n, cudaMemcpyDeviceToHost, stream), "D2H valid");
    if (out->poses && P) {
      d_pose16.ensure(16 * n);
      for (size_t p = 0; p < P; ++p) {
        sbk::download_poses(world->view(), places[p].dev.object, d_pose16.p, world->s());
        cuda_check(cudaMemcpyAsync(out->poses + 16 * n * p, d_pose16.p, 16 * n * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H poses");
      }
    }
    cuda_check(cudaStreamSynchronize(stream), "sync");
  }
};

// ===================================================================== C ABI
namespace {
template <class F>
sb_status guard(F&& f) {
  try {
    f();
    return SB_OK;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return SB_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_error = e.what();
    return SB_ERR_OUT_OF_RANGE;
  } catch (const std::logic_error& e) {
    g_error = e.what();
    return SB_ERR_LOGIC;
  } catch (const CudaError& e) {
    g_error = e.what();
    return SB_ERR_CUDA;
  } catch (const std::exception& e) {
    g_error = e.what();
    std::string w = e.what();
    return w.rfind("CUDA", 0) == 0 ? SB_ERR_CUDA : SB_ERR_RUNTIME;
  }
}

sb_status mesh_out(const sbh::Mesh& m, double* v, uint32_t* nv, uint32_t* t, uint32_t* nt) {
  if (nv) *nv = static_cast<uint32_t>(m.v.size());
  if (nt) *nt = static_cast<uint32_t>(m.t.size());
  if (v)
    for (size_t i = 0; i < m.v.size(); ++i)
      for (int c = 0; c < 3; ++c) v[3 * i + c] = m.v[i][c];
  if (t)
    for (size_t i = 0; i < m.t.size(); ++i)
      for (int c = 0; c < 3; ++c) t[3 * i + c] = m.t[i][c];
  return SB_OK;
}

sbh::Mesh mesh_in(const double* v, uint32_t nv, const uint32_t* t, uint32_t nt) {
  if ((nv && !v) || (nt && !t)) throw std::invalid_argument("mesh arrays are NULL");
  sbh::Mesh m;
  m.v.resize(nv);
  m.t.resize(nt);
  for (uint32_t i = 0; i < nv; ++i) m.v[i] = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
  for (uint32_t i = 0; i < nt; ++i) m.t[i] = {t[3 * i], t[3 * i + 1], t[3 * i + 2]};
  return m;
}
}  // namespace

extern "C" {

const char* sb_last_error(void) { return g_error.c_str(); }
int sb_abi_version(void) { return SB_ABI_VERSION; }
int sb_device_available(void) {
  return guard([] { current_device_checked(0); }) == SB_OK ? 1 : 0;
}

sb_status sb_make_box(double sx, double sy, double sz, double* v, uint32_t* nv, uint32_t* t,
                      uint32_t* nt) {
  return guard([&] { mesh_out(sbh::make_box(sx, sy, sz), v, nv, t, nt); });
}
sb_status sb_make_cylinder(double r, double h, int seg, double* v, uint32_t* nv, uint32_t* t,
                           uint32_t* nt) {
  return guard([&] { mesh_out(sbh::make_cylinder(r, h, seg), v, nv, t, nt); });
}
sb_status sb_make_sphere(double r, int st, int sl, double* v, uint32_t* nv, uint32_t* t,
                         uint32_t* nt) {
  return guard([&] { mesh_out(sbh::make_sphere(r, st, sl), v, nv, t, nt); });
}
sb_status sb_transform_vertices(const double pose[16], double* v, uint32_t nv) {
  return guard([&] {
    if (!pose || (nv && !v)) throw std::invalid_argument("NULL argument");
    for (uint32_t i = 0; i < nv; ++i) {
      double p[3] = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
      for (int r = 0; r < 3; ++r)  // transform_point: ((R p) + t), left to right
        v[3 * i + r] = ((pose[r] * p[0] + pose[4 + r] * p[1]) + pose[8 + r] * p[2]) + pose[12 + r];
    }
  });
}
sb_status sb_mesh_fingerprint(const double* v, uint32_t nv, const uint32_t* t, uint32_t nt,
                              uint64_t* out) {
  return guard([&] { *out = sbh::mesh_fingerprint(mesh_in(v, nv, t, nt)); });
}
sb_status sb_rest_z_offset(const double* v, uint32_t nv, double* z) {
  return guard([&] {
    sbh::Mesh m = mesh_in(v, nv, nullptr, 0);
    double box[6];
    sbh::mesh_aabb(m, box);
    if (!(box[2] <= box[5]) || !std::isfinite(box[2])) throw std::invalid_argument("rest_pose: degenerate bounding box");
    *z = -box[2] + 1e-3;
  });
}

sb_status sb_bvh_info(const double* v, uint32_t nv, const uint32_t* t, uint32_t nt,
                      int32_t info[4]) {
  return guard([&] {
    sbh::Mesh m = mesh_in(v, nv, t, nt);
    sbh::drop_degenerate(m);
    sbh::EffectiveBvh b = sbh::build_effective_bvh(m);
    info[0] = b.full_nodes;
    info[1] = b.full_depth;
    info[2] = static_cast<int32_t>(b.nodes.size());
    info[3] = b.reachable_tris;
  });
}

sb_status sb_triangulate_ring(const double* ring_xy, uint32_t n, double* tris_out,
                              uint32_t max_tris, uint32_t* n_tris) {
  return guard([&] {
    std::vector<sbh::V2> ring(n);
    for (uint32_t i = 0; i < n; ++i) ring[i] = {ring_xy[2 * i], ring_xy[2 * i + 1]};
    auto t = sbh::triangulate_ring(ring);
    *n_tris = static_cast<uint32_t>(t.size());
    for (size_t i = 0; i < t.size() && i < max_tris; ++i)
      for (int k = 0; k < 3; ++k) {
        tris_out[6 * i + 2 * k] = t[i][k][0];
        tris_out[6 * i + 2 * k + 1] = t[i][k][1];
      }
  });
}

uint64_t sb_mix64(uint64_t x) { return sbh::mix64(x); }
uint64_t sb_stream_key(const uint64_t* parts, uint32_t n) {
  uint64_t h = 0x853c49e6748fea9bULL;
  for (uint32_t i = 0; i < n; ++i) h = sbh::mix64(h ^ parts[i]);
  return h;
}
sb_status sb_stream_doubles(uint64_t seed, const uint64_t* c, uint32_t nc, double* out, uint32_t n) {
  return guard([&] {
    uint64_t h = sbh::mix64(seed);
    for (uint32_t i = 0; i < nc; ++i) h = sbh::mix64(h ^ c[i]);
    const uint64_t mult = 6364136223846793005ULL, inc = (0xda3e39cb94b95bdbULL << 1u) | 1u;
    uint64_t st = inc;
    st += h;
    st = st * mult + inc;
    for (uint32_t k = 0; k < n; ++k) {
      uint64_t w = 0;
      for (int half = 0; half < 2; ++half) {
        uint64_t old = st;
        st = old * mult + inc;
        uint32_t xs = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
        uint32_t rot = static_cast<uint32_t>(old >> 59u);
        uint32_t r = (xs >> rot) | (xs << ((32u - rot) & 31u));
        w = (w << 32) | r;
      }
      out[k] = static_cast<double>(w >> 11) * 0x1.0p-53;
    }
  });
}

sb_status sb_world_create(uint64_t n, double margin, int device, sb_world** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("out is NULL");
    *out = new sb_world(n, margin, device);
  });
}
void sb_world_destroy(sb_world* w) { delete w; }
sb_status sb_register_geometry(sb_world* w, const double* v, uint32_t nv, const uint32_t* t,
                               uint32_t nt, int32_t* id) {
  return guard([&] { *id = w->register_geometry(mesh_in(v, nv, t, nt)); });
}
sb_status sb_add_object(sb_world* w, const char* name, int32_t geom, int32_t* id) {
  return guard([&] { *id = w->add_object(name ? name : "", geom); });
}
sb_status sb_set_enabled(sb_world* w, int32_t obj, const uint32_t* inst, uint64_t n, int en) {
  return guard([&] { w->set_enabled(obj, inst, n, en != 0); });
}
sb_status sb_set_enabled_all(sb_world* w, int32_t obj, int en) {
  return guard([&] { w->set_enabled_all(obj, en != 0); });
}
sb_status sb_update_transforms(sb_world* w, int32_t obj, const double* poses) {
  return guard([&] { w->update_transforms(obj, poses); });
}
sb_status sb_update_transform(sb_world* w, int32_t obj, uint64_t inst, const double pose[16]) {
  return guard([&] { w->update_transform(obj, inst, pose); });
}
sb_status sb_object_pose(sb_world* w, int32_t obj, uint64_t inst, double pose[16]) {
  return guard([&] { w->object_pose(obj, inst, pose); });
}
sb_status sb_enabled(sb_world* w, int32_t obj, uint64_t inst, int* en) {
  return guard([&] { *en = w->enabled(obj, inst) ? 1 : 0; });
}
sb_status sb_check_batch(sb_world* w, int32_t geom, const double* poses, const uint32_t* active,
                         uint64_t m, uint8_t* free_out, int32_t* contact_out) {
  return guard([&] { w->check_batch(geom, poses, active, m, free_out, contact_out); });
}
sb_status sb_get_stats(sb_world* w, sb_stats* out) {
  return guard([&] { *out = w->stats; });
}
sb_status sb_reset_stats(sb_world* w) {
  return guard([&] { w->stats = sb_stats{}; });
}

sb_status sb_engine_create(const sb_scene* sc, const sb_shard* shard, int device, sb_engine** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("out is NULL");
    *out = new sb_engine(sc, shard, device);
  });
}
void sb_engine_destroy(sb_engine* e) { delete e; }
sb_status sb_engine_generate(sb_engine* e, uint64_t run_seed, sb_result* out, sb_run_stats* st) {
  return guard([&] {
    e->generate(run_seed, st, out);  // results (if requested) are downloaded by generate
  });
}
sb_status sb_engine_download(sb_engine* e, sb_result* out) {
  return guard([&] { e->download(out); });
}
sb_world* sb_engine_world(sb_engine* e) { return e->world.get(); }
uint64_t sb_engine_local_instances(const sb_engine* e) { return e->n; }
uint64_t sb_engine_last_launches(const sb_engine* e) { return e->last_launches; }
sb_status sb_debug_narrow_profile(uint64_t out[8]) {
  return guard([&] {
    unsigned long long v[8], u[8];
    sbk::narrow_profile(v, true);        // placement kernels (sb_place.cu)
    sbk::narrow_profile_check(u, true);  // world API check_batch (sb_kernels.cu)
    for (int k = 0; k < 8; ++k) out[k] = v[k] + u[k];
  });
}

sb_status sb_debug_region_profile(uint64_t out[8]) {
  return guard([&] {
    unsigned long long v[8];
    sbk::region_profile(v, true);
    for (int k = 0; k < 8; ++k) out[k] = v[k];
  });
}

sb_status sb_device_math(int fn, const double* in, uint64_t n, double* out) {
  return guard([&] {
    if (fn < 0 || fn > 2) throw std::invalid_argument("sb_device_math: fn must be 0, 1 or 2");
    current_device_checked(0);
    const uint64_t nin = fn == 2 ? 2 * n : n;
    DevArray<double> din, dout;
    din.alloc(nin);
    dout.alloc(n);
    cuda_check(cudaMemcpy(din.p, in, nin * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    sbk::debug_math(fn, din.p, n, dout.p, nullptr);
    cuda_check(cudaMemcpy(out, dout.p, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  });
}

sb_status sb_engine_phase_profile(const sb_engine* e, double out[16]) {
  return guard([&] {
    const_cast<sb_engine*>(e)->resolve_timing();
    for (int k = 0; k < 16; ++k) out[k] = e->last_prof[k];
  });
}
sb_status sb_engine_last_timing(const sb_engine* e, double* total_ms, double* check_ms,
                                uint64_t* check_launches) {
  return guard([&] {
    const_cast<sb_engine*>(e)->resolve_timing();
    if (total_ms) *total_ms = e->last_total_ms;
    if (check_ms) *check_ms = e->last_check_ms;
    if (check_launches) *check_launches = e->last_check_launches;
  });
}

}  // extern "C"

// ===================================================================== PositionSampler
// The reference's PositionSampler (sampler.hpp:66-96, sampler.cpp:54-127) as a standalone
// device-backed object. The SampleCache (sampler.hpp:18-36) is kept on the host as FIFO
// ranges of draw indices of the cache stream -- a queued point is fully determined by its
// draw index (polygon.cpp:390-391: 3 doubles = 6 PCG steps per point) and by the region
// table, which only changes together with the fingerprint (and then clears the queue).
// So refill / drain / bind_stream are index bookkeeping, and the points themselves are
// drawn on the device by jump-ahead (k_sampler_fifo), one thread per active entry.
namespace {

// region_fingerprint (polygon.cpp:422-444) of hole-free parts.
uint64_t rings_fingerprint(const double* xy, const uint32_t* off, uint32_t r0, uint32_t r1) {
  uint64_t h = 0x9e3779b97f4a7c15ULL;
  auto feed = [&h](double v) {
    uint64_t bits;
    std::memcpy(&bits, &v, sizeof bits);
    h = sbh::mix64(h ^ bits);
  };
  for (uint32_t r = r0; r < r1; ++r) {
    h = sbh::mix64(h ^ static_cast<uint64_t>(off[r + 1] - off[r]));
    for (uint32_t k = off[r]; k < off[r + 1]; ++k) {
      feed(xy[2 * k]);
      feed(xy[2 * k + 1]);
    }
  }
  return h;
}

sbh::SamplerTable rings_table(const double* xy, const uint32_t* off, uint32_t r0, uint32_t r1) {
  std::vector<std::vector<sbh::V2>> parts;
  for (uint32_t r = r0; r < r1; ++r) {
    std::vector<sbh::V2> ring;
    for (uint32_t k = off[r]; k < off[r + 1]; ++k) ring.push_back({xy[2 * k], xy[2 * k + 1]});
    parts.push_back(std::move(ring));
  }
  return sbh::sampler_table(parts);
}

uint64_t cache_state0(uint64_t run_seed, uint64_t salt) {  // Pcg32(make_stream(seed, {salt, "cach"}))
  const uint64_t h = sbh::mix64(sbh::mix64(sbh::mix64(run_seed) ^ salt) ^ 0x63616368ULL);
  const uint64_t mult = 6364136223846793005ULL, inc = (0xda3e39cb94b95bdbULL << 1u) | 1u;
  uint64_t st = inc;
  st += h;
  return st * mult + inc;
}

}  // namespace

struct sb_sampler {
  uint64_t salt;
  int device;
  cudaStream_t stream = nullptr;
  bool prepared = false, per_instance = false, region_empty = true;
  uint64_t n = 0, run_seed = 0, region_fp = 0;
  int region_nt = 0;
  // SampleCache (sampler.hpp:18-36): queue of [first, end) draw-index ranges
  uint64_t cache_fp = 0, cache_stream = 0, refill_count = 0, queue_size = 0, rng_pos = 0;
  std::vector<std::pair<uint64_t, uint64_t>> queue;  // front at queue_head
  size_t queue_head = 0;
  DevArray<SbRegionTri> d_tris;  // canonical table, or all per-instance tables
  DevArray<double> d_cum;
  DevArray<uint32_t> d_inst_tab;  // per instance: (first table row, rows)
  bool stride_tables = false;     // relation tables: [n][table_cap] rows, d_inst_n each
  int table_cap = 0;
  DevArray<int32_t> d_inst_n;
  DevArray<double> d_states;
  DevArray<int32_t> d_rflags;
  DevArray<sbk::SbArcTable> d_arcs;
  DevArray<double> d_sup, d_pos;
  DevArray<uint32_t> d_active;
  DevArray<uint8_t> d_pl;
  DevArray<uint64_t> d_seg;
  PinnedArray<double> h_sup;
  PinnedArray<uint64_t> h_seg;

  sb_sampler(uint64_t salt_, int dev) : salt(salt_), device(current_device_checked(dev)) {
    cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
  }
  ~sb_sampler() {
    if (ev_seg) cudaEventDestroy(ev_seg);
    if (stream) {
      cudaSetDevice(device);
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
  }

  void clear_queue() {
    queue.clear();
    queue_head = 0;
    queue_size = 0;
  }

  // PositionSampler::prepare (sampler.cpp:54-67) + the region tables PolygonSampler builds.
  void prepare(const double* xy, const uint32_t* off, uint32_t n_rings, const uint32_t* inst_rings,
               uint64_t batch, uint64_t seed) {
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    if (n_rings && (!xy || !off)) throw std::invalid_argument("ring arrays are NULL");
    for (uint32_t r = 0; r < n_rings; ++r)
      if (off[r + 1] < off[r]) throw std::invalid_argument("ring_offsets must be non-decreasing");
    if (batch > 0xffffffffull) throw std::invalid_argument("batch_size exceeds 2^32");
    std::vector<SbRegionTri> tris;
    std::vector<double> cum;
    if (inst_rings) {
      std::vector<uint32_t> tab(2 * batch);
      std::unordered_map<uint64_t, uint64_t> seen;  // ring range -> first instance using it
      for (uint64_t i = 0; i < batch; ++i) {
        const uint32_t r0 = inst_rings[i], r1 = inst_rings[i + 1];
        if (r1 < r0 || r1 > n_rings) throw std::invalid_argument("instance_rings out of range");
        auto ins = seen.emplace((static_cast<uint64_t>(r0) << 32) | r1, i);
        if (!ins.second) {  // same rings as an earlier instance: share its table
          tab[2 * i] = tab[2 * ins.first->second];
          tab[2 * i + 1] = tab[2 * ins.first->second + 1];
          continue;
        }
        auto t = rings_table(xy, off, r0, r1);
        tab[2 * i] = static_cast<uint32_t>(tris.size());
        tab[2 * i + 1] = static_cast<uint32_t>(t.tris.size());
        tris.insert(tris.end(), t.tris.begin(), t.tris.end());
        cum.insert(cum.end(), t.cum.begin(), t.cum.end());
      }
      d_inst_tab.ensure(std::max<uint64_t>(1, 2 * batch));
      if (batch)
        cuda_check(cudaMemcpy(d_inst_tab.p, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice),
                   "H2D instance tables");
    } else {
      region_empty = n_rings == 0;
      region_fp = rings_fingerprint(xy, off, 0, n_rings);
      auto t = rings_table(xy, off, 0, n_rings);
      tris = std::move(t.tris);
      cum = std::move(t.cum);
      region_nt = static_cast<int>(tris.size());
    }
    d_tris.ensure(std::max<size_t>(1, tris.size()));
    d_cum.ensure(std::max<size_t>(1, cum.size()));
    if (!tris.empty()) {
      cuda_check(cudaMemcpy(d_tris.p, tris.data(), tris.size() * sizeof(SbRegionTri), cudaMemcpyHostToDevice), "H2D table");
      cuda_check(cudaMemcpy(d_cum.p, cum.data(), cum.size() * sizeof(double), cudaMemcpyHostToDevice), "H2D table");
    }
    per_instance = inst_rings != nullptr;
    stride_tables = false;
    n = batch;
    run_seed = seed;
    const uint64_t parts[3] = {seed, salt, 0x63616368ULL};  // bind_stream(stream_key(...))
    uint64_t key = 0x853c49e6748fea9bULL;
    for (uint64_t p : parts) key = sbh::mix64(key ^ p);
    if (cache_stream != key) {
      clear_queue();
      cache_stream = key;
    }
    rng_pos = 0;  // cache_rng_ = make_stream(run_seed, {salt, "cach"})
    prepared = true;
  }

  // build_constraint_region (relationships.cpp:161-218) on the device for a batch of
  // anchor states (x, y, yaw per instance, support frame), then prepare(). The region
  // kernel decides per_instance exactly as the reference (any anchor moving by > 1e-12);
  // a canonical region's cache fingerprint is a hash of its sampler table (the polygon
  // itself never leaves the device).
  void prepare_relation(const sb_relation& rel, const double rect[4], const double* states,
                        uint64_t batch, uint64_t seed) {
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    if (batch == 0) throw std::invalid_argument("anchor state batch is empty");
    if (batch > 0xffffffffull) throw std::invalid_argument("batch_size exceeds 2^32");
    SbPlacementDev pd;
    std::memset(&pd, 0, sizeof pd);
    const bool hole = relation_to_dev(rel, pd);
    for (int k = 0; k < 4; ++k) pd.rect[k] = rect[k];
    if (rel.anchor < 0) {  // no anchors: region = support (relationships.cpp:168-171)
      const double xy[8] = {rect[0], rect[1], rect[2], rect[1], rect[2], rect[3], rect[0], rect[3]};
      const uint32_t off[2] = {0, 4};
      prepare(xy, off, 1, nullptr, batch, seed);
      return;
    }
    if (!states) throw std::invalid_argument("anchor states are NULL");
    int sms = 0;
    cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "attr");
    table_cap = hole ? sbp::kHoleCap : SB_REGION_MAX_VERTS;
    d_tris.ensure(batch * table_cap);
    d_cum.ensure(batch * table_cap);
    d_inst_n.ensure(batch);
    d_states.ensure(3 * batch);
    d_rflags.ensure(2);
    cuda_check(cudaMemcpyAsync(d_states.p, states, 3 * batch * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D states");
    cuda_check(cudaMemsetAsync(d_rflags.p, 0, 2 * sizeof(int32_t), stream), "memset");
    sbk::RelationRegionParams rp;
    std::memset(&rp, 0, sizeof rp);
    rp.w.n = batch;
    rp.pl = pd;
    rp.anchor_object = -1;
    rp.cap = table_cap;
    rp.hole = hole ? 1 : 0;
    sbk::SbArcTable arc_tab;
    if (!hole && sbk::arc_table_host(pd, arc_tab)) {
      d_arcs.ensure(1);
      cuda_check(cudaMemcpyAsync(d_arcs.p, &arc_tab, sizeof arc_tab, cudaMemcpyHostToDevice, stream), "H2D arcs");
      rp.arcs = d_arcs.p;
    }
    rp.states = d_states.p;
    rp.tris = d_tris.p;
    rp.cum = d_cum.p;
    rp.ntri = d_inst_n.p;
    rp.flags = d_rflags.p;
    sbk::relation_regions(rp, sms, reinterpret_cast<sb_stream_t>(stream));
    int32_t flags[2], n0 = 0;
    cuda_check(cudaMemcpyAsync(flags, d_rflags.p, sizeof flags, cudaMemcpyDeviceToHost, stream), "D2H flags");
    cuda_check(cudaMemcpyAsync(&n0, d_inst_n.p, 4, cudaMemcpyDeviceToHost, stream), "D2H n");
    cuda_check(cudaStreamSynchronize(stream), "sync");
    if (flags[1] != 0)
      throw std::runtime_error("constraint region build failed (status " + std::to_string(flags[1]) + ")");
    per_instance = flags[0] != 0;
    stride_tables = true;
    n = batch;
    region_nt = per_instance ? 0 : n0;
    region_empty = !per_instance && n0 == 0;  // an empty (or zero-area) region_for(0)
    if (!per_instance && n0 > 0) {  // fingerprint of the canonical table
      std::vector<SbRegionTri> t(n0);
      std::vector<double> c(n0);
      cuda_check(cudaMemcpy(t.data(), d_tris.p, n0 * sizeof(SbRegionTri), cudaMemcpyDeviceToHost), "D2H table");
      cuda_check(cudaMemcpy(c.data(), d_cum.p, n0 * sizeof(double), cudaMemcpyDeviceToHost), "D2H table");
      uint64_t h = 0x9e3779b97f4a7c15ULL ^ 0x7461626cULL;  // "tabl": never a ring fingerprint
      auto feed = [&h](const void* p, size_t bytes) {
        const uint64_t* w = static_cast<const uint64_t*>(p);
        for (size_t k = 0; k < bytes / 8; ++k) h = sbh::mix64(h ^ w[k]);
      };
      feed(t.data(), t.size() * sizeof(SbRegionTri));
      feed(c.data(), c.size() * sizeof(double));
      region_fp = h;
    }
    run_seed = seed;
    const uint64_t parts[3] = {seed, salt, 0x63616368ULL};
    uint64_t key = 0x853c49e6748fea9bULL;
    for (uint64_t q : parts) key = sbh::mix64(key ^ q);
    if (cache_stream != key) {
      clear_queue();
      cache_stream = key;
    }
    rng_pos = 0;
    prepared = true;
  }

  // refill_cache (sampler.cpp:14-28) on draw indices
  void refill(uint64_t k) {
    if (region_fp != cache_fp) {
      clear_queue();
      cache_fp = region_fp;
    }
    uint64_t target = static_cast<uint64_t>(4.0 * static_cast<double>(k));
    if (target < k) target = k;
    if (queue_size >= target) return;
    const uint64_t need = target - queue_size;
    queue.push_back({rng_pos, rng_pos + need});
    rng_pos += need;
    queue_size += need;
    ++refill_count;
  }

  // drain_cache (sampler.cpp:30-43): pops k points as segments (first entry, first draw).
  int drain(uint64_t k) {
    if (region_fp != cache_fp || queue_size < k) refill(std::max<uint64_t>(k, 1));
    std::vector<uint64_t> first, draw;
    uint64_t j = 0;
    while (j < k) {
      auto& r = queue[queue_head];
      const uint64_t take = std::min(k - j, r.second - r.first);
      first.push_back(j);
      draw.push_back(r.first);
      r.first += take;
      j += take;
      if (r.first == r.second) ++queue_head;
    }
    queue_size -= k;
    if (queue_head > 64 && queue_head * 2 > queue.size()) {
      queue.erase(queue.begin(), queue.begin() + queue_head);
      queue_head = 0;
    }
    const int nseg = static_cast<int>(first.size());
    h_seg.ensure(std::max(2, 2 * nseg));
    std::copy(first.begin(), first.end(), h_seg.p);
    std::copy(draw.begin(), draw.end(), h_seg.p + nseg);
    return nseg;
  }

  void sample(const double* support, const uint32_t* active, uint64_t m, uint64_t attempt,
              double* pos, uint8_t* placeable) {
    if (!prepared) throw std::logic_error("PositionSampler: prepare() not called");
    if (m && (!active || !pos || !placeable || !support))
      throw std::invalid_argument("sample: NULL array");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    if (!per_instance && region_empty) {  // sampler.cpp:81-84
      std::memset(pos, 0, 3 * m * sizeof(double));
      std::memset(placeable, 0, m);
      return;
    }
    if (!per_instance && region_nt == 0)
      throw std::invalid_argument("sample: canonical region has zero area");
    if (m == 0) {
      if (!per_instance) drain(0);
      return;
    }
    h_sup.ensure(12 * m);
    for (uint64_t j = 0; j < m; ++j) {
      if (active[j] >= n) throw std::out_of_range("sample: active index >= batch_size");
      colmajor_to_34(support + 16 * static_cast<uint64_t>(active[j]), h_sup.p + 12 * j);
    }
    d_sup.ensure(12 * m);
    d_pos.ensure(3 * m);
    cuda_check(cudaMemcpyAsync(d_sup.p, h_sup.p, 12 * m * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D support");
    if (!per_instance) {
      const int nseg = drain(m);
      d_seg.ensure(2 * nseg);
      cuda_check(cudaMemcpyAsync(d_seg.p, h_seg.p, 2 * nseg * sizeof(uint64_t), cudaMemcpyHostToDevice, stream), "H2D segments");
      sbk::sampler_fifo(d_sup.p, nullptr, nullptr, m, d_seg.p, d_seg.p + nseg, nseg,
                        cache_state0(run_seed, salt),
                        d_tris.p, d_cum.p, region_nt, d_pos.p, stream);
      cuda_check(cudaMemcpyAsync(pos, d_pos.p, 3 * m * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H positions");
      cuda_check(cudaStreamSynchronize(stream), "sync");
      std::memset(placeable, 1, m);
      return;
    }
    d_active.ensure(m);
    d_pl.ensure(m);
    cuda_check(cudaMemcpyAsync(d_active.p, active, m * 4, cudaMemcpyHostToDevice, stream), "H2D active");
    sbk::sampler_fallback(d_sup.p, nullptr, d_active.p, m, run_seed, salt, attempt,
                          stride_tables ? nullptr : d_inst_tab.p, d_inst_n.p, table_cap, d_tris.p,
                          d_cum.p, d_pos.p, d_pl.p, stream);
    cuda_check(cudaMemcpyAsync(pos, d_pos.p, 3 * m * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H positions");
    cuda_check(cudaMemcpyAsync(placeable, d_pl.p, m, cudaMemcpyDeviceToHost, stream), "D2H placeable");
    cuda_check(cudaStreamSynchronize(stream), "sync");
  }

  // Device-resident variant: supports (N column-major Mat4), active, positions and
  // placeable are device pointers; everything is enqueued on `st` (no host round trip but
  // the SampleCache bookkeeping, which stays on the host).
  cudaEvent_t ev_seg = nullptr;
  void sample_device(const double* d_sup16, const uint32_t* d_act, uint64_t m, uint64_t attempt,
                     double* d_out, uint8_t* d_placeable, cudaStream_t st) {
    if (!prepared) throw std::logic_error("PositionSampler: prepare() not called");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    if (m && (!d_sup16 || !d_act || !d_out || !d_placeable))
      throw std::invalid_argument("sample_device: NULL array");
    if (!per_instance && region_empty) {
      if (m) {
        cuda_check(cudaMemsetAsync(d_out, 0, 3 * m * sizeof(double), st), "memset");
        cuda_check(cudaMemsetAsync(d_placeable, 0, m, st), "memset");
      }
      return;
    }
    if (!per_instance && region_nt == 0)
      throw std::invalid_argument("sample: canonical region has zero area");
    if (!per_instance) {
      if (!ev_seg) cuda_check(cudaEventCreateWithFlags(&ev_seg, cudaEventDisableTiming), "event");
      cuda_check(cudaEventSynchronize(ev_seg), "sync segments");  // h_seg reusable
      const int nseg = drain(m);
      if (m == 0) return;
      d_seg.ensure(2 * nseg);
      cuda_check(cudaMemcpyAsync(d_seg.p, h_seg.p, 2 * nseg * sizeof(uint64_t), cudaMemcpyHostToDevice, st), "H2D segments");
      cuda_check(cudaEventRecord(ev_seg, st), "event");
      sbk::sampler_fifo(nullptr, d_sup16, d_act, m, d_seg.p, d_seg.p + nseg, nseg,
                        cache_state0(run_seed, salt), d_tris.p, d_cum.p, region_nt, d_out,
                        reinterpret_cast<sb_stream_t>(st));
      cuda_check(cudaMemsetAsync(d_placeable, 1, m, st), "memset");
      return;
    }
    if (m == 0) return;
    sbk::sampler_fallback(nullptr, d_sup16, d_act, m, run_seed, salt, attempt,
                          stride_tables ? nullptr : d_inst_tab.p, d_inst_n.p, table_cap, d_tris.p,
                          d_cum.p, d_out, d_placeable, reinterpret_cast<sb_stream_t>(st));
  }
};

namespace {
struct OrientScratch {  // per host thread: reused device buffers of sb_sample_orientations
  int device = -1;
  cudaStream_t stream = nullptr;
  DevArray<uint32_t> active;
  DevArray<double> pos, face, yaws;
  void bind(int dev) {
    if (device == dev) return;
    active.release();
    pos.release();
    face.release();
    yaws.release();
    if (stream) cudaStreamDestroy(stream);
    stream = nullptr;
    device = dev;
    cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
  }
};
thread_local OrientScratch g_orient;
}  // namespace

extern "C" {

sb_status sb_sampler_create(uint64_t salt, int device, sb_sampler** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("out is NULL");
    *out = new sb_sampler(salt, device);
  });
}
void sb_sampler_destroy(sb_sampler* s) { delete s; }
sb_status sb_sampler_prepare(sb_sampler* s, const double* xy, const uint32_t* off, uint32_t n_rings,
                             const uint32_t* inst_rings, uint64_t n, uint64_t run_seed) {
  return guard([&] { s->prepare(xy, off, n_rings, inst_rings, n, run_seed); });
}
sb_status sb_sampler_sample(sb_sampler* s, const double* support, const uint32_t* active, uint64_t m,
                            uint64_t attempt, double* pos, uint8_t* placeable) {
  return guard([&] { s->sample(support, active, m, attempt, pos, placeable); });
}
sb_status sb_sampler_prepare_relation(sb_sampler* s, const sb_relation* rel,
                                      const double support_rect[4], const double* anchor_states,
                                      uint64_t n, uint64_t run_seed) {
  return guard([&] {
    if (!rel || !support_rect) throw std::invalid_argument("relation / support rect is NULL");
    s->prepare_relation(*rel, support_rect, anchor_states, n, run_seed);
  });
}
sb_status sb_sampler_sample_device(sb_sampler* s, const double* d_support16, const uint32_t* d_active,
                                   uint64_t m, uint64_t attempt, double* d_positions,
                                   uint8_t* d_placeable, void* cuda_stream) {
  return guard([&] {
    s->sample_device(d_support16, d_active, m, attempt, d_positions, d_placeable,
                     static_cast<cudaStream_t>(cuda_stream));
  });
}
sb_status sb_sampler_cache_info(const sb_sampler* s, uint64_t* queue_size, uint64_t* refills) {
  return guard([&] {
    if (queue_size) *queue_size = s->queue_size;
    if (refills) *refills = s->refill_count;
  });
}

// sample_orientations (sampler.cpp:129-156)
sb_status sb_sample_orientations(int kind, const uint32_t* active, uint64_t m, const double* pos,
                                 const double* face_xy, uint64_t n_targets, uint64_t run_seed,
                                 uint64_t salt, uint64_t attempt, double* yaws, int device) {
  return guard([&] {
    if (kind < SB_ORIENT_FIXED || kind > SB_ORIENT_FACE_TO)
      throw std::invalid_argument("sample_orientations: unknown orientation kind");
    if (kind == SB_ORIENT_FACE_TO && !face_xy)
      throw std::invalid_argument("sample_orientations: face_to target positions missing");
    if (m && (!active || !yaws || (kind == SB_ORIENT_FACE_TO && !pos)))
      throw std::invalid_argument("sample_orientations: NULL array");
    if (kind == SB_ORIENT_FACE_TO)
      for (uint64_t j = 0; j < m; ++j)
        if (active[j] >= n_targets)
          throw std::out_of_range("sample_orientations: active index >= n_targets");
    current_device_checked(device);
    if (m == 0) return;
    OrientScratch& o = g_orient;
    o.bind(device);
    o.active.ensure(m);
    o.yaws.ensure(m);
    cuda_check(cudaMemcpyAsync(o.active.p, active, m * 4, cudaMemcpyHostToDevice, o.stream), "H2D active");
    if (kind == SB_ORIENT_FACE_TO) {
      o.pos.ensure(3 * m);
      o.face.ensure(std::max<uint64_t>(1, 2 * n_targets));
      cuda_check(cudaMemcpyAsync(o.pos.p, pos, 3 * m * sizeof(double), cudaMemcpyHostToDevice, o.stream), "H2D positions");
      cuda_check(cudaMemcpyAsync(o.face.p, face_xy, 2 * n_targets * sizeof(double), cudaMemcpyHostToDevice, o.stream), "H2D targets");
    }
    sbk::orientations(kind, o.active.p, m, o.pos.p, o.face.p, run_seed, salt, attempt, o.yaws.p, o.stream);
    cuda_check(cudaMemcpyAsync(yaws, o.yaws.p, m * sizeof(double), cudaMemcpyDeviceToHost, o.stream), "D2H yaws");
    cuda_check(cudaStreamSynchronize(o.stream), "sync");
  });
}

}  // extern "C"

// ===================================================================== BatchedSceneGraph
// scene_graph.hpp:33-94. Names, parents and joint specs are host metadata; every per-
// instance batch (edges, bases, joint values, validity) lives in HBM (sb_graph.cu).
namespace {
bool homogeneous16(const double* m) {  // is_homogeneous (transform.hpp:28-30)
  return m[3] == 0.0 && m[7] == 0.0 && m[11] == 0.0 && m[15] == 1.0;
}
}  // namespace

struct sb_graph {
  uint64_t n;
  int device;
  cudaStream_t stream = nullptr;
  struct Node {
    std::string name;
    uint32_t parent = 0;
    int64_t geometry = -1;
    bool joint = false;
    sb_joint spec{};
    std::unique_ptr<DevArray<double>> edge, base, values;
  };
  std::vector<Node> nodes;
  std::unordered_map<std::string, uint32_t> by_name;
  DevArray<uint8_t> d_valid;
  mutable DevArray<double> d_tmp16;
  mutable DevArray<const double*> d_chain;
  mutable DevArray<unsigned long long> d_count;

  sb_graph(uint64_t batch, int dev) : n(batch), device(current_device_checked(dev)) {
    if (batch == 0) throw std::invalid_argument("batch_size must be >= 1");
    cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
    d_valid.alloc(n);
    cuda_check(cudaMemsetAsync(d_valid.p, 1, n, stream), "memset");
    Node world;
    world.name = "world";
    world.edge = std::make_unique<DevArray<double>>();
    identity_batch(*world.edge);
    by_name.emplace("world", 0);
    nodes.push_back(std::move(world));
    sync();
  }
  ~sb_graph() {
    if (ev_chain) cudaEventDestroy(ev_chain);
    if (stream) {
      cudaSetDevice(device);
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
  }
  sb_stream_t s() const { return reinterpret_cast<sb_stream_t>(stream); }
  void activate() const { cuda_check(cudaSetDevice(device), "cudaSetDevice"); }
  void sync() const { cuda_check(cudaStreamSynchronize(stream), "sync"); }

  void identity_batch(DevArray<double>& a) {
    a.alloc(12 * n);
    std::vector<double> one(16, 0.0);
    one[0] = one[5] = one[10] = one[15] = 1.0;
    d_tmp16.ensure(16 * n);
    std::vector<double> host(16 * n);
    for (uint64_t i = 0; i < n; ++i) std::memcpy(&host[16 * i], one.data(), sizeof(double) * 16);
    cuda_check(cudaMemcpyAsync(d_tmp16.p, host.data(), 16 * n * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D");
    sbk::graph_colmajor_to_34(d_tmp16.p, n, a.p, s());
    sync();
  }
  const Node& at(uint32_t id) const {
    if (id >= nodes.size()) throw std::out_of_range("unknown node");
    return nodes[id];
  }
  Node& at(uint32_t id) {
    if (id >= nodes.size()) throw std::out_of_range("unknown node");
    return nodes[id];
  }
  static sbk::GraphJoint gj(const sb_joint& j) {
    sbk::GraphJoint g;
    g.kind = j.kind;
    for (int k = 0; k < 3; ++k) g.axis[k] = j.axis[k];
    return g;
  }
  // edge = base * motion(values) over all instances (or motion alone when base == NULL)
  void compose(Node& nd, bool with_base) {
    sbk::graph_joint_compose(with_base ? nd.base->p : nullptr, nd.values->p, 0, n, gj(nd.spec),
                             nd.edge->p, s());
  }

  uint32_t add_node(uint32_t parent, const char* name_c, int64_t geometry, const sb_joint* joint) {
    activate();
    at(parent);
    if (!name_c) throw std::invalid_argument("node name is NULL");
    const std::string name(name_c);
    if (by_name.count(name)) throw std::invalid_argument("duplicate node name: " + name);
    Node nd;
    nd.name = name;
    nd.parent = parent;
    nd.geometry = geometry;
    nd.edge = std::make_unique<DevArray<double>>();
    if (joint) {  // JointSpec ctor (scene_graph.cpp:9-17)
      sb_joint j = *joint;
      if (j.kind != 0 && j.kind != 1) throw std::invalid_argument("JointSpec: unknown kind");
      if (j.lo > j.hi) throw std::invalid_argument("JointSpec: lo > hi");
      const double nrm = std::sqrt((j.axis[0] * j.axis[0] + j.axis[1] * j.axis[1]) + j.axis[2] * j.axis[2]);
      if (std::abs(nrm - 1.0) > 1e-9) {
        if (nrm < 1e-12) throw std::invalid_argument("JointSpec: zero axis");
        for (int k = 0; k < 3; ++k) j.axis[k] = j.axis[k] / nrm;
      }
      nd.joint = true;
      nd.spec = j;
      nd.base = std::make_unique<DevArray<double>>();
      identity_batch(*nd.base);
      nd.values = std::make_unique<DevArray<double>>();
      nd.values->alloc(n);
      std::vector<double> lo(n, j.lo);
      cuda_check(cudaMemcpyAsync(nd.values->p, lo.data(), n * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D");
      nd.edge->alloc(12 * n);
      compose(nd, false);  // every edge = motion(lo)
      sync();
    } else {
      identity_batch(*nd.edge);
    }
    const uint32_t id = static_cast<uint32_t>(nodes.size());
    by_name.emplace(name, id);
    nodes.push_back(std::move(nd));
    return id;
  }

  void set_edge_batch(uint32_t parent, uint32_t child, const double* t16) {
    activate();
    Node& nd = at(child);
    if (nd.parent != parent || child == 0)
      throw std::invalid_argument("no such edge: " + at(parent).name + " -> " + nd.name);
    if (!t16) throw std::invalid_argument("transform batch is NULL");
    for (uint64_t i = 0; i < n; ++i)
      if (!homogeneous16(t16 + 16 * i)) throw std::invalid_argument("non-homogeneous matrix in batch");
    d_tmp16.ensure(16 * n);
    cuda_check(cudaMemcpyAsync(d_tmp16.p, t16, 16 * n * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D");
    sbk::graph_colmajor_to_34(d_tmp16.p, n, nd.joint ? nd.base->p : nd.edge->p, s());
    if (nd.joint) compose(nd, true);
    sync();
  }

  void set_edge(uint32_t child, uint64_t i, const double* m16) {
    activate();
    Node& nd = at(child);
    if (child == 0) throw std::invalid_argument("cannot set edge on root");
    if (i >= n) throw std::out_of_range("instance out of range");
    if (!m16 || !homogeneous16(m16)) throw std::invalid_argument("non-homogeneous matrix");
    double r[12];
    colmajor_to_34(m16, r);
    double* dst = (nd.joint ? nd.base->p : nd.edge->p) + 12 * i;
    cuda_check(cudaMemcpyAsync(dst, r, sizeof r, cudaMemcpyHostToDevice, stream), "H2D");
    if (nd.joint)
      sbk::graph_joint_compose(nd.base->p, nd.values->p, i, 1, gj(nd.spec), nd.edge->p, s());
    sync();
  }

  void edge_batch(uint32_t child, double* out16) const {
    activate();
    const Node& nd = at(child);
    download16(nd.edge->p, out16);
  }
  void download16(const double* d12, double* out16) const {
    d_tmp16.ensure(16 * n);
    sbk::graph_34_to_colmajor(d12, n, d_tmp16.p, s());
    cuda_check(cudaMemcpyAsync(out16, d_tmp16.p, 16 * n * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
  }

  void set_joint_states(uint32_t node, const double* v) {
    activate();
    Node& nd = at(node);
    if (!nd.joint) throw std::invalid_argument("node is not articulated: " + nd.name);
    if (!v) throw std::invalid_argument("joint values are NULL");
    for (uint64_t i = 0; i < n; ++i)
      if (v[i] < nd.spec.lo - 1e-12 || v[i] > nd.spec.hi + 1e-12)
        throw std::invalid_argument("joint value out of limits for " + nd.name);
    cuda_check(cudaMemcpyAsync(nd.values->p, v, n * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D");
    compose(nd, true);
    sync();
  }
  void joint_states(uint32_t node, double* out) const {
    activate();
    const Node& nd = at(node);
    if (!nd.joint) throw std::invalid_argument("node is not articulated: " + nd.name);
    cuda_check(cudaMemcpyAsync(out, nd.values->p, n * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
  }

  // root -> node chain as device pointers, chain[0] = node
  int upload_chain(uint32_t node) const {
    std::vector<const double*> chain;
    for (uint32_t cur = node; cur != 0; cur = nodes[cur].parent) {
      chain.push_back(nodes[cur].edge->p);
      if (chain.size() > nodes.size()) throw std::logic_error("scene graph is not a tree");
    }
    if (!chain.empty()) {
      d_chain.ensure(chain.size());
      cuda_check(cudaMemcpyAsync(d_chain.p, chain.data(), chain.size() * sizeof(void*), cudaMemcpyHostToDevice, stream), "H2D chain");
    }
    return static_cast<int>(chain.size());
  }
  void world_poses(uint32_t node, double* out16) const {
    activate();
    at(node);
    const int depth = upload_chain(node);
    if (depth == 0) {  // the root: N identities
      download16(nodes[0].edge->p, out16);
      return;
    }
    d_tmp16.ensure(16 * n);
    sbk::graph_world_poses(d_chain.p, depth, n, d_tmp16.p, s());
    cuda_check(cudaMemcpyAsync(out16, d_tmp16.p, 16 * n * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
  }
  // batched FK into device memory on the caller's stream
  void world_poses_device(uint32_t node, double* d_out16, cudaStream_t st) const {
    activate();
    at(node);
    cuda_check(cudaStreamSynchronize(stream), "sync");  // the graph's own updates are done
    std::vector<const double*> chain;
    for (uint32_t cur = node; cur != 0; cur = nodes[cur].parent) chain.push_back(nodes[cur].edge->p);
    if (chain.empty()) {
      sbk::graph_34_to_colmajor(nodes[0].edge->p, n, d_out16, reinterpret_cast<sb_stream_t>(st));
      return;
    }
    if (!ev_chain) cuda_check(cudaEventCreateWithFlags(&ev_chain, cudaEventDisableTiming), "event");
    cuda_check(cudaEventSynchronize(ev_chain), "sync");  // the previous chain upload is consumed
    d_chain.ensure(chain.size());
    h_chain.ensure(chain.size());
    std::copy(chain.begin(), chain.end(), h_chain.p);
    cuda_check(cudaMemcpyAsync(d_chain.p, h_chain.p, chain.size() * sizeof(void*), cudaMemcpyHostToDevice, st), "H2D chain");
    sbk::graph_world_poses(d_chain.p, static_cast<int>(chain.size()), n, d_out16,
                           reinterpret_cast<sb_stream_t>(st));
    cuda_check(cudaEventRecord(ev_chain, st), "event");
  }
  mutable cudaEvent_t ev_chain = nullptr;
  mutable PinnedArray<const double*> h_chain;
  void world_pose(uint32_t node, uint64_t i, double* out16) const {
    activate();
    if (i >= n) throw std::out_of_range("instance out of range");
    at(node);
    const int depth = upload_chain(node);
    d_tmp16.ensure(16);
    sbk::graph_world_pose_one(d_chain.p, depth, i, d_tmp16.p, s());
    cuda_check(cudaMemcpyAsync(out16, d_tmp16.p, 16 * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
  }
  bool is_tree() const {  // scene_graph.cpp:174-187
    for (uint32_t i = 1; i < nodes.size(); ++i) {
      std::vector<bool> seen(nodes.size(), false);
      uint32_t cur = i;
      while (cur != 0) {
        if (seen[cur]) return false;
        seen[cur] = true;
        cur = nodes[cur].parent;
      }
    }
    return true;
  }
  uint64_t valid_count() const {
    activate();
    d_count.ensure(1);
    cuda_check(cudaMemsetAsync(d_count.p, 0, sizeof(unsigned long long), stream), "memset");
    sbk::graph_count_valid(d_valid.p, n, d_count.p, s());
    unsigned long long c = 0;
    cuda_check(cudaMemcpyAsync(&c, d_count.p, sizeof c, cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
    return c;
  }
};

void sb_engine::write_back(uint32_t p, sb_graph& g, uint32_t node) {
  if (p >= places.size()) throw std::out_of_range("placement index out of range");
  if (g.n != n) throw std::invalid_argument("write_back: graph batch size != engine local instances");
  if (g.device != world->device) throw std::invalid_argument("write_back: graph and engine on different devices");
  sb_graph::Node& nd = g.at(node);
  if (node == 0 || nd.parent != 0)
    throw std::invalid_argument("write_back: node must be a child of the root (world-frame edge)");
  world->activate();
  cuda_check(cudaStreamSynchronize(world->stream), "sync");  // the last run is complete
  const SbWorldView wv = world->view();
  sbk::graph_gather_object_poses(wv.pose, 12ull * static_cast<uint64_t>(places[p].dev.object),
                                 12ull * static_cast<uint64_t>(wv.obj_stride), n,
                                 nd.joint ? nd.base->p : nd.edge->p, g.s());
  if (nd.joint) g.compose(nd, true);
  sbk::graph_and_valid(g.d_valid.p, d_valid.p, n, g.s());
  g.sync();
}

extern "C" {

sb_status sb_graph_create(uint64_t batch, int device, sb_graph** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("out is NULL");
    *out = new sb_graph(batch, device);
  });
}
void sb_graph_destroy(sb_graph* g) { delete g; }
sb_status sb_graph_add_node(sb_graph* g, uint32_t parent, const char* name, int64_t geometry,
                            const sb_joint* joint, uint32_t* id) {
  return guard([&] {
    const uint32_t v = g->add_node(parent, name, geometry, joint);
    if (id) *id = v;
  });
}
sb_status sb_graph_set_edge_batch(sb_graph* g, uint32_t parent, uint32_t child, const double* t16) {
  return guard([&] { g->set_edge_batch(parent, child, t16); });
}
sb_status sb_graph_set_edge(sb_graph* g, uint32_t child, uint64_t i, const double pose[16]) {
  return guard([&] { g->set_edge(child, i, pose); });
}
sb_status sb_graph_edge_batch(const sb_graph* g, uint32_t child, double* out16) {
  return guard([&] { g->edge_batch(child, out16); });
}
sb_status sb_graph_set_joint_states(sb_graph* g, uint32_t node, const double* v) {
  return guard([&] { g->set_joint_states(node, v); });
}
sb_status sb_graph_joint_states(const sb_graph* g, uint32_t node, double* out) {
  return guard([&] { g->joint_states(node, out); });
}
sb_status sb_graph_world_poses(const sb_graph* g, uint32_t node, double* out16) {
  return guard([&] { g->world_poses(node, out16); });
}
sb_status sb_graph_world_pose(const sb_graph* g, uint32_t node, uint64_t i, double pose[16]) {
  return guard([&] { g->world_pose(node, i, pose); });
}
sb_status sb_graph_world_poses_device(const sb_graph* g, uint32_t node, double* d_out16,
                                      void* cuda_stream) {
  return guard([&] { g->world_poses_device(node, d_out16, static_cast<cudaStream_t>(cuda_stream)); });
}
sb_status sb_graph_find(const sb_graph* g, const char* name, int64_t* id) {
  return guard([&] {
    if (!name || !id) throw std::invalid_argument("NULL argument");
    auto it = g->by_name.find(name);
    *id = it == g->by_name.end() ? -1 : static_cast<int64_t>(it->second);
  });
}
sb_status sb_graph_node_info(const sb_graph* g, uint32_t node, const char** name, uint32_t* parent,
                             int64_t* geometry, int* articulated, sb_joint* joint) {
  return guard([&] {
    const sb_graph::Node& nd = g->at(node);
    if (name) *name = nd.name.c_str();
    if (parent) *parent = nd.parent;
    if (geometry) *geometry = nd.geometry;
    if (articulated) *articulated = nd.joint ? 1 : 0;
    if (joint && nd.joint) *joint = nd.spec;
  });
}
uint64_t sb_graph_node_count(const sb_graph* g) { return g->nodes.size(); }
sb_status sb_graph_children(const sb_graph* g, uint32_t node, uint32_t* out, uint32_t cap,
                            uint32_t* count) {
  return guard([&] {
    g->at(node);
    uint32_t c = 0;
    for (uint32_t i = 1; i < g->nodes.size(); ++i)
      if (g->nodes[i].parent == node) {
        if (out && c < cap) out[c] = i;
        ++c;
      }
    if (count) *count = c;
  });
}
sb_status sb_graph_is_tree(const sb_graph* g, int* t) {
  return guard([&] { *t = g->is_tree() ? 1 : 0; });
}
sb_status sb_graph_valid_mask(const sb_graph* g, uint8_t* mask) {
  return guard([&] {
    g->activate();
    cuda_check(cudaMemcpyAsync(mask, g->d_valid.p, g->n, cudaMemcpyDeviceToHost, g->stream), "D2H");
    g->sync();
  });
}
sb_status sb_graph_mark_invalid(sb_graph* g, uint64_t i) {
  return guard([&] {
    if (i >= g->n) throw std::out_of_range("instance out of range");
    g->activate();
    cuda_check(cudaMemsetAsync(g->d_valid.p + i, 0, 1, g->stream), "memset");
    g->sync();
  });
}
sb_status sb_graph_reset_validity(sb_graph* g) {
  return guard([&] {
    g->activate();
    cuda_check(cudaMemsetAsync(g->d_valid.p, 1, g->n, g->stream), "memset");
    g->sync();
  });
}
sb_status sb_graph_valid_count(const sb_graph* g, uint64_t* count) {
  return guard([&] { *count = g->valid_count(); });
}

sb_status sb_engine_write_back(sb_engine* e, uint32_t placement, sb_graph* g, uint32_t node) {
  return guard([&] { e->write_back(placement, *g, node); });
}

}  // extern "C"

// ===================================================================== ReachMap4D
// reachability.cpp:10-273. Grid metadata on the host (same arithmetic as the reference),
// occupancy bitsets and sample counts in HBM (sb_reach.cu), SBRM v1 files on the host.
struct sb_reach_map {
  int device;
  cudaStream_t stream = nullptr;
  uint64_t samples = 0;
  sbk::ReachGrid g{};
  uint64_t words = 0;
  DevArray<unsigned long long> d_occ, d_any, d_count;
  DevArray<unsigned> d_counts;  // empty after load
  DevArray<double> d_base, d_targets, d_frames;
  DevArray<const double*> d_frame_ptrs;
  DevArray<uint32_t> d_active;
  DevArray<uint8_t> d_out;

  explicit sb_reach_map(int dev) : device(current_device_checked(dev)) {
    cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
  }
  ~sb_reach_map() {
    if (stream) {
      cudaSetDevice(device);
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
  }
  sb_stream_t s() const { return reinterpret_cast<sb_stream_t>(stream); }
  void sync() const { cuda_check(cudaStreamSynchronize(stream), "sync"); }
  uint64_t cells() const { return g.nr * g.nz * g.npsi; }

  // occ_any from occ (build and load)
  void finish_any() {
    d_any.alloc(std::max<uint64_t>(1, (g.nr * g.nz + 63) / 64));
    cuda_check(cudaMemsetAsync(d_any.p, 0, d_any.count * 8, stream), "memset");
    sbk::reach_any(g, d_occ.p, d_any.p, s());
  }

  void build(const sb_chain_link* links, uint32_t n_links, const double* ee16, uint64_t n_samples,
             double res, double psi_res, uint64_t seed) {
    if (n_links == 0 || !links) throw std::invalid_argument("build: chain has no joints");
    if (n_samples < 1) throw std::invalid_argument("build: need at least one sample");
    if (res <= 0.0 || psi_res <= 0.0) throw std::invalid_argument("build: resolution must be positive");
    std::vector<double> L(18 * n_links);
    double ee[12];
    if (ee16) {
      if (!homogeneous16(ee16)) throw std::invalid_argument("build: non-homogeneous ee_offset");
      colmajor_to_34(ee16, ee);
    } else {
      for (int k = 0; k < 12; ++k) ee[k] = (k % 5 == 0) ? 1.0 : 0.0;
    }
    auto norm3 = [](double x, double y, double z) { return std::sqrt((x * x + y * y) + z * z); };
    double reach = norm3(ee[3], ee[7], ee[11]);  // KinematicChain::max_reach (:20-28)
    for (uint32_t l = 0; l < n_links; ++l) {
      const sb_chain_link& k = links[l];
      if (!homogeneous16(k.origin)) throw std::invalid_argument("build: non-homogeneous link origin");
      sb_joint j = k.joint;  // JointSpec ctor (scene_graph.cpp:9-17)
      if (j.kind != 0 && j.kind != 1) throw std::invalid_argument("JointSpec: unknown kind");
      if (j.lo > j.hi) throw std::invalid_argument("JointSpec: lo > hi");
      const double nrm = norm3(j.axis[0], j.axis[1], j.axis[2]);
      if (std::abs(nrm - 1.0) > 1e-9) {
        if (nrm < 1e-12) throw std::invalid_argument("JointSpec: zero axis");
        for (int c = 0; c < 3; ++c) j.axis[c] = j.axis[c] / nrm;
      }
      colmajor_to_34(k.origin, &L[18 * l]);
      L[18 * l + 12] = j.kind;
      for (int c = 0; c < 3; ++c) L[18 * l + 13 + c] = j.axis[c];
      L[18 * l + 16] = j.lo;
      L[18 * l + 17] = j.hi;
      reach += norm3(k.origin[12], k.origin[13], k.origin[14]);
      if (j.kind == 1) reach += std::max(std::abs(j.lo), std::abs(j.hi));
    }
    samples = n_samples;
    g.res = res;
    g.psi_res = psi_res;
    g.r_max = reach + res;
    g.z_min = -reach - res;
    g.z_max = reach + res;
    g.nr = static_cast<uint64_t>(std::ceil(g.r_max / res));
    g.nz = static_cast<uint64_t>(std::ceil((g.z_max - g.z_min) / res));
    g.npsi = static_cast<uint64_t>(std::ceil(M_PI / psi_res));
    if (cells() > (1ull << 34)) throw std::invalid_argument("build: grid too fine");
    words = (cells() + 63) / 64;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    d_occ.alloc(std::max<uint64_t>(1, words));
    d_counts.alloc(std::max<uint64_t>(1, cells()));
    cuda_check(cudaMemsetAsync(d_occ.p, 0, d_occ.count * 8, stream), "memset");
    cuda_check(cudaMemsetAsync(d_counts.p, 0, d_counts.count * 4, stream), "memset");
    DevArray<double> d_links;
    d_links.alloc(L.size());
    cuda_check(cudaMemcpyAsync(d_links.p, L.data(), L.size() * 8, cudaMemcpyHostToDevice, stream), "H2D");
    sbk::reach_build(d_links.p, static_cast<int>(n_links), ee, samples, seed, g, d_occ.p,
                     d_counts.p, s());
    finish_any();
    sync();
  }

  uint64_t occupied() const {
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    auto& self = const_cast<sb_reach_map&>(*this);
    self.d_count.ensure(1);
    cuda_check(cudaMemsetAsync(self.d_count.p, 0, 8, stream), "memset");
    sbk::reach_popcount(d_occ.p, words, self.d_count.p, s());
    unsigned long long c = 0;
    cuda_check(cudaMemcpyAsync(&c, self.d_count.p, 8, cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
    return c;
  }

  // SBRM v1 (reachability.cpp:192-273)
  void save(const char* path) const {
    if (!path) throw std::invalid_argument("path is NULL");
    std::vector<unsigned long long> occ(words);
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    if (words)
      cuda_check(cudaMemcpy(occ.data(), d_occ.p, words * 8, cudaMemcpyDeviceToHost), "D2H occ");
    FILE* f = std::fopen(path, "wb");
    if (!f) throw std::runtime_error(std::string("cannot open for write: ") + path);
    const uint32_t version = 1;
    const uint64_t hdr[1] = {samples};
    bool ok = std::fwrite("SBRM", 1, 4, f) == 4;
    ok = ok && std::fwrite(&version, 4, 1, f) == 1 && std::fwrite(hdr, 8, 1, f) == 1;
    const double dv[5] = {g.res, g.psi_res, g.r_max, g.z_min, g.z_max};
    ok = ok && std::fwrite(dv, 8, 5, f) == 5;
    const uint64_t nv[4] = {g.nr, g.nz, g.npsi, words};
    ok = ok && std::fwrite(nv, 8, 4, f) == 4;
    ok = ok && (words == 0 || std::fwrite(occ.data(), 8, words, f) == words);
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw std::runtime_error(std::string("write failed: ") + path);
  }
  void load(const char* path) {
    if (!path) throw std::invalid_argument("path is NULL");
    FILE* f = std::fopen(path, "rb");
    if (!f) throw std::runtime_error(std::string("cannot open reach map: ") + path);
    char magic[4];
    uint32_t version = 0;
    double dv[5];
    uint64_t nv[4];
    const bool head = std::fread(magic, 1, 4, f) == 4;
    if (!head || std::memcmp(magic, "SBRM", 4) != 0) {
      std::fclose(f);
      throw std::runtime_error(std::string("not a reach map file: ") + path);
    }
    if (std::fread(&version, 4, 1, f) != 1 || version != 1) {
      std::fclose(f);
      throw std::runtime_error("unsupported reach map version");
    }
    bool ok = std::fread(&samples, 8, 1, f) == 1 && std::fread(dv, 8, 5, f) == 5 &&
              std::fread(nv, 8, 4, f) == 4;
    std::vector<unsigned long long> occ;
    if (ok) {
      occ.resize(nv[3]);
      ok = nv[3] == 0 || std::fread(occ.data(), 8, nv[3], f) == nv[3];
    }
    std::fclose(f);
    if (!ok) throw std::runtime_error(std::string("truncated reach map: ") + path);
    g.res = dv[0];
    g.psi_res = dv[1];
    g.r_max = dv[2];
    g.z_min = dv[3];
    g.z_max = dv[4];
    g.nr = nv[0];
    g.nz = nv[1];
    g.npsi = nv[2];
    words = nv[3];
    if (words * 64 < cells()) throw std::runtime_error("reach map bitset shorter than its grid");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    d_occ.alloc(std::max<uint64_t>(1, words));
    if (words)
      cuda_check(cudaMemcpyAsync(d_occ.p, occ.data(), words * 8, cudaMemcpyHostToDevice, stream), "H2D occ");
    d_counts.release();
    finish_any();
    sync();
  }

  void query_batch(const double* base16, const double* targets, uint64_t n, bool has_incl,
                   double incl, uint8_t* out) {
    if (n && (!base16 || !targets || !out)) throw std::invalid_argument("query_batch: NULL array");
    if (!n) return;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    d_base.ensure(16 * n);
    d_targets.ensure(3 * n);
    d_out.ensure(n);
    cuda_check(cudaMemcpyAsync(d_base.p, base16, 16 * n * 8, cudaMemcpyHostToDevice, stream), "H2D");
    cuda_check(cudaMemcpyAsync(d_targets.p, targets, 3 * n * 8, cudaMemcpyHostToDevice, stream), "H2D");
    sbk::reach_query_batch(g, d_occ.p, d_any.p, d_base.p, d_targets.p, n,
                           has_incl ? incl : std::nan(""), d_out.p, s());
    cuda_check(cudaMemcpyAsync(out, d_out.p, n, cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
  }

  void placement_filter(const double* base16, uint64_t n, const double* const* frames,
                        uint32_t n_frames, const uint32_t* active, uint64_t m, uint8_t* out) {
    if (m && (!base16 || !active || !out)) throw std::invalid_argument("placement_filter: NULL array");
    if (!m) return;
    for (uint64_t j = 0; j < m; ++j)
      if (active[j] >= n) throw std::out_of_range("placement_filter: active index >= N");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    d_base.ensure(16 * n);
    cuda_check(cudaMemcpyAsync(d_base.p, base16, 16 * n * 8, cudaMemcpyHostToDevice, stream), "H2D");
    uint32_t present = 0;
    for (uint32_t f = 0; f < n_frames; ++f) present += frames && frames[f] ? 1 : 0;
    d_frames.ensure(std::max<uint64_t>(1, 16 * n * present));
    std::vector<const double*> ptrs(std::max<uint32_t>(1, n_frames), nullptr);
    for (uint32_t f = 0, k = 0; f < n_frames; ++f) {
      if (!frames || !frames[f]) continue;
      double* dst = d_frames.p + 16 * n * k++;
      cuda_check(cudaMemcpyAsync(dst, frames[f], 16 * n * 8, cudaMemcpyHostToDevice, stream), "H2D frames");
      ptrs[f] = dst;
    }
    d_frame_ptrs.ensure(ptrs.size());
    cuda_check(cudaMemcpyAsync(d_frame_ptrs.p, ptrs.data(), ptrs.size() * sizeof(void*), cudaMemcpyHostToDevice, stream), "H2D");
    d_active.ensure(m);
    d_out.ensure(m);
    cuda_check(cudaMemcpyAsync(d_active.p, active, m * 4, cudaMemcpyHostToDevice, stream), "H2D");
    sbk::reach_placement_filter(g, d_any.p, d_base.p, d_frame_ptrs.p, static_cast<int>(n_frames),
                                d_active.p, m, d_out.p, s());
    cuda_check(cudaMemcpyAsync(out, d_out.p, m, cudaMemcpyDeviceToHost, stream), "D2H");
    sync();
  }
};

extern "C" {

sb_status sb_reach_build(const sb_chain_link* links, uint32_t n_links, const double ee[16],
                         uint64_t samples, double res, double psi_res, uint64_t seed, int device,
                         sb_reach_map** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("out is NULL");
    std::unique_ptr<sb_reach_map> m(new sb_reach_map(device));
    m->build(links, n_links, ee, samples, res, psi_res, seed);
    *out = m.release();
  });
}
sb_status sb_reach_load(const char* path, int device, sb_reach_map** out) {
  return guard([&] {
    if (!out) throw std::invalid_argument("out is NULL");
    std::unique_ptr<sb_reach_map> m(new sb_reach_map(device));
    m->load(path);
    *out = m.release();
  });
}
sb_status sb_reach_save(const sb_reach_map* m, const char* path) {
  return guard([&] { m->save(path); });
}
void sb_reach_destroy(sb_reach_map* m) { delete m; }
sb_status sb_reach_get_info(const sb_reach_map* m, sb_reach_info* o) {
  return guard([&] {
    o->samples = m->samples;
    o->resolution = m->g.res;
    o->psi_resolution = m->g.psi_res;
    o->max_radius = m->g.r_max;
    o->z_min = m->g.z_min;
    o->z_max = m->g.z_max;
    o->nr = m->g.nr;
    o->nz = m->g.nz;
    o->npsi = m->g.npsi;
    o->cell_count = m->cells();
    o->occupied_cells = m->occupied();
  });
}
sb_status sb_reach_cell_samples(const sb_reach_map* m, uint64_t ir, uint64_t iz, uint64_t ip,
                                uint32_t* count) {
  return guard([&] {
    *count = 0;
    if (m->d_counts.count == 0) return;
    if (ir >= m->g.nr || iz >= m->g.nz || ip >= m->g.npsi) throw std::out_of_range("cell out of range");
    cuda_check(cudaSetDevice(m->device), "cudaSetDevice");
    const uint64_t idx = (ir * m->g.nz + iz) * m->g.npsi + ip;
    cuda_check(cudaMemcpy(count, m->d_counts.p + idx, 4, cudaMemcpyDeviceToHost), "D2H");
  });
}
sb_status sb_reach_query_batch(const sb_reach_map* m, const double* base16, const double* targets,
                               uint64_t n, int has_incl, double incl, uint8_t* out) {
  return guard([&] {
    const_cast<sb_reach_map*>(m)->query_batch(base16, targets, n, has_incl != 0, incl, out);
  });
}
sb_status sb_reach_query_batch_device(const sb_reach_map* m, const double* d_base16,
                                      const double* d_targets, uint64_t n, int has_incl,
                                      double incl, uint8_t* d_out, void* cuda_stream) {
  return guard([&] {
    if (!n) return;
    if (!d_base16 || !d_targets || !d_out) throw std::invalid_argument("query_batch: NULL array");
    cuda_check(cudaSetDevice(m->device), "cudaSetDevice");
    sbk::reach_query_batch(m->g, m->d_occ.p, m->d_any.p, d_base16, d_targets, n,
                           has_incl ? incl : std::nan(""), d_out,
                           reinterpret_cast<sb_stream_t>(static_cast<cudaStream_t>(cuda_stream)));
  });
}
sb_status sb_reach_placement_filter(const sb_reach_map* m, const double* base16, uint64_t n,
                                    const double* const* frames, uint32_t n_frames,
                                    const uint32_t* active, uint64_t m_active, uint8_t* out) {
  return guard([&] {
    const_cast<sb_reach_map*>(m)->placement_filter(base16, n, frames, n_frames, active, m_active, out);
  });
}

}  // extern "C"

extern "C" sb_status sb_engine_set_reach_filter(sb_engine* e, uint32_t placement,
                                                const sb_reach_map* m, const double* base16) {
  return guard([&] {
    if (placement >= e->places.size()) throw std::out_of_range("placement index out of range");
    e->reach.resize(e->places.size());
    sb_engine::ReachFilter& f = e->reach[placement];
    if (!m) {  // clear
      f = sb_engine::ReachFilter();
      return;
    }
    if (!base16) throw std::invalid_argument("robot base poses are NULL");
    if (m->device != e->world->device) throw std::invalid_argument("reach map on another device");
    std::vector<double> rows(12 * e->n);
    for (uint64_t i = 0; i < e->n; ++i) {
      if (!homogeneous16(base16 + 16 * i)) throw std::invalid_argument("non-homogeneous robot base pose");
      colmajor_to_34(base16 + 16 * i, &rows[12 * i]);
    }
    e->world->activate();
    f.base = std::make_unique<DevArray<double>>();
    f.base->alloc(rows.size());
    cuda_check(cudaMemcpy(f.base->p, rows.data(), rows.size() * sizeof(double), cudaMemcpyHostToDevice), "H2D base");
    f.any = m->d_any.p;
    f.grid = m->g;
  });
}
