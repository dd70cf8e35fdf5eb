// Host runtime + C ABI (include/scenebatch_b200.h). C++17, CUDA runtime API only.
//
// World  = CollisionWorld (collision.hpp:76-127) with all per-instance state in HBM.
// Engine = the reference's absent rejection loop (contract frozen in
//          DESIGN.md) driving the fused per-round kernel; one engine per GPU / shard.
#include "sb_comm.h"
#include "sb_rt.hpp"
#include "sb_graph_rt.hpp"
#include "sb_reach_rt.hpp"
#include "sb_glibcm.cuh"


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
  DevArray<uint64_t> d_xsend, d_xgather;  // relation exchange: [4] out, [world][4] in
  PinnedArray<unsigned long long> h_xrecv;
  int attempts = 0;

  struct Placement {
    SbPlacementDev dev;
    double support16[16];
    double inv_support[12];
    int canon_n = 0;  // host-built canonical table size (no anchor)
    bool hole = false;  // serial region path (holed annulus, wide sector, polygon support,
                        // middle / multi-anchor relation): k_relation_regions<true>
    std::vector<std::array<double, 2>> support_ring;  // the support polygon as given
    bool shared_arcs = false;  // arc table in d_arcs[p] (no local-frame direction)
    double ratio = 0.0;        // ratio_on_support (no-relation placements)
    int mesh = 0;
  };
  std::vector<Placement> places;
  std::vector<std::unique_ptr<DevArray<double>>> sup_frames;  // per-instance support frames
  int32_t first_place_obj = 0;
  int inst_cap = 0;  // region table stride (canonical and per instance)

  DevArray<uint8_t> d_valid;
  DevArray<int16_t> d_accepted;
  DevArray<uint32_t> d_tile_list;   // [ntiles * tile_inst] survivors per tile
  DevArray<uint32_t> d_tile_cnt;    // [2][ntiles]
  // wide round 0 (sbk::place_wide_round0) scratch, per round-0 slot (tile * kPlaceBlock + e)
  bool use_wide = false;
  unsigned wide_pgrid = 0;
  DevArray<double> d_wpose;
  DevArray<int32_t> d_wcontact;
  DevArray<uint32_t> d_wovm, d_wpairs, d_wpairs2, d_wpinst2, d_wtoff, d_wlist2;
  // dense placements: survivors after each wide round in the last run, and the wide rounds
  // the next run gives each placement (1 = round 0 only)
  DevArray<unsigned long long> d_wsurv;
  PinnedArray<unsigned long long> h_wsurv;
  std::vector<int> wide_rounds;
  unsigned long long wide_more = 32768;
  DevArray<uint32_t> d_wcnt2;
  // persistent fast rounds with a decoupled look-back on the tile counts instead of a grid
  // barrier per round (sbk lookback_rounds); SB_LOOKBACK=0: grid barrier
  bool lookback = true;
  // SB_PLACE1=1: FIFO placements without a relation run the 1-CTA-per-SM persistent kernel
  // (no register spills, half the warps) on grid1 CTAs
  bool place1 = true;
  bool fifo1 = false;  // every FIFO placement on the 1-CTA build (scenes without relations)
  unsigned grid1 = 0;
  unsigned long long place1_max = 8192;  // SB_PLACE1_MAX: survivors below which it is taken
  std::vector<char> place1_ok;           // per placement, from the previous run's survivors
  DevArray<unsigned long long> d_lb;  // [attempts + 1][ntiles]
  uint32_t lb_epoch = 0;
  uint32_t lb_sleep = 256;  // SB_LB_SLEEP: ns between polls (0 / 64 / 256: C1 0.744 / 0.735 / 0.727 ms)
  DevArray<uint8_t> d_wflag;
  DevArray<unsigned long long> d_wctl;
  DevArray<uint64_t> d_jump;        // FIFO draw jump table (sbd::pcg_jump_table_host)
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
  // SB_PLACE_EVENTS=1: an event pair around every placement (per-placement times). Off by
  // default: an event between two kernels breaks their programmatic-launch edge (C4 28.47 ->
  // 27.66 ms, C2 3.75 -> 3.60 ms without them); the run is then timed as one interval.
  bool place_events = false;
  bool timing_pending = false;
  std::vector<char> pending_per_inst;
  std::vector<uint32_t> pending_rounds;
  int num_sms = 0;
  // tile decomposition of the shard (sb_place.h) and launch shape of the placement kernel
  uint32_t ntiles = 0;
  int tile_inst = 0, tile_inst_pi = 0, max_tris = 1, max_nodes = 1, ws_bytes = 0;
  int spec_target = 64;
  // per-instance placements: each tile's processing time in the last run and the claim
  // order for the next one (slowest first); results do not depend on the order
  DevArray<uint32_t> d_tile_ns, d_tile_perm;
  PinnedArray<uint32_t> h_tile_ns;
  std::vector<char> tile_perm_ok;
  bool lpt_tiles = true;  // SB_LPT=0: claim order = tile order
  int solo_max = 0;  // SB_SOLO: CTA 0 alone below this many survivors (r02: off measured best, C2 +0.9 %, C4 -2.7 %)
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
  DevArray<uint64_t> d_seed;  // run seed read by the placement kernels (graph replays)
  PinnedArray<uint64_t> h_seed;
  struct GraphSlot {  // one captured run per result mode (poses piped or not)
    cudaGraphExec_t exec = nullptr;
    uint64_t launches = 0, round_launches = 0, gen = 0;
    SbWorldView view{};
  };
  GraphSlot graphs[2];
  uint64_t graph_gen = 0;  // bumped when a placement's launch parameters change
  bool use_graphs = std::getenv("SB_GRAPH") != nullptr;  // measured: no faster
  DevArray<unsigned long long> d_nvalid;
  bool host_times = std::getenv("SB_HOST_TIMES") != nullptr;  // end-of-run counters / ctrl words / region flags / timers  // [P][n][16] result poses written at accept (pipelined download)
  PinnedArray<uint64_t> h_count;
  cudaStream_t copy_stream = nullptr;  // pipelined result download
  std::vector<cudaEvent_t> ev_pose;
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
  cudaEvent_t ev_chunk[2] = {nullptr, nullptr};  // sharded FIFO rounds: chunk completion (no timing)

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
      if (sc->fixed[f].poses16) {  // a TransformBatch (update_transforms): this shard's range
        world->upload_poses(sc->fixed[f].poses16 + 16 * begin, n);
        sbk::update_transforms(world->view(), obj, world->d_scratch_poses.p, nullptr, n, 16, world->s());
      } else {
        require_homogeneous(sc->fixed[f].pose);
        world->upload_poses(sc->fixed[f].pose, 1);
        // broadcast one pose to every instance (stride 0)
        sbk::update_transforms(world->view(), obj, world->d_scratch_poses.p, nullptr, n, 0, world->s());
      }
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
      pl.dev.support_object = -1;
      if (sup.on_placement >= 0 || sup.poses16) {  // support_world per instance
        if (sup.on_placement >= 0 && static_cast<uint32_t>(sup.on_placement) >= p)
          throw std::invalid_argument("support on_placement must be an earlier placement");
        auto S = std::make_unique<DevArray<double>>();
        auto I = std::make_unique<DevArray<double>>();
        S->alloc(12 * n);
        I->alloc(12 * n);
        if (sup.on_placement >= 0) {
          pl.dev.support_object = first_place_obj + sup.on_placement;
        } else {
          for (uint64_t i = 0; i < n; ++i) require_homogeneous(sup.poses16 + 16 * (begin + i));
          world->upload_poses(sup.poses16 + 16 * begin, n);
          sbk::graph_colmajor_to_34(world->d_scratch_poses.p, n, S->p, world->s());
          sbk::support_frames(world->view(), -1, pl.dev.support, S->p, I->p, world->s());
          cuda_check(cudaStreamSynchronize(world->stream), "sync");
        }
        pl.dev.support_inst = S->p;
        pl.dev.inv_support_inst = I->p;
        sup_frames.push_back(std::move(S));
        sup_frames.push_back(std::move(I));
      }
      pl.support_ring = support_to_dev(sup, pl.dev);
      const sb_relation& r = sp.relation;
      // holed annulus / wide sector (erosion of those: only where the clipped ring is convex
      // and hole-free, else a region-build error as the reference's buffer throws)
      const bool big = relation_to_dev(r, pl.dev);
      if (sp.ratio_on_support != 0.0) {  // apply_ratio_on_support's checks (relationships.cpp:222-227)
        if (sp.ratio_on_support < 0.0 || sp.ratio_on_support > 1.0)
          throw std::invalid_argument("apply_ratio_on_support: ratio outside [0,1]");
        if (!(footprint[sp.mesh][0] > 0.0) || !(footprint[sp.mesh][1] > 0.0))
          throw std::invalid_argument("apply_ratio_on_support: footprint edges must be positive");
      }
      pl.ratio = sp.ratio_on_support;
      pl.mesh = sp.mesh;
      const int na = pl.dev.n_anchors;
      if (na > 0 && sp.ratio_on_support > 0.0)  // relation regions erode on the device
        pl.dev.erode_r = sp.ratio_on_support * std::min(footprint[sp.mesh][0], footprint[sp.mesh][1]) / 2.0;
      for (int k = 0; k < na; ++k) {
        const int32_t a = k == 0 ? r.anchor : r.extra_anchors[k - 1];
        if (a < 0 || static_cast<uint32_t>(a) >= p)
          throw std::invalid_argument("relationship: anchor must be an earlier placement");
        pl.dev.anchor_objects[k] = first_place_obj + a;
      }
      pl.dev.anchor_object = na > 0 ? pl.dev.anchor_objects[0] : -1;
      // serial per-instance region path (big_region_lane): ring shapes past the group
      // path's capacity, polygon supports, `middle` and multi-anchor relations
      pl.hole = big || (na > 0 && (pl.dev.poly_n > 0 || na > 1 || r.distance_type == SB_DIST_MIDDLE));
      pl.dev.serial = pl.hole ? 1 : 0;
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
      // region = the support polygon as given (relationships.cpp:168-171)
      std::vector<sbh::V2> ring;
      for (const auto& v : places[p].support_ring) ring.push_back({v[0], v[1]});
      if (places[p].ratio > 0.0) {  // apply_ratio_on_support (relationships.cpp:220-230)
        const auto& fp = footprint[places[p].mesh];
        const double r = places[p].ratio * std::min(fp[0], fp[1]) / 2.0;
        if (r > 0.0) {  // erode -> to_boost: bg::correct (counter-clockwise, vertex 0 first)
          double a = 0.0;
          for (size_t i = 0; i < ring.size(); ++i)
            a += ring[i][0] * ring[(i + 1) % ring.size()][1] - ring[(i + 1) % ring.size()][0] * ring[i][1];
          if (0.5 * a < 0.0) std::reverse(ring.begin() + 1, ring.end());
          ring = sbh::erode_convex(ring, r);
        }
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
      d_anchor.alloc(3 * SB_MAX_ANCHORS);  // instance 0's anchor states (sharded runs)
    }
    d_s0.alloc(3 * SB_MAX_ANCHORS);
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
    if (const char* e = std::getenv("SB_PLACE1")) place1 = std::atoi(e) != 0;
    grid1 = place1 ? static_cast<unsigned>(sbk::place_grid(num_sms, smem, true)) : 0u;
    if (const char* e = std::getenv("SB_PLACE1_MAX")) place1_max = std::strtoull(e, nullptr, 10);
    place1_ok.assign(places.size(), 0);
    bool any_fifo = false;
    for (const Placement& pl : places) any_fifo = any_fifo || pl.dev.anchor_object < 0;
    // wide round 0: single GPU, or sharded with the device-side exchange (round 0's counts
    // gathered between k_fast_init and the wide kernels); measured slower below 131072 (C2, C3)
    use_wide = (world_size == 1 || allgather_dev) && any_fifo && n >= 131072;
    if (const char* e = std::getenv("SB_WIDE"))
      use_wide = (world_size == 1 || allgather_dev) && any_fifo && std::atoi(e) != 0;
    {  // below the wide size, scenes without relation placements (every placement FIFO) take
       // the 1-CTA build on a tile layout sized for its grid: C1 0.730 -> 0.712 ms. With
       // relations it loses (the per-instance tiles want the warps: C2 3.34 -> 3.49, C3
       // 16.40 -> 18.35 ms), so SB_FIFO1=1 only forces it there.
      bool any_rel = false;
      for (const Placement& pl : places) any_rel = any_rel || pl.dev.anchor_object >= 0;
      fifo1 = !any_rel;
      if (const char* e = std::getenv("SB_FIFO1")) fifo1 = std::atoi(e) != 0;
      fifo1 = fifo1 && place1 && grid1 > 0 && world_size == 1 && !use_wide;
    }
    {  // tiles: a multiple of the grid, at most kPlaceBlock instances each
      const uint64_t per_wave = static_cast<uint64_t>(fifo1 ? grid1 : grid) * sbk::kPlaceBlock;
      const uint64_t waves = (n + per_wave - 1) / per_wave;
      const uint64_t want = static_cast<uint64_t>(fifo1 ? grid1 : grid) * waves;
      tile_inst = static_cast<int>((n + want - 1) / want);
      // Wide engines: full 256-instance tiles. Round 0's grid-wide kernels launch a CTA per
      // tile (no idle threads), and the persistent rounds work on the re-dealt survivor list,
      // so the tile count need not be a multiple of the persistent grid (SB_WIDE_FULL_TILES=0:
      // the balanced size).
      static const bool full_tiles = [] {
        const char* e = std::getenv("SB_WIDE_FULL_TILES");
        return !e || std::atoi(e) != 0;
      }();
      if (use_wide && full_tiles) tile_inst = sbk::kPlaceBlock;
      // per-instance placements: smaller tiles, taken dynamically, so a dense tile's heavy
      // narrow phase does not hold the whole placement (SB_PI_SPLIT; measured best: 1)
      // default: ~56 instances per per-instance tile (C2 at 55: split 1 / 2 / 4 = 3.76 / 3.97 /
      // 4.08 ms; C3 at 221: 19.35 / 19.11 / 18.88 ms)
      int split = std::max(1, (tile_inst + 40) / 56);
      if (const char* e = std::getenv("SB_PI_SPLIT")) split = std::max(1, std::atoi(e));
      tile_inst_pi = std::max(1, (tile_inst + split - 1) / split);
      ntiles = static_cast<uint32_t>((n + tile_inst - 1) / tile_inst);
      if ((ntiles + grid - 1) / grid > static_cast<uint32_t>(sbk::kPlaceMaxOwnedTiles))
        throw std::invalid_argument("shard too large for one device: " + std::to_string(n) + " instances");
    }
    d_tile_list.alloc(static_cast<size_t>(ntiles) * tile_inst);
    if (const char* e = std::getenv("SB_LPT")) lpt_tiles = std::atoi(e) != 0;
    {
      bool any_rel = false;
      for (const Placement& pl : places) any_rel = any_rel || pl.dev.anchor_object >= 0;
      // only with several per-instance tiles per CTA (C3: 4 -> 18.80 to 17.35 ms; C2 at ~1
      // per CTA: 3.72 -> 3.79 ms, so off there)
      lpt_tiles = lpt_tiles && any_rel && pp_ntiles_pi() * 2 > 3 * static_cast<size_t>(grid);
      if (lpt_tiles) {
        const size_t cnt = std::max<size_t>(1, places.size()) * pp_ntiles_pi();
        d_tile_ns.alloc(cnt);
        d_tile_perm.alloc(cnt);
        h_tile_ns.ensure(cnt);
        tile_perm_ok.assign(places.size(), 0);
      }
    }
    d_tile_cnt.alloc(2 * static_cast<size_t>(ntiles));
    if (const char* e = std::getenv("SB_LOOKBACK")) lookback = std::atoi(e) != 0;
    if (const char* e = std::getenv("SB_LB_SLEEP")) lb_sleep = static_cast<uint32_t>(std::atoi(e));
    if (lookback) {  // look-back count board of the persistent fast rounds, epochs from 1
      d_lb.alloc(static_cast<size_t>(attempts + 1) * ntiles);
      cuda_check(cudaMemset(d_lb.p, 0, d_lb.count * sizeof(unsigned long long)), "memset");
    }
    {  // wide round 0 scratch (use_wide decided above)
      wide_pgrid = grid;  // persistent grid for rounds >= 1 (SB_WIDE_PGRID: fewer CTAs)
      if (const char* e = std::getenv("SB_WIDE_PGRID"))
        wide_pgrid = std::max<unsigned>(
            (ntiles + sbk::kPlaceMaxOwnedTiles - 1) / sbk::kPlaceMaxOwnedTiles,  // owned-tile cap
            std::min<unsigned>(grid, static_cast<unsigned>(std::max(1, std::atoi(e)))));
      if (use_wide) {
        const size_t slots = static_cast<size_t>(ntiles) * sbk::kPlaceBlock;
        d_wpose.alloc(slots * sbk::kWideRec);
        d_wcontact.alloc(slots);
        d_wovm.alloc(slots * 8);
        d_wflag.alloc(slots);
        d_wpairs.alloc(std::max<size_t>(1, static_cast<size_t>(n) * world->view().n_objects));
        d_wpairs2.alloc(d_wpairs.count);
        d_wpinst2.alloc(d_wpairs.count);
        d_wtoff.alloc(ntiles);
        d_wctl.alloc(16);
        d_wsurv.alloc(static_cast<size_t>(sbk::kWideSurvRounds) * std::max<size_t>(1, places.size()));
        wide_rounds.assign(places.size(), 1);
        if (const char* e = std::getenv("SB_WIDE_MORE"))  // survivors that earn another wide round
          wide_more = std::strtoull(e, nullptr, 10);
        d_wcnt2.alloc(2 * static_cast<size_t>(ntiles));
        d_wlist2.alloc(static_cast<size_t>(ntiles) * tile_inst);
      }
    }
    {
      std::vector<uint64_t> jt(SB_PCG_JUMP_LEVELS * 256 * 2);
      sb_pcg_jump_table_host(jt.data());
      d_jump.alloc(jt.size());
      cuda_check(cudaMemcpy(d_jump.p, jt.data(), jt.size() * 8, cudaMemcpyHostToDevice), "H2D jump");
    }
    if (static_cast<uint64_t>(n) * static_cast<uint64_t>(attempts) >= (1ull << 32))
      throw std::invalid_argument("engine: variations x attempts per shard must stay below 2^32 draws");
    d_cpose.alloc(static_cast<size_t>(grid) * sbk::kPlaceBlock * 12);
    d_cinv.alloc(static_cast<size_t>(grid) * sbk::kPlaceBlock * 12);
    {  // occupancy grid over the supports' XY extent, widened by the largest object radius
      double bx0 = HUGE_VAL, by0 = HUGE_VAL, bx1 = -HUGE_VAL, by1 = -HUGE_VAL, rad = 0.0;
      for (uint32_t k = 0; k < sc->n_supports; ++k) {
        const sb_support& su = sc->supports[k];
        std::vector<std::array<double, 2>> pts;
        if (su.n_polygon >= 3 && su.polygon_xy) {
          for (uint32_t v = 0; v < su.n_polygon; ++v) pts.push_back({su.polygon_xy[2 * v], su.polygon_xy[2 * v + 1]});
        } else {
          pts = {{su.rect[0], su.rect[1]}, {su.rect[2], su.rect[1]}, {su.rect[2], su.rect[3]}, {su.rect[0], su.rect[3]}};
        }
        for (const auto& q : pts) {
          const double wx = su.pose[0] * q[0] + su.pose[4] * q[1] + su.pose[12];
          const double wy = su.pose[1] * q[0] + su.pose[5] * q[1] + su.pose[13];
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
    place_events = place_times;
    if (const char* e = std::getenv("SB_PLACE_EVENTS")) place_events = std::atoi(e) != 0 || place_times;
    if (const char* st = std::getenv("SB_SPEC_TARGET")) spec_target = std::max(1, std::atoi(st));
    if (const char* so = std::getenv("SB_SOLO")) solo_max = std::max(0, std::min(sbk::kPlaceBlock, std::atoi(so)));
    if (const char* ss = std::getenv("SB_SOLO_SPEC")) solo_spec = std::max(0, std::min(sbk::kPlaceBlock, std::atoi(ss)));
    if (round_debug) d_dbg.alloc(3 * static_cast<size_t>(attempts) * std::max<size_t>(1, places.size()) + 16);
    d_counters.alloc(8);
    cuda_check(cudaEventCreate(&ev_start), "event");
    cuda_check(cudaEventCreate(&ev_stop), "event");
    for (cudaEvent_t& e : ev_chunk) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    cuda_check(cudaDeviceSynchronize(), "sync");
  }

  ~sb_engine() {
    if (world) cudaSetDevice(world->device);
    for (GraphSlot& g : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    for (cudaEvent_t e : {ev_start, ev_stop, ev_chunk[0], ev_chunk[1]})
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

  // Instance 0's anchor states (x, y, yaw in the support frame) of every anchor into d_anchor.
  void anchor_states0(const Placement& pl, const SbWorldView& wv, uint64_t& launches) {
    SbWorldView w1 = wv;
    w1.n = 1;
    for (int k = 0; k < std::max(1, pl.dev.n_anchors); ++k) {
      sbk::anchor_states(w1, pl.dev.anchor_objects[k], pl.inv_support, pl.dev.inv_support_inst,
                         d_anchor.p + 3 * k, world->s());
      ++launches;
    }
  }

  // Sharded runs: instance 0's anchor state and the variation flag are exchanged.
  // Returns true if the anchors vary (per-instance path); else fills the canonical slot.
  bool relation_prep_sharded(size_t p, Placement& pl, const SbWorldView& wv, uint64_t& launches,
                             int& canon_n) {
    cudaStream_t stream = world->stream;
    sb_stream_t s = world->s();
    const int na = std::max(1, pl.dev.n_anchors);
    double s0[3 * SB_MAX_ANCHORS] = {};
    if (begin == 0) {
      anchor_states0(pl, wv, launches);
      cuda_check(cudaMemcpyAsync(s0, d_anchor.p, 3 * na * sizeof(double), cudaMemcpyDeviceToHost, stream), "D2H s0");
      cuda_check(cudaStreamSynchronize(stream), "sync");
    }
    std::vector<uint64_t> send(3 * na + 1, 0);
    std::memcpy(send.data(), s0, 3 * na * sizeof(double));
    send[3 * na] = begin == 0 ? 1 : 0;
    std::vector<uint64_t> recv = exchange(send);
    for (int r = 0; r < world_size; ++r)
      if (recv[(3 * na + 1) * r + 3 * na]) std::memcpy(s0, &recv[(3 * na + 1) * r], 3 * na * sizeof(double));
    cuda_check(cudaMemcpyAsync(d_s0.p, s0, 3 * na * sizeof(double), cudaMemcpyHostToDevice, stream), "H2D s0");
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

  // Sharded relation placement with the device exchange (sb_shard.allgather_dev): instance
  // 0's anchor state and the "anchors vary" flag travel through the device all-gather, and
  // both region sets are built -- this rank's per-instance tables and the canonical
  // region_for(0) from the exchanged state (relationships.cpp:178-190) -- so the path is
  // picked on the device (PlaceParams::shard_vary) with no host round trip.
  void relation_prep_sharded_dev(size_t p, Placement& pl, const SbWorldView& wv, uint64_t& launches) {
    sb_stream_t s = world->s();
    cudaStream_t stream = world->stream;
    const size_t W = static_cast<size_t>(world_size);
    // send words are unique per (placement, exchange): an all-gather may still read them
    // after this stream has moved on (the sb_shard contract allows a lazy reader)
    const int na = std::max(1, pl.dev.n_anchors);
    const uint32_t nsend = 3 * na + 1;
    d_xsend.ensure(32 * places.size());
    d_xgather.ensure((3 * SB_MAX_ANCHORS + 1) * W);
    uint64_t* send_anchor = d_xsend.p + 32 * p;
    uint64_t* send_flag = send_anchor + nsend;
    auto gather = [&](const uint64_t* send, uint32_t k) {
      if (allgather_dev(allgather_dev_ctx, send, k, d_xgather.p, stream) != 0)
        throw std::runtime_error("sb_shard.allgather_dev failed");
    };
    if (begin == 0) anchor_states0(pl, wv, launches);
    sbk::shard_anchor_pack(begin == 0 ? d_anchor.p : nullptr, na, send_anchor, s);
    gather(send_anchor, nsend);
    sbk::shard_anchor_pick(d_xgather.p, world_size, na, d_s0.p, s);
    launches += 2;
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
    sbk::shard_flag_pack(rp.flags, send_flag, s);
    gather(send_flag, 1);
    sbk::shard_flag_or(d_xgather.p, world_size, rp.flags, s);  // flags[0] = OR over ranks
    rp.from_s0 = 1;
    rp.tris = d_canon_tris.p + p * inst_cap;
    rp.cum = d_canon_cum.p + p * inst_cap;
    rp.ntri = d_canon_n.p + p;
    sbk::relation_regions(rp, num_sms, s);
    launches += 4;
  }

  // Results requested with the call (sb_engine_generate with an sb_result) are downloaded
  // while later placements compute: placement p's poses are final once its kernel ends, so
  // a copy stream converts them (k_pose_colmajor) and copies them to the host behind an event.
  // Placement-stepped runs (sb_engine_place): [run_lo, run_hi) of the last call; a run
  // is open while placements remain; counters that span calls accumulate in run_acc_*.
  size_t run_lo = 0, run_hi = 0;
  bool run_open = false;
  uint64_t run_seed_open = 0;
  uint64_t run_acc_rounds_host = 0, run_acc_per_inst = 0;
  std::vector<char> device_rounds_run;

  size_t pp_ntiles_pi() const {
    return static_cast<size_t>((n + tile_inst_pi - 1) / std::max(1, tile_inst_pi));
  }

  void generate(uint64_t run_seed, sb_run_stats* st, sb_result* out = nullptr) {
    generate_range(run_seed, 0, places.size(), st, out);
  }

  // Placements [lo, hi) of a run: lo == 0 starts a run (reset), lo > 0 continues the open
  // run at its next placement with the same seed; hi == P completes it (fixups, `out`).
  void generate_range(uint64_t run_seed, size_t lo, size_t hi, sb_run_stats* st,
                      sb_result* out = nullptr) {
    const size_t P_all = places.size();
    if (hi > P_all || lo > hi || (lo == hi && P_all != 0))
      throw std::invalid_argument("placement range out of bounds");
    if (lo > 0 && (!run_open || lo != run_hi || run_seed != run_seed_open))
      throw std::logic_error("sb_engine_place: continue the open run at its next placement with its seed");
    if (out && hi != P_all)
      throw std::invalid_argument("sb_engine_place: results are available when the run completes");
    const bool full = lo == 0 && hi == P_all;
    if (lo == 0) run_acc_rounds_host = run_acc_per_inst = 0;
    run_lo = lo;
    run_hi = hi;
    run_open = hi < P_all;
    run_seed_open = run_seed;
    const auto th0 = std::chrono::steady_clock::now();
    world->activate();
    const bool pipe = full && out && out->poses && !places.empty();
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
    std::vector<char> shard_dev_relation(places.size(), 0);
    std::vector<char> device_rounds(places.size(), world_size == 1 ? 1 : 0);
    while (ev_place.size() < 2 * P + 2) {
      cudaEvent_t e;
      cuda_check(cudaEventCreate(&e), "event");
      ev_place.push_back(e);
    }
    // The device work of one run. capturing: recorded into a CUDA graph (single GPU, replayed
    // by later calls; the run seed is read from d_seed on the device), so copies to the
    // caller's buffers stay outside and events are external event nodes.
    auto rec = [&](cudaEvent_t e, bool capturing) {
      cuda_check(capturing ? cudaEventRecordWithFlags(e, stream, cudaEventRecordExternal)
                           : cudaEventRecord(e, stream),
                 "event");
    };
    h_seed.ensure(1);
    d_seed.ensure(1);
    if (lo == 0) {
      h_seed.p[0] = run_seed;
      cuda_check(cudaMemcpyAsync(d_seed.p, h_seed.p, 8, cudaMemcpyHostToDevice, stream), "H2D seed");
    }
    auto enqueue = [&](bool capturing) {
      rec(ev_start, capturing);
      if (lo == 0) {  // a new run: reset the world's placed objects, counters, grid
        cuda_check(cudaMemsetAsync(d_counters.p, 0, 8 * sizeof(unsigned long long), stream), "memset");
        cuda_check(cudaMemsetAsync(d_prof.p, 0, 8 * sizeof(uint64_t), stream), "memset");
        if (round_debug) cuda_check(cudaMemsetAsync(d_dbg.p, 0, d_dbg.count * sizeof(unsigned), stream), "memset");
        cuda_check(cudaMemsetAsync(d_ctrl.p, 0, d_ctrl.count * sizeof(uint32_t), stream), "memset");
        cuda_check(cudaMemsetAsync(d_rflags.p, 0, d_rflags.count * sizeof(int32_t), stream), "memset");
        sbk::engine_reset(wv, first_place_obj, static_cast<int32_t>(P), d_valid.p, d_accepted.p,
                          static_cast<int32_t>(P), s);
        launches += 1;
        if (cell_grid.g) {
          sbk::cells_reset(wv, cell_grid, first_place_obj, s);
          ++launches;
        }
      }
      for (size_t p = lo; p < hi; ++p) {
        Placement& pl = places[p];
        bool fast = true;
        int canon_n = pl.canon_n;
        const SbRegionTri* canon_tris = d_canon_tris.p + p * inst_cap;
        const double* canon_cum = d_canon_cum.p + p * inst_cap;
        const bool relation = pl.dev.anchor_object >= 0;
        if (place_events) rec(ev_place[2 * p], capturing);
        if (pl.dev.support_object >= 0) {  // surface of a placed object: this run's poses
          sbk::support_frames(wv, pl.dev.support_object, pl.dev.support,
                              const_cast<double*>(pl.dev.support_inst),
                              const_cast<double*>(pl.dev.inv_support_inst), s);
          ++launches;
        }
        bool dev_relation = false;  // sharded, path picked on the device
        if (relation) {
          if (world_size == 1) {
            relation_prep_device(p, pl, wv, launches);
          } else if (allgather_dev) {
            relation_prep_sharded_dev(p, pl, wv, launches);
            dev_relation = true;
            shard_dev_relation[p] = 1;
          } else {
            fast = !relation_prep_sharded(p, pl, wv, launches, canon_n);
            if (!fast) ++per_inst_host;
          }
        }
        if (place_events) rec(ev_place[2 * p + 1], capturing);
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
        pp.seed_dev = d_seed.p;
        pp.global_begin = begin;
        pp.fast_state0 = fast_state0;
        pp.jump = d_jump.p;
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
        if (relation && lpt_tiles) {
          pp.tile_ns = d_tile_ns.p + static_cast<size_t>(p) * pp_ntiles_pi();
          pp.tile_perm = tile_perm_ok[p] ? d_tile_perm.p + static_cast<size_t>(p) * pp_ntiles_pi() : nullptr;
        }
        if (p < reach.size() && reach[p].any) {
          pp.reach_any = reach[p].any;
          pp.reach_grid = reach[p].grid;
          pp.reach_base = reach[p].base->p;
        }
        if (world_size == 1) {
          const bool one = place1 && !relation && grid1 > 0 && ((use_wide && place1_ok[p]) || fifo1) &&
                           (ntiles + grid1 - 1) / grid1 <= static_cast<uint32_t>(sbk::kPlaceMaxOwnedTiles);
          if (use_wide && !relation) {  // round 0 grid-wide, then the persistent kernel
            pp.w_pose = d_wpose.p;
            pp.w_contact = d_wcontact.p;
            pp.w_ovm = d_wovm.p;
            pp.w_flag = d_wflag.p;
            pp.w_pairs = d_wpairs.p;
            pp.w_pairs2 = d_wpairs2.p;
            pp.w_pinst2 = d_wpinst2.p;
            pp.w_toff = d_wtoff.p;
            pp.w_ctl = d_wctl.p;
            pp.w_list2 = d_wlist2.p;
            pp.w_cnt2 = d_wcnt2.p;
            pp.w_surv = d_wsurv.p + sbk::kWideSurvRounds * p;
            // dense placements (the last run left >= wide_more survivors after round r) run
            // round r + 1 grid-wide too; the persistent kernel takes the rounds after
            const int R = std::min<int>(attempts, wide_rounds[p]);
            sbk::place_fast_init(pp, grid, smem, s);
            ++launches;
            for (int r = 0; r < R; ++r) {
              pp.wide_round = r;
              launches += sbk::place_wide_round0_a(pp, num_sms, s);
              launches += sbk::place_wide_round0_c(pp, grid, s, one ? grid1 : wide_pgrid, r + 1 == R);
            }
            pp.start_round = R;  // rounds R.. on the re-dealt survivor list
            pp.start_draws = d_wctl.p + 4;
            pp.tile_list = d_wlist2.p;
            pp.tile_cnt = d_wcnt2.p;
            pp.ntiles_dev = d_wctl.p + 6;
          }
          pp.lb_board = nullptr;
          if (lookback && d_lb.p && !capturing) {
            pp.lb_board = d_lb.p;
            pp.lb_stride = ntiles;
            if (++lb_epoch == 0) ++lb_epoch;
            pp.lb_epoch = lb_epoch;
            pp.lb_sleep = lb_sleep;
          }
          if (!sbk::place_persistent(pp, one ? grid1 : use_wide && !relation ? wide_pgrid : grid, smem, s, one))
            throw CudaError("cooperative launch of the placement kernel is not possible");
          ++launches;
          ++round_launches;
        } else if (!fast) {
          // per-instance regions: tiles are independent, no exchange
          device_rounds[p] = 1;
          sbk::place_instances(pp, grid, smem, s);
          ++launches;
          ++round_launches;
        } else if (allgather_dev) {
          if (dev_relation) {  // per-instance kernel first; each side no-ops on the other path
            device_rounds[p] = 1;
            pp.shard_vary = d_rflags.p + 2 * p;
            pp.canon_n_dev = d_canon_n.p + p;
            sbk::place_instances(pp, grid, smem, s);
            ++launches;
            ++round_launches;
          }
          // FIFO fast path, device-side exchange: round a's kernel reads the gathered counts
          // and the draws before it from device memory, the all-gather of its survivors is
          // enqueued behind it; the host checks for completion once per kChunk rounds.
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
          sbk::place_fast_init(pp, grid, smem, s);
          ++launches;
          gather(0);
          int32_t a = 0;
          if (use_wide && !relation) {
            // round 0 grid-wide (draw base from the gathered counts), survivors left in
            // their tiles for the per-round kernels, this rank's count gathered for round 1
            pp.w_pose = d_wpose.p;
            pp.w_contact = d_wcontact.p;
            pp.w_ovm = d_wovm.p;
            pp.w_flag = d_wflag.p;
            pp.w_pairs = d_wpairs.p;
            pp.w_pairs2 = d_wpairs2.p;
            pp.w_pinst2 = d_wpinst2.p;
            pp.w_toff = d_wtoff.p;
            pp.w_ctl = d_wctl.p;
            launches += sbk::place_wide_round0_rest(pp, grid, num_sms, s, 0, false);
            ++round_launches;
            gather(1);
            a = 1;
          }
          // The host stays one chunk of rounds ahead of the device: after enqueuing chunk
          // c it reads the gathered total at the end of chunk c-1 (copied behind an event,
          // normally complete by then), so the device never idles on the host; rounds
          // enqueued past the last one with survivors return at once.
          int pending = -1;  // ev_chunk slot whose total is in flight
          int32_t pending_round = 0;
          for (;;) {
            const int32_t stop = std::min<int32_t>(attempts, a + kChunk);
            for (; a < stop; ++a) {
              sbk::place_fast_round(pp, a, grid, smem, s);
              launches += 1;
              round_launches += 1;
              gather(a + 1);
            }
            const int slot = pending == 0 ? 1 : 0;
            cuda_check(cudaMemcpyAsync(h_xrecv.p + a * W, d_xrecv.p + a * W, W * 8, cudaMemcpyDeviceToHost, stream), "D2H counts");
            cuda_check(cudaEventRecord(ev_chunk[slot], stream), "event");
            bool done = a >= attempts;
            if (pending >= 0) {
              cuda_check(cudaEventSynchronize(ev_chunk[pending]), "sync chunk");
              uint64_t t = 0;
              for (size_t r = 0; r < W; ++r) t += h_xrecv.p[static_cast<size_t>(pending_round) * W + r];
              done = done || t == 0;
            }
            pending = slot;
            pending_round = a;
            if (done) break;
          }
          cuda_check(cudaMemcpyAsync(h_xrecv.p, d_xrecv.p, K1 * W * 8, cudaMemcpyDeviceToHost, stream), "D2H counts");
          cuda_check(cudaStreamSynchronize(stream), "sync");
          for (int32_t r = 0; r < a; ++r) {  // rounds the reference runs: total > 0
            uint64_t t = 0;
            for (size_t k = 0; k < W; ++k) t += h_xrecv.p[r * W + k];
            if (t > 0) ++rounds_host;
          }
          if (a == attempts && h_xrecv.p[static_cast<size_t>(a) * W + rank] > 0) {
            pp.xrecv = nullptr;  // mark this rank's K-attempt survivors invalid
            sbk::place_fast_finish(pp, a, grid, s);
            ++launches;
          }
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
              sbk::place_fast_round(pp, a, grid, smem, s);
              launches += 1;
              round_launches += 1;
              m = read_total(a + 1);
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
        if (pipe) {  // identity result poses where placement p accepted nothing
          sbk::out16_fixup(n, d_accepted.p + p * n, d_out16.p + p * 16 * n, s);
          ++launches;
        }
        if (pipe && capturing) {  // graph: the copy follows the launch (graph_copies)
          rec(ev_pose[p], true);
        } else if (pipe) {  // placement p is final: copy its poses behind an event
          // (k_place wrote them at accept: a DMA only, no SM work beside the next placement)
          cuda_check(cudaEventRecord(ev_pose[p], stream), "event");
          cuda_check(cudaStreamWaitEvent(copy_stream, ev_pose[p], 0), "wait");
          cuda_check(cudaMemcpyAsync(out->poses + 16 * n * p, d_out16.p + 16 * n * p,
                                     16 * n * sizeof(double), cudaMemcpyDeviceToHost, copy_stream),
                     "D2H poses");
        }
      }
      if (hi == P) {  // objects left unaccepted keep add_object's identity pose / local box
        sbk::unaccepted_fixup(wv, first_place_obj, static_cast<int32_t>(P), d_accepted.p, s);
        ++launches;
      }
    };
    const bool graphable = full && world_size == 1 && !round_debug && !place_times && use_graphs;
    if (graphable) {
      GraphSlot& gs = graphs[pipe ? 1 : 0];
      const SbWorldView now = world->view();
      if (!gs.exec || gs.gen != graph_gen || std::memcmp(&now, &gs.view, sizeof now) != 0) {
        if (gs.exec) cudaGraphExecDestroy(gs.exec);
        gs.exec = nullptr;
        const uint64_t l0 = launches, r0 = round_launches;
        cuda_check(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal), "begin capture");
        try {
          enqueue(true);
        } catch (...) {
          cudaGraph_t gbad = nullptr;
          cudaStreamEndCapture(stream, &gbad);
          if (gbad) cudaGraphDestroy(gbad);
          throw;
        }
        cudaGraph_t gr = nullptr;
        cuda_check(cudaStreamEndCapture(stream, &gr), "end capture");
        const cudaError_t ie = cudaGraphInstantiate(&gs.exec, gr, 0);
        cudaGraphDestroy(gr);
        cuda_check(ie, "graph instantiate");
        gs.launches = launches - l0;
        gs.round_launches = round_launches - r0;
        gs.view = now;
        gs.gen = graph_gen;
      } else {
        launches += gs.launches;
        round_launches += gs.round_launches;
      }
      cuda_check(cudaGraphLaunch(gs.exec, stream), "graph launch");
      if (pipe)  // graph_copies: each placement's poses behind its event, on the copy stream
        for (size_t p = 0; p < P; ++p) {
          cuda_check(cudaStreamWaitEvent(copy_stream, ev_pose[p], 0), "wait");
          cuda_check(cudaMemcpyAsync(out->poses + 16 * n * p, d_out16.p + 16 * n * p,
                                     16 * n * sizeof(double), cudaMemcpyDeviceToHost, copy_stream),
                     "D2H poses");
        }
    } else {
      enqueue(false);
    }
    if (out) {
      if (out->poses && !pipe && P) {  // a stepped run's last call: poses from the world
        d_pose16.ensure(16 * n);
        for (size_t p = 0; p < P; ++p) {
          sbk::download_poses(world->view(), places[p].dev.object, d_pose16.p, s);
          ++launches;
          cuda_check(cudaMemcpyAsync(out->poses + 16 * n * p, d_pose16.p, 16 * n * sizeof(double),
                                     cudaMemcpyDeviceToHost, stream), "D2H poses");
        }
      }
      if (out->accepted && P)
        cuda_check(cudaMemcpyAsync(out->accepted, d_accepted.p, P * n * sizeof(int16_t), cudaMemcpyDeviceToHost, stream), "D2H accepted");
      if (out->valid)
        cuda_check(cudaMemcpyAsync(out->valid, d_valid.p, n, cudaMemcpyDeviceToHost, stream), "D2H valid");
    }
    cuda_check(cudaEventRecord(ev_place[2 * hi], stream), "event");
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
    if (lpt_tiles && full)
      cuda_check(cudaMemcpyAsync(h_tile_ns.p, d_tile_ns.p, d_tile_ns.count * 4, cudaMemcpyDeviceToHost, stream),
                 "D2H tile times");
    const bool wide_hist = use_wide && world_size == 1 && full;
    if (wide_hist) {
      h_wsurv.ensure(d_wsurv.count);
      cuda_check(cudaMemcpyAsync(h_wsurv.p, d_wsurv.p, d_wsurv.count * 8, cudaMemcpyDeviceToHost, stream),
                 "D2H wide survivors");
    }
    if (st) {  // valid instances counted on the device (no N-byte readback)
      d_nvalid.ensure(1);
      cuda_check(cudaMemsetAsync(d_nvalid.p, 0, 8, stream), "memset");
      sbk::graph_count_valid(d_valid.p, n, d_nvalid.p, s);
      ++launches;
      cuda_check(cudaMemcpyAsync(nvalid, d_nvalid.p, 8, cudaMemcpyDeviceToHost, stream), "D2H nvalid");
    }
    const auto th1 = std::chrono::steady_clock::now();
    cuda_check(cudaStreamSynchronize(stream), "sync");
    const auto th2 = std::chrono::steady_clock::now();
    if (wide_hist) {  // the next run's wide rounds per placement from this run's survivors
      for (size_t p = 0; p < P; ++p) {
        const int R = wide_rounds[p];
        const unsigned long long* sv = h_wsurv.p + sbk::kWideSurvRounds * p;
        int r_next = 1;
        while (r_next < std::min(R + 1, sbk::kWideSurvRounds) && sv[r_next - 1] >= wide_more) ++r_next;
        wide_rounds[p] = r_next;
        // few survivors after the wide rounds: the next run's persistent rounds take the
        // 1-CTA-per-SM kernel (a latency chain of a handful of instances per CTA)
        if (place1_ok.size() == P) place1_ok[p] = R >= 1 && sv[std::min(R, sbk::kWideSurvRounds) - 1] < place1_max;
      }
    }
    for (size_t p = lo; p < hi; ++p) {
      if (rflags[2 * p + 1] != 0)
        throw std::runtime_error("constraint region build failed for placement " + std::to_string(p) +
                                 " (status " + std::to_string(rflags[2 * p + 1]) +
                                 ": capacity overflow or unsupported annulus)");
    }
    // CUDA-event timings are resolved lazily (resolve_timing: ~2.5 us per
    // cudaEventElapsedTime, 2 per placement) -- only phase_profile / last_timing need them.
    pending_per_inst.assign(P, 0);
    for (size_t p = lo; p < hi; ++p)
      pending_per_inst[p] = places[p].dev.anchor_object >= 0 && rflags[2 * p] != 0;
    if (lpt_tiles && full) {  // next run: each per-instance placement's slowest tiles first
      const size_t nt = pp_ntiles_pi();
      std::vector<uint32_t> perm(nt);
      for (size_t p = 0; p < P; ++p) {
        if (!pending_per_inst[p]) continue;
        const uint32_t* ns = h_tile_ns.p + p * nt;
        for (size_t k = 0; k < nt; ++k) perm[k] = static_cast<uint32_t>(k);
        std::stable_sort(perm.begin(), perm.end(), [&](uint32_t x, uint32_t y) { return ns[x] > ns[y]; });
        cuda_check(cudaMemcpy(d_tile_perm.p + p * nt, perm.data(), nt * 4, cudaMemcpyHostToDevice), "H2D tile order");
        tile_perm_ok[p] = 1;
      }
    }
    pending_rounds.assign(P, 0);
    for (size_t p = lo; p < hi; ++p) pending_rounds[p] = device_rounds[p] ? ctrl_all[8 * p + 2] : 0u;
    timing_pending = true;
    const auto th2a = std::chrono::steady_clock::now();
    if (lo == 0) device_rounds_run.assign(P, 0);
    for (size_t p = lo; p < hi; ++p) device_rounds_run[p] = device_rounds[p];
    run_acc_rounds_host += rounds_host;
    uint64_t rounds = run_acc_rounds_host;  // the run so far (placements [0, hi))
    for (size_t p = 0; p < hi; ++p)
      if (device_rounds_run[p]) rounds += ctrl_all[8 * p + 2];
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
      uint64_t per_inst_dev = 0;  // sharded relation placements decided on the device
      for (size_t p = lo; p < hi; ++p) per_inst_dev += shard_dev_relation[p] && rflags[2 * p] != 0;
      run_acc_per_inst += per_inst_host + per_inst_dev;
      st->per_instance_placements = c[7] + run_acc_per_inst;
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
    for (size_t p = run_lo; p < run_hi && p < P && !place_events; ++p) {
      // no per-placement events: the run's device time split evenly (phase profile only)
      const double b = total_ms / (double)(run_hi - run_lo);
      place_ms += b;
      (pending_per_inst[p] ? inst_ms : fast_ms) += b;
    }
    for (size_t p = run_lo; p < run_hi && p < P && place_events; ++p) {
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
    last_check_ms = place_ms;  // placement intervals (sharded: incl. exchange waits)
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
sb_status sb_load_obj(const char* path, double* v, uint32_t* nv, uint32_t* t, uint32_t* nt) {
  return guard([&] {
    if (!path) throw std::invalid_argument("path is NULL");
    mesh_out(sbh::load_obj(path), v, nv, t, nt);
  });
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

sb_status sb_extract_support_surfaces(const double* vertices, uint32_t n_vertices,
                                      const uint32_t* triangles, uint32_t n_triangles,
                                      int32_t mode, sb_surface* out, uint32_t cap,
                                      uint32_t* n_out) {
  return guard([&] {
    if (!n_out || (cap && !out)) throw std::invalid_argument("NULL argument");
    if (mode < SB_SURFACE_ALL || mode > SB_SURFACE_INSIDE) throw std::invalid_argument("surface mode");
    sbh::Mesh m;
    if ((n_vertices && !vertices) || (n_triangles && !triangles)) throw std::invalid_argument("mesh arrays are NULL");
    m.v.resize(n_vertices);
    m.t.resize(n_triangles);
    for (uint32_t k = 0; k < n_vertices; ++k) m.v[k] = {vertices[3 * k], vertices[3 * k + 1], vertices[3 * k + 2]};
    for (uint32_t k = 0; k < n_triangles; ++k) {
      m.t[k] = {triangles[3 * k], triangles[3 * k + 1], triangles[3 * k + 2]};
      for (int c = 0; c < 3; ++c)
        if (m.t[k][c] >= n_vertices) throw std::out_of_range("triangle vertex index");
    }
    std::vector<sbh::Surface> all = sbh::extract_all_support_surfaces(m);
    uint32_t k = 0;
    for (const sbh::Surface& sf : all) {  // extract_support_surfaces (surface.cpp:145-153)
      if (mode != SB_SURFACE_ALL && (mode == SB_SURFACE_INSIDE) != sf.roofed) continue;
      if (k < cap) {
        sb_surface& o = out[k];
        std::memset(&o, 0, sizeof o);
        o.frame[0] = o.frame[5] = o.frame[10] = o.frame[15] = 1.0;
        o.frame[14] = sf.z_top;
        o.area = sf.area;
        o.roofed = sf.roofed ? 1 : 0;
        if (sf.polygon.size() > SB_MAX_SURFACE_VERTS)
          throw std::invalid_argument("support surface polygon exceeds SB_MAX_SURFACE_VERTS");
        o.n_polygon = static_cast<uint32_t>(sf.polygon.size());
        for (size_t v = 0; v < sf.polygon.size(); ++v) {
          o.polygon_xy[2 * v] = sf.polygon[v][0];
          o.polygon_xy[2 * v + 1] = sf.polygon[v][1];
        }
      }
      ++k;
    }
    *n_out = k;
  });
}

// Host restatement of region_for(0) (relationships.cpp:161-230, the serial path of
// k_relation_regions with glibc as libm) + n PolygonSampler draws from
// Pcg32(make_stream(seed, c)); test hook for the region pipeline on CPU.
sb_status sb_region_draws_host(const sb_relation* rel, const sb_support* sup,
                               const double* states, double erode_r, uint64_t seed,
                               const uint64_t* c, uint32_t nc, double* out_xy, uint32_t n,
                               int32_t* n_tris) {
  return guard([&] {
    if (!rel || !sup || !n_tris || (n && !out_xy)) throw std::invalid_argument("NULL argument");
    SbPlacementDev pd;
    std::memset(&pd, 0, sizeof pd);
    const std::vector<std::array<double, 2>> given = support_to_dev(*sup, pd);
    relation_to_dev(*rel, pd);
    const int na = pd.n_anchors;
    if (na > 0 && !states) throw std::invalid_argument("anchor states are NULL");
    std::vector<SbRegionTri> tris(sbp::kHoleCap);
    std::vector<double> cum(sbp::kHoleCap);
    sbp::TableSink sink{tris.data(), cum.data(), 0, sbp::kHoleCap, 0.0};
    const sbp::SupportClip clip{pd.rect, pd.poly_n, pd.poly_x, pd.poly_y};
    int st = sbp::kRegionOk;
    if (na == 0) {  // region = the support as given (+ erode of its corrected ring)
      std::vector<sbh::V2> ring;
      for (const auto& v : given) ring.push_back({v[0], v[1]});
      if (erode_r > 0.0) {
        double a = 0.0;
        for (size_t i = 0; i < ring.size(); ++i)
          a += ring[i][0] * ring[(i + 1) % ring.size()][1] - ring[(i + 1) % ring.size()][0] * ring[i][1];
        if (0.5 * a < 0.0) std::reverse(ring.begin() + 1, ring.end());
        ring = sbh::erode_convex(ring, erode_r);
      }
      sbh::SamplerTable t = sbh::sampler_table({ring});
      sink.n = static_cast<int>(t.tris.size());
      for (int k = 0; k < sink.n; ++k) {
        tris[k] = t.tris[k];
        cum[k] = t.cum[k];
      }
    } else if (pd.distance_type == SB_DIST_MIDDLE) {
      double mx[SB_MAX_ANCHORS], my[SB_MAX_ANCHORS];
      for (int k = 0; k < na; ++k) {
        mx[k] = states[3 * k];
        my[k] = states[3 * k + 1];
      }
      sbp::Ring r, tmp;
      st = sbp::middle_region_table<sbp::HostMath>(mx, my, na, clip, erode_r, r, tmp, sink);
      if (st == sbp::kRegionOk) sbp::finish_table(sink);
    } else {
      const double ax = states[0], ay = states[1], ayaw = states[2];
      double min_r = 0.0, max_r = HUGE_VAL;  // distance_band (relationships.cpp:101-122)
      if (pd.distance_type == SB_DIST_GREATER) min_r = pd.distance;
      if (pd.distance_type == SB_DIST_LESS) max_r = pd.distance;
      if (pd.distance_type == SB_DIST_EQUAL) {
        const double half = std::max(0.05 * pd.distance, 0.01);
        min_r = std::max(0.0, pd.distance - half);
        max_r = pd.distance + half;
      }
      const double theta = pd.angle_threshold > 0 ? pd.angle_threshold : (pd.direction == SB_DIR_NONE ? M_PI : M_PI / 4.0);
      double vx = 1.0, vy = 0.0;  // resolve_direction (relationships.cpp:78-99)
      switch (pd.direction) {
        case SB_DIR_LEFT: vx = -1.0; vy = 0.0; break;
        case SB_DIR_RIGHT: vx = 1.0; vy = 0.0; break;
        case SB_DIR_FRONT: vx = 0.0; vy = -1.0; break;
        case SB_DIR_BACK: vx = 0.0; vy = 1.0; break;
        case SB_DIR_VECTOR: {
          const double nrm = std::sqrt(pd.direction_vector[0] * pd.direction_vector[0] +
                                       pd.direction_vector[1] * pd.direction_vector[1]);
          vx = pd.direction_vector[0] / nrm;
          vy = pd.direction_vector[1] / nrm;
          break;
        }
        default: break;
      }
      if (pd.direction != SB_DIR_NONE && pd.frame == SB_FRAME_LOCAL) {
        const double cs = std::cos(ayaw), sn = std::sin(ayaw);
        const double rx = cs * vx - sn * vy, ry = sn * vx + cs * vy;
        vx = rx;
        vy = ry;
      }
      const double bx0 = std::min(pd.bounds[0], ax), by0 = std::min(pd.bounds[1], ay);
      const double bx1 = std::max(pd.bounds[2], ax), by1 = std::max(pd.bounds[3], ay);
      const double ddx = bx1 - bx0, ddy = by1 - by0;
      const double diag = bx0 > bx1 ? 0.0 : std::sqrt(ddx * ddx + ddy * ddy);
      if (std::isinf(max_r)) max_r = std::fmax(diag, min_r + 1e-6);
      sbp::HoleScratch sc;
      if (theta >= M_PI - 1e-12 && min_r > 0.0)
        st = sbp::hole_annulus_table<sbp::HostMath>(ax, ay, min_r, max_r, clip, erode_r, sc, sink);
      else
        st = sbp::big_region_table<sbp::HostMath>(ax, ay, vx, vy, theta, min_r, max_r, clip, erode_r, sc, sink);
      if (st == sbp::kRegionOk) sbp::finish_table(sink);
    }
    if (st != sbp::kRegionOk && st != sbp::kRegionEmpty)
      throw std::invalid_argument("region build failed (status " + std::to_string(st) + ")");
    const int nt = st == sbp::kRegionOk ? sink.n : 0;
    *n_tris = nt;
    if (nt == 0 || n == 0) return;
    std::vector<double> d(3 * static_cast<size_t>(n));
    if (sb_stream_doubles(seed, c, nc, d.data(), 3 * n) != SB_OK) throw std::runtime_error(g_error);
    for (uint32_t k = 0; k < n; ++k)
      sbp::draw_point(tris.data(), cum.data(), nt, d[3 * k], d[3 * k + 1], d[3 * k + 2],
                      out_xy[2 * k], out_xy[2 * k + 1]);
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
sb_status sb_engine_place(sb_engine* e, uint64_t run_seed, uint32_t first, uint32_t count,
                          sb_result* out, sb_run_stats* st) {
  return guard([&] {
    e->generate_range(run_seed, first, static_cast<size_t>(first) + count, st, out);
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

sb_status sb_host_math(int fn, const double* in, uint64_t n, double* out) {
  return guard([&] {
    if (fn < 0 || fn > 4) throw std::invalid_argument("sb_host_math: fn must be in [0, 4]");
    if (n && (!in || !out)) throw std::invalid_argument("NULL argument");
    for (uint64_t i = 0; i < n; ++i) {
      double s, c;
      switch (fn) {
        case 2: out[i] = sbg::atan2(in[2 * i], in[2 * i + 1]); break;
        case 3: out[i] = sbg::sin(in[i]); break;
        case 4: out[i] = sbg::cos(in[i]); break;
        default: sbg::sincos(in[i], &s, &c); out[i] = fn == 0 ? s : c;
      }
    }
  });
}

sb_status sb_device_math(int fn, const double* in, uint64_t n, double* out) {
  return guard([&] {
    if (fn < 0 || fn > 4) throw std::invalid_argument("sb_device_math: fn must be in [0, 4]");
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

extern "C" sb_status sb_engine_write_back(sb_engine* e, uint32_t placement, sb_graph* g, uint32_t node) {
  return guard([&] { e->write_back(placement, *g, node); });
}

extern "C" sb_status sb_engine_set_reach_filter(sb_engine* e, uint32_t placement,
                                                const sb_reach_map* m, const double* base16) {
  return guard([&] {
    if (placement >= e->places.size()) throw std::out_of_range("placement index out of range");
    e->reach.resize(e->places.size());
    ++e->graph_gen;  // the captured launches carry the filter parameters
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

