// sm_100a kernels for the Sceniris hot path. Build: -gencode arch=compute_100a,code=sm_100a
// -fmad=false (see sb_dev.cuh for why every FP64 op must round exactly once).
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "sb_dev.cuh"
#include "sb_kernels.h"
#include "sb_poly.h"
#include "sb_warp.cuh"

#include "../../include/scenebatch_b200.h"

using namespace sbd;

namespace {

constexpr int kBlock = 128;

inline unsigned grid_for(uint64_t n, int block = kBlock) {
  return static_cast<unsigned>((n + block - 1) / block);
}

inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Warp-aggregated counter update (all lanes of the warp must call it).
__device__ __forceinline__ void warp_add(unsigned long long* dst, unsigned v) {
  unsigned s = __reduce_add_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(dst, static_cast<unsigned long long>(s));
}

__device__ __forceinline__ void identity34(M34& P) {
#pragma unroll
  for (int k = 0; k < 12; ++k) P.m[k] = 0.0;
  P.m[0] = P.m[5] = P.m[10] = 1.0;
}

__device__ __forceinline__ void store_local_box(const WorldView& w, int32_t obj, uint64_t i) {
  const SbGeom g = w.geoms[w.obj_geom[obj]];
  double2* bp = reinterpret_cast<double2*>(w.box + ((uint64_t)obj * w.n + i) * 6);
  bp[0] = make_double2(g.box_min[0], g.box_min[1]);
  bp[1] = make_double2(g.box_min[2], g.box_max[0]);
  bp[2] = make_double2(g.box_max[1], g.box_max[2]);
}

// add_object (collision.cpp:365-376): identity pose, local box, disabled.
__global__ void k_init_object(WorldView w, int32_t obj) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= w.n) return;
  M34 P;
  identity34(P);
  double2* pp = reinterpret_cast<double2*>(w.pose + ((uint64_t)obj * w.n + i) * 12);
#pragma unroll
  for (int k = 0; k < 6; ++k) pp[k] = make_double2(P.m[2 * k], P.m[2 * k + 1]);
  store_local_box(w, obj, i);
  w.enabled[(uint64_t)(obj >> 5) * w.n + i] &= ~(1u << (obj & 31));
}

__global__ void k_set_enabled_list(WorldView w, int32_t obj, const uint32_t* inst, uint64_t n,
                                   int enabled) {
  uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  uint32_t* word = w.enabled + (uint64_t)(obj >> 5) * w.n + inst[j];
  uint32_t bit = 1u << (obj & 31);
  if (enabled) atomicOr(word, bit);
  else atomicAnd(word, ~bit);
}

__global__ void k_set_enabled_all(WorldView w, int32_t obj, int enabled) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= w.n) return;
  uint32_t* word = w.enabled + (uint64_t)(obj >> 5) * w.n + i;
  uint32_t bit = 1u << (obj & 31);
  *word = enabled ? (*word | bit) : (*word & ~bit);
}

__global__ void k_update_transforms(WorldView w, int32_t obj, const double* poses16,
                                    const uint32_t* inst, uint64_t n, uint64_t stride) {
  uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  M34 P;
  from_colmajor(poses16 + stride * j, P);
  store_pose(w, obj, inst ? inst[j] : j, P);
}

__global__ void __launch_bounds__(kBlock) k_check_batch(WorldView w, int32_t geom,
                                                        const double* poses16,
                                                        const uint32_t* active, uint64_t m,
                                                        uint8_t* free_out, int32_t* contact_out,
                                                        unsigned long long* counters) {
  __shared__ WarpScratch ws[kBlock / 32];
  __shared__ double invs[kBlock / 32][32][12];
  __shared__ GeomCache gc;
  const SbGeom gA = w.geoms[geom];
  load_geom_cache(w, gA, gc);
  __syncthreads();
  uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  CheckCounters cnt{0, 0, 0, 0};
  const bool act = j < m;
  uint32_t inst = act ? active[j] : 0u;
  M34 P;
  if (act) from_colmajor(poses16 + 16 * j, P);
  int hit = warp_check(w, gA, gc, act, P, inst, ws[threadIdx.x >> 5], invs[threadIdx.x >> 5], cnt);
  if (act && hit >= 0) {
    free_out[inst] = 0;
    contact_out[inst] = hit;
  }
  warp_add(counters + 1, cnt.narrow);
  warp_add(counters + 2, cnt.pairs);
  warp_add(counters + 4, cnt.broad);
  warp_add(counters + 5, cnt.nodes);
}

// ------------------------------------------------------------------ engine kernels
__global__ void k_engine_reset(WorldView w, int32_t first_obj, int32_t n_obj, uint8_t* valid,
                               int16_t* accepted, int32_t n_place) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= w.n) return;
  M34 P;
  identity34(P);
  for (int32_t o = first_obj; o < first_obj + n_obj; ++o) {
    double2* pp = reinterpret_cast<double2*>(w.pose + ((uint64_t)o * w.n + i) * 12);
#pragma unroll
    for (int k = 0; k < 6; ++k) pp[k] = make_double2(P.m[2 * k], P.m[2 * k + 1]);
    store_local_box(w, o, i);
  }
  for (int32_t wd = 0; wd < w.n_words; ++wd) {
    uint32_t clear = 0u;
    for (int32_t o = first_obj; o < first_obj + n_obj; ++o)
      if ((o >> 5) == wd) clear |= 1u << (o & 31);
    if (clear) w.enabled[(uint64_t)wd * w.n + i] &= ~clear;
  }
  valid[i] = 1;
  for (int32_t p = 0; p < n_place; ++p) accepted[(uint64_t)p * w.n + i] = -1;
}

// Fused PositionSampler::sample (sampler.cpp:70-127) + sample_orientations
// (sampler.cpp:129-156) + pose compose (Appendix C.3) + check_batch (collision.cpp:433-449)
// + accept (update_transform / set_enabled) for one (placement, attempt) round.
// One thread per active slot; slot j of this rank draws fast-path point draw_base + j.
__global__ void __launch_bounds__(kBlock) k_round(sbk::RoundParams p) {
  __shared__ WarpScratch ws[kBlock / 32];
  __shared__ double invs[kBlock / 32][32][12];
  __shared__ GeomCache gc;
  const SbPlacementDev& pl = p.pl;
  const SbGeom gA = p.w.geoms[pl.geom];
  load_geom_cache(p.w, gA, gc);
  __syncthreads();
  const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  CheckCounters cnt{0, 0, 0, 0};
  unsigned checked = 0, sampled = 0, accepted_now = 0;
  const bool act = j < p.m;
  const uint32_t inst = act ? p.act[j] : 0u;
  const uint64_t gid = p.global_begin + inst;
  bool placeable = act;
  M34 pose;
  if (act) {
    double lx = 0.0, ly = 0.0;
    if (p.fast) {
      Pcg r{p.fast_state0};
      r.advance(6ull * (p.draw_base + j));
      double u = r.next_double(), r1 = r.next_double(), r2 = r.next_double();
      sbp::draw_point(p.canon_tris, p.canon_cum, p.canon_n, u, r1, r2, lx, ly);
    } else {
      const int nt = p.inst_n[inst];
      if (nt == 0) {
        placeable = false;
      } else {
        Pcg r = Pcg::seeded(stream_seed4(p.run_seed, pl.salt, kFallbackSalt, gid,
                                         static_cast<uint64_t>(p.attempt)));
        double u = r.next_double(), r1 = r.next_double(), r2 = r.next_double();
        const uint64_t off = (uint64_t)inst * p.inst_cap;
        sbp::draw_point(p.inst_tris + off, p.inst_cum + off, nt, u, r1, r2, lx, ly);
      }
    }
    sampled = 1;
    if (placeable) {
      M34 S;
#pragma unroll
      for (int k = 0; k < 12; ++k) S.m[k] = pl.support[k];
      double px, py, pz;
      xform(S, lx, ly, 0.0, px, py, pz);
      double yaw = 0.0;
      if (pl.orientation == SB_ORIENT_UNIFORM_YAW) {
        Pcg r = Pcg::seeded(
            stream_seed4(p.run_seed, pl.salt, kYawSalt, gid, static_cast<uint64_t>(p.attempt)));
        const double two_pi = 2.0 * 3.14159265358979323846;
        yaw = 0.0 + (two_pi - 0.0) * r.next_double();  // Pcg32::uniform (rng.hpp:50)
      } else if (pl.orientation == SB_ORIENT_FACE_TO) {
        const double* tp = p.w.pose + ((uint64_t)pl.face_object * p.w.n + inst) * 12;
        double dx = tp[3] - px, dy = tp[7] - py;  // face_to_yaw (relationships.cpp:232-239)
        yaw = sqrt(dx * dx + dy * dy) < 1e-12 ? 0.0 : atan2(dy, dx);
      }
      double c = cos(yaw), s = sin(yaw);
      // translation(p + z_off z) * rotation_z(yaw)  (transform.hpp:40-54)
      M34 T, Rz;
      identity34(T);
      T.m[3] = px + 0.0;
      T.m[7] = py + 0.0;
      T.m[11] = pz + pl.z_off;
      identity34(Rz);
      Rz.m[0] = c;
      Rz.m[1] = -s;
      Rz.m[4] = s;
      Rz.m[5] = c;
      mul34(T, Rz, pose);
      checked = 1;
    }
  }
  const bool chk = checked != 0;
  const int hit = warp_check(p.w, gA, gc, chk, pose, inst, ws[threadIdx.x >> 5], invs[threadIdx.x >> 5], cnt);
  if (act) {
    bool ok = chk && hit < 0;
    if (ok) {
      store_pose(p.w, pl.object, inst, pose);
      p.w.enabled[(uint64_t)(pl.object >> 5) * p.w.n + inst] |= 1u << (pl.object & 31);
      p.accepted[inst] = static_cast<int16_t>(p.attempt);
      accepted_now = 1;
    }
    p.fail[j] = ok ? 0 : 1;
  }
  warp_add(p.counters + 0, checked);
  warp_add(p.counters + 1, cnt.narrow);
  warp_add(p.counters + 2, cnt.pairs);
  warp_add(p.counters + 3, sampled);
  warp_add(p.counters + 4, cnt.broad);
  warp_add(p.counters + 5, cnt.nodes);
  warp_add(p.counters + 6, accepted_now);
}

__global__ void k_invalidate(const uint32_t* act, uint64_t m, uint8_t* valid) {
  uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j < m) valid[act[j]] = 0;
}

// AnchorState in the support frame: inverse_rigid(support) * anchor pose; position is the
// translation, yaw = yaw_of (transform.hpp:77).
__global__ void k_anchor_states(WorldView w, int32_t anchor_obj, M34 inv_support, double* out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= w.n) return;
  const double* pp = w.pose + ((uint64_t)anchor_obj * w.n + i) * 12;
  M34 P, rel;
#pragma unroll
  for (int k = 0; k < 12; ++k) P.m[k] = pp[k];
  mul34(inv_support, P, rel);
  out[3 * i + 0] = rel.m[3];
  out[3 * i + 1] = rel.m[7];
  out[3 * i + 2] = atan2(rel.m[4], rel.m[0]);
}

// build_constraint_region's variation test (relationships.cpp:178-186).
__global__ void k_vary_flag(const double* st, uint64_t n, double x0, double y0, double yaw0,
                            int32_t* flag) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  bool vary = false;
  if (i < n) {
    double dx = st[3 * i] - x0, dy = st[3 * i + 1] - y0;
    vary = sqrt(dx * dx + dy * dy) > 1e-12 || fabs(st[3 * i + 2] - yaw0) > 1e-12;
  }
  if (__any_sync(0xffffffffu, vary) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// region_for(i) (relationships.cpp:188-205) + PolygonSampler ctor, one thread per instance.
__global__ void __launch_bounds__(64) k_build_regions(sbk::RegionParams p) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= p.count) return;
  const SbPlacementDev& pl = p.pl;
  const double ax = p.anchors[3 * i], ay = p.anchors[3 * i + 1], ayaw = p.anchors[3 * i + 2];
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double min_r = 0.0, max_r = inf;  // distance_band (relationships.cpp:101-122)
  if (pl.distance_type == SB_DIST_GREATER) {
    min_r = pl.distance;
    max_r = inf;
  } else if (pl.distance_type == SB_DIST_LESS) {
    min_r = 0.0;
    max_r = pl.distance;
  } else if (pl.distance_type == SB_DIST_EQUAL) {
    double half = dmax(0.05 * pl.distance, 0.01);
    min_r = dmax(0.0, pl.distance - half);
    max_r = pl.distance + half;
  }
  const double pi = 3.14159265358979323846;
  double theta = pl.angle_threshold > 0.0 ? pl.angle_threshold
                                          : (pl.direction == SB_DIR_NONE ? pi : pi / 4.0);
  double vx = 1.0, vy = 0.0;  // resolve_direction (relationships.cpp:78-99)
  if (pl.direction != SB_DIR_NONE) {
    switch (pl.direction) {
      case SB_DIR_LEFT: vx = -1; vy = 0; break;
      case SB_DIR_RIGHT: vx = 1; vy = 0; break;
      case SB_DIR_FRONT: vx = 0; vy = -1; break;
      case SB_DIR_BACK: vx = 0; vy = 1; break;
      default: {
        double nrm = sqrt(pl.direction_vector[0] * pl.direction_vector[0] +
                          pl.direction_vector[1] * pl.direction_vector[1]);
        vx = pl.direction_vector[0] / nrm;
        vy = pl.direction_vector[1] / nrm;
      }
    }
    if (pl.frame == SB_FRAME_LOCAL) {
      double c = cos(ayaw), s = sin(ayaw);
      double nx = c * vx - s * vy, ny = s * vx + c * vy;
      vx = nx;
      vy = ny;
    }
  }
  // clip bound = bounds(support) expanded by the anchor (relationships.cpp:190-193)
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
  double ddx = bx1 - bx0, ddy = by1 - by0;
  double diag = bx0 > bx1 ? 0.0 : sqrt(ddx * ddx + ddy * ddy);

  sbp::Ring ring, tmp;
  int st = sbp::annulus_sector(ax, ay, vx, vy, theta, min_r, max_r, diag, ring);
  if (st == sbp::kRegionOk) st = sbp::intersect_rect(ring, tmp, pl.rect);
  int n = 0;
  if (st == sbp::kRegionOk) {
    sbp::TableSink sink{p.tris + i * p.cap, p.cum + i * p.cap, 0, p.cap, 0.0};
    if (!sbp::ear_clip_into(ring, sink)) st = sbp::kRegionOverflow;
    else n = sbp::finish_table(sink);
  }
  if (st == sbp::kRegionEmpty) st = sbp::kRegionOk;
  if (st != sbp::kRegionOk) {
    atomicMax(p.status, st);
    n = 0;
  }
  p.ntri[i] = n;
}

__global__ void k_pose_colmajor(WorldView w, int32_t obj, double* out16) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= w.n) return;
  const double* pp = w.pose + ((uint64_t)obj * w.n + i) * 12;
  double* o = out16 + 16 * i;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) o[4 * c + r] = pp[4 * r + c];
  o[3] = o[7] = o[11] = 0.0;
  o[15] = 1.0;
}

}  // namespace

namespace sbk {

void init_object(const SbWorldView& w, int32_t obj, sb_stream_t s) {
  k_init_object<<<grid_for(w.n), kBlock, 0, s>>>(w, obj);
  check_launch("init_object");
}
void set_enabled_list(const SbWorldView& w, int32_t obj, const uint32_t* inst, uint64_t n,
                      int enabled, sb_stream_t s) {
  if (n == 0) return;
  k_set_enabled_list<<<grid_for(n), kBlock, 0, s>>>(w, obj, inst, n, enabled);
  check_launch("set_enabled");
}
void set_enabled_all(const SbWorldView& w, int32_t obj, int enabled, sb_stream_t s) {
  k_set_enabled_all<<<grid_for(w.n), kBlock, 0, s>>>(w, obj, enabled);
  check_launch("set_enabled_all");
}
void update_transforms(const SbWorldView& w, int32_t obj, const double* poses16,
                       const uint32_t* inst, uint64_t n, uint64_t stride, sb_stream_t s) {
  if (n == 0) return;
  k_update_transforms<<<grid_for(n), kBlock, 0, s>>>(w, obj, poses16, inst, n, stride);
  check_launch("update_transforms");
}
void check_batch(const SbWorldView& w, int32_t geom, const double* poses16,
                 const uint32_t* active, uint64_t m, uint8_t* free_out, int32_t* contact_out,
                 unsigned long long* counters, sb_stream_t s) {
  if (m == 0) return;
  k_check_batch<<<grid_for(m), kBlock, 0, s>>>(w, geom, poses16, active, m, free_out,
                                                contact_out, counters);
  check_launch("check_batch");
}
void engine_reset(const SbWorldView& w, int32_t first_obj, int32_t n_obj, uint8_t* valid,
                  int16_t* accepted, int32_t n_place, sb_stream_t s) {
  k_engine_reset<<<grid_for(w.n), kBlock, 0, s>>>(w, first_obj, n_obj, valid, accepted, n_place);
  check_launch("engine_reset");
}
size_t select_temp_bytes(uint64_t n) {
  size_t a = 0, b = 0;
  cub::CountingInputIterator<uint32_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, a, it, (const uint8_t*)nullptr, (uint32_t*)nullptr,
                             (uint64_t*)nullptr, static_cast<int64_t>(n));
  cub::DeviceSelect::Flagged(nullptr, b, (const uint32_t*)nullptr, (const uint8_t*)nullptr,
                             (uint32_t*)nullptr, (uint64_t*)nullptr, static_cast<int64_t>(n));
  return a > b ? a : b;
}
void select_valid(const uint8_t* valid, uint64_t n, uint32_t* out, uint64_t* d_count, void* temp,
                  size_t temp_bytes, sb_stream_t s) {
  cub::CountingInputIterator<uint32_t> it(0);
  cudaError_t e = cub::DeviceSelect::Flagged(temp, temp_bytes, it, valid, out, d_count,
                                             static_cast<int64_t>(n), s);
  if (e != cudaSuccess) throw std::runtime_error(std::string("select_valid: ") + cudaGetErrorString(e));
}
void select_flagged(const uint32_t* in, const uint8_t* flags, uint64_t m, uint32_t* out,
                    uint64_t* d_count, void* temp, size_t temp_bytes, sb_stream_t s) {
  cudaError_t e = cub::DeviceSelect::Flagged(temp, temp_bytes, in, flags, out, d_count,
                                             static_cast<int64_t>(m), s);
  if (e != cudaSuccess) throw std::runtime_error(std::string("select_flagged: ") + cudaGetErrorString(e));
}
void round_kernel(const RoundParams& p, sb_stream_t s) {
  if (p.m == 0) return;
  k_round<<<grid_for(p.m), kBlock, 0, s>>>(p);
  check_launch("round");
}
void invalidate(const uint32_t* act, uint64_t m, uint8_t* valid, sb_stream_t s) {
  if (m == 0) return;
  k_invalidate<<<grid_for(m), kBlock, 0, s>>>(act, m, valid);
  check_launch("invalidate");
}
void anchor_states(const SbWorldView& w, int32_t anchor_obj, const double inv_support[12],
                   double* out, sb_stream_t s) {
  M34 inv;
  for (int k = 0; k < 12; ++k) inv.m[k] = inv_support[k];
  k_anchor_states<<<grid_for(w.n), kBlock, 0, s>>>(w, anchor_obj, inv, out);
  check_launch("anchor_states");
}
void vary_flag(const double* states, uint64_t n, double x0, double y0, double yaw0,
               int32_t* flag, sb_stream_t s) {
  k_vary_flag<<<grid_for(n), kBlock, 0, s>>>(states, n, x0, y0, yaw0, flag);
  check_launch("vary_flag");
}
void build_regions(const RegionParams& p, sb_stream_t s) {
  if (p.count == 0) return;
  k_build_regions<<<grid_for(p.count, 64), 64, 0, s>>>(p);
  check_launch("build_regions");
}
void download_poses(const SbWorldView& w, int32_t obj, double* out16, sb_stream_t s) {
  k_pose_colmajor<<<grid_for(w.n), kBlock, 0, s>>>(w, obj, out16);
  check_launch("download_poses");
}

}  // namespace sbk
