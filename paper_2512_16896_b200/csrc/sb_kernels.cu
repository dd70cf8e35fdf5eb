// sm_100a kernels for CollisionWorld maintenance, the world-API check_batch and engine
// bookkeeping. Build: -gencode arch=compute_100a,code=sm_100a -fmad=false (see sb_dev.cuh
// for why every FP64 op must round exactly once).
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "../../include/scenebatch_b200.h"
#include "sb_crmath.cuh"
#include "sb_glibcm.cuh"
#include "sb_dev.cuh"
#include "sb_kernels.h"
#include "sb_poly.h"
#include "sb_warp.cuh"

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

__device__ __forceinline__ void store_identity(const WorldView& w, int32_t obj, uint64_t i) {
  M34 P;
  identity34(P);
  double2* pp = reinterpret_cast<double2*>(w.pose + sb_pose_off(w, obj, i));
#pragma unroll
  for (int k = 0; k < 6; ++k) pp[k] = make_double2(P.m[2 * k], P.m[2 * k + 1]);
}

__device__ __forceinline__ void store_local_box(const WorldView& w, int32_t obj, uint64_t i) {
  const SbGeom g = w.geoms[w.obj_geom[obj]];
  double2* bp = reinterpret_cast<double2*>(w.box + sb_box_off(w, obj, i));
  bp[0] = make_double2(g.box_min[0], g.box_min[1]);
  bp[1] = make_double2(g.box_min[2], g.box_max[0]);
  bp[2] = make_double2(g.box_max[1], g.box_max[2]);
}

// add_object (collision.cpp:365-376): identity pose, local box, disabled.
__global__ void k_init_object(WorldView w, int32_t obj) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= w.n) return;
  store_identity(w, obj, i);
  store_local_box(w, obj, i);
  w.enabled[sb_word_off(w, obj >> 5, i)] &= ~(1u << (obj & 31));
}

// set_enabled (collision.cpp:386-389); atomics because `instances` may repeat.
__global__ void k_set_enabled_list(WorldView w, int32_t obj, const uint32_t* inst, uint64_t n,
                                   int enabled) {
  uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  uint32_t* word = w.enabled + sb_word_off(w, obj >> 5, inst[j]);
  uint32_t bit = 1u << (obj & 31);
  if (enabled) atomicOr(word, bit);
  else atomicAnd(word, ~bit);
}

__global__ void k_set_enabled_all(WorldView w, int32_t obj, int enabled) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= w.n) return;
  uint32_t* word = w.enabled + sb_word_off(w, obj >> 5, i);
  uint32_t bit = 1u << (obj & 31);
  *word = enabled ? (*word | bit) : (*word & ~bit);
}

// update_transform(s) (collision.cpp:395-412): pose record + world box.
__global__ void k_update_transforms(WorldView w, int32_t obj, const double* poses16,
                                    const uint32_t* inst, uint64_t n, uint64_t stride) {
  uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  M34 P;
  from_colmajor(poses16 + stride * j, P);
  store_pose(w, obj, inst ? inst[j] : j, P);
}

// check_batch (collision.cpp:418-461): lane per candidate, warp-pooled exact narrow phase.
__global__ void __launch_bounds__(kBlock) k_check_batch(WorldView w, int32_t geom,
                                                        const double* poses16,
                                                        const uint32_t* active, uint64_t m,
                                                        uint8_t* free_out, int32_t* contact_out,
                                                        unsigned long long* counters) {
  extern __shared__ __align__(16) unsigned char ws_dyn[];  // [kBlock / 32] WarpScratch
  __shared__ double invs[kBlock / 32][32][12];
  WarpScratch* ws = reinterpret_cast<WarpScratch*>(ws_dyn);
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

// generate() start: placement objects back to add_object state; valid = 1; accepted = -1.
// generate() start: placement objects leave the world (enable bits), every instance is
// valid, no attempt accepted. Poses / boxes of placement objects are left as they are:
// a disabled object is never read by the collision check, and k_unaccepted_fixup gives
// the objects a run leaves unaccepted the identity pose / local box at the end.
__global__ void k_engine_reset(WorldView w, int32_t first_obj, int32_t n_obj, uint8_t* valid,
                               int16_t* accepted, int32_t n_place) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= w.n) return;
  for (int32_t wd = 0; wd < w.n_words; ++wd) {
    uint32_t clear = 0u;
    for (int32_t o = first_obj; o < first_obj + n_obj; ++o)
      if ((o >> 5) == wd) clear |= 1u << (o & 31);
    if (clear) w.enabled[sb_word_off(w, wd, i)] &= ~clear;
  }
  valid[i] = 1;
  for (int32_t p = 0; p < n_place; ++p) accepted[(uint64_t)p * w.n + i] = -1;
}

// Per-instance support frames of a placement (sampler.hpp:78-80): S[i] = pose(obj, i) *
// frame when obj >= 0 (a surface of a placed object, Mat4 product in the shim's order),
// else S[i] as given; inv[i] = inverse_rigid(S[i]) (transform.hpp:63-69).
__global__ void k_support_frames(WorldView w, int32_t obj, M34 frame, double* S, double* inv) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= w.n) return;
  M34 F, I;
  if (obj >= 0) {
    const double* pp = w.pose + sb_pose_off(w, obj, i);
    M34 P;
#pragma unroll
    for (int k = 0; k < 12; ++k) P.m[k] = pp[k];
    mul34(P, frame, F);
#pragma unroll
    for (int k = 0; k < 12; ++k) S[i * 12 + k] = F.m[k];
  } else {
#pragma unroll
    for (int k = 0; k < 12; ++k) F.m[k] = S[i * 12 + k];
  }
  inverse_rigid(F, I);
#pragma unroll
  for (int k = 0; k < 12; ++k) inv[i * 12 + k] = I.m[k];
}

// generate() end: an object whose placement accepted nothing for instance i keeps the
// state add_object gave it (collision.cpp:365-376): identity pose, local box.
__global__ void k_unaccepted_fixup(WorldView w, int32_t first_obj, int32_t n_place,
                                   const int16_t* accepted) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= w.n) return;
  for (int32_t p = 0; p < n_place; ++p)
    if (accepted[(uint64_t)p * w.n + i] < 0) {
      store_identity(w, first_obj + p, i);
      store_local_box(w, first_obj + p, i);
    }
}

// Result poses of one placement (column-major Mat4): the identity where nothing was
// accepted (k_place writes the accepted ones at accept time).
__global__ void k_out16_fixup(uint64_t n, const int16_t* accepted, double* out16) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n || accepted[i] >= 0) return;
  double2* o = reinterpret_cast<double2*>(out16 + i * 16);
#pragma unroll
  for (int k = 0; k < 8; ++k)
    o[k] = make_double2((2 * k) % 5 == 0 ? 1.0 : 0.0, (2 * k + 1) % 5 == 0 ? 1.0 : 0.0);
}

// Occupancy grid at generate() start: cells cleared, then the enabled fixed objects
// (ids < first_obj) inserted from their world boxes. Thread per instance.
// The occupancy grid of every instance written in one coalesced pass (replaces a memset
// of the grid + k_cells_insert_fixed): thread per (instance, cell); a cell's words are the
// bits of the enabled fixed objects (ids < first_obj) whose world box meets the cell, with
// cell_range's rounding. The fixed objects' boxes of an instance are read by the 32 lanes
// of its cells at once (broadcast loads).
__global__ void __launch_bounds__(256) k_cells_init(WorldView w, SbCellGrid G, int32_t first_obj) {
  const uint64_t cells = (uint64_t)G.g * G.g;
  const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (k >= w.n * cells) return;
  const uint64_t i = k / cells;
  const int c = (int)(k - i * cells), cy = c / G.g, cx = c - cy * G.g;
  uint32_t word[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // G.words <= 8 (256 objects)
  for (int32_t o = 0; o < first_obj; ++o) {
    if (!((__ldg(w.enabled + sb_word_off(w, o >> 5, i)) >> (o & 31)) & 1u)) continue;
    const double* b = w.box + sb_box_off(w, o, i);
    double mn[3] = {__ldg(b), __ldg(b + 1), __ldg(b + 2)}, mx[3] = {__ldg(b + 3), __ldg(b + 4), __ldg(b + 5)};
    int cx0, cx1, cy0, cy1;
    cell_range(G, mn, mx, cx0, cx1, cy0, cy1);
    if (cx >= cx0 && cx <= cx1 && cy >= cy0 && cy <= cy1) {
#pragma unroll
      for (int wd = 0; wd < 8; ++wd)
        if ((o >> 5) == wd) word[wd] |= 1u << (o & 31);
    }
  }
  uint32_t* out = G.cells + k * G.words;
  if (G.words == 4) {
    *reinterpret_cast<uint4*>(out) = make_uint4(word[0], word[1], word[2], word[3]);
  } else {
#pragma unroll
    for (int wd = 0; wd < 8; ++wd)
      if (wd < G.words) out[wd] = word[wd];
  }
}

__global__ void k_cells_insert_fixed(WorldView w, SbCellGrid G, int32_t first_obj) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= w.n) return;
  for (int32_t o = 0; o < first_obj; ++o) {
    if (!((w.enabled[sb_word_off(w, o >> 5, i)] >> (o & 31)) & 1u)) continue;
    const double* b = w.box + sb_box_off(w, o, i);
    cell_insert(G, i, o, b, b + 3);
  }
}

// AnchorState in the support frame: inverse_rigid(support) * anchor pose; position is the
// translation, yaw = yaw_of (transform.hpp:77).
__global__ void k_anchor_states(WorldView w, int32_t anchor_obj, M34 inv_support,
                                const double* inv_inst, double* out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= w.n) return;
  const double* pp = w.pose + sb_pose_off(w, anchor_obj, i);
  M34 P, rel;
#pragma unroll
  for (int k = 0; k < 12; ++k) P.m[k] = pp[k];
  if (inv_inst) {  // per-instance support frames
#pragma unroll
    for (int k = 0; k < 12; ++k) inv_support.m[k] = inv_inst[i * 12 + k];
  }
  mul34(inv_support, P, rel);
  out[3 * i + 0] = rel.m[3];
  out[3 * i + 1] = rel.m[7];
  out[3 * i + 2] = sbg::atan2(rel.m[4], rel.m[0]);
}

__global__ void k_pose_colmajor(WorldView w, int32_t obj, double* out16) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= w.n) return;
  const double* pp = w.pose + sb_pose_off(w, obj, i);
  double* o = out16 + 16 * i;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) o[4 * c + r] = pp[4 * r + c];
  o[3] = o[7] = o[11] = 0.0;
  o[15] = 1.0;
}

// Test hook with the device functions the hot path uses (sb_glibcm.cuh): fn 0 / 1 = the
// sine / cosine of glibc's sincos (what the reference's merged std::sin + std::cos calls
// run), 2 = atan2(in[2i], in[2i+1]), 3 / 4 = glibc's sin / cos on their own.
__global__ void k_debug_math(int fn, const double* in, uint64_t n, double* out) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (fn == 2) {
    out[i] = sbg::atan2(in[2 * i], in[2 * i + 1]);
  } else if (fn == 3) {
    out[i] = sbg::sin(in[i]);
  } else if (fn == 4) {
    out[i] = sbg::cos(in[i]);
  } else {
    double s, c;
    sbg::sincos(in[i], &s, &c);
    out[i] = fn == 0 ? s : c;
  }
}

// ------------------------------------------------------------ standalone PositionSampler
// Fast path (sampler.cpp:78-97): the j-th active entry takes FIFO point j, which is draw
// number seg_draw[s] + (j - seg_first[s]) of the cache stream (the host keeps the queue as
// draw-index ranges, SampleCache semantics). Draw d = 6d PCG steps in (polygon.cpp:390-400).
// Support pose of active entry j: host-gathered row-major 3x4 (sup34), or column-major Mat4
// of instance active[j] read in place (device-resident API).
__device__ __forceinline__ void support_of(const double* sup34, const double* sup16,
                                           const uint32_t* active, uint64_t j, M34& S) {
  if (sup34) {
#pragma unroll
    for (int k = 0; k < 12; ++k) S.m[k] = __ldg(sup34 + 12 * j + k);
  } else {
    const double* c = sup16 + 16 * (uint64_t)__ldg(active + j);
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int k = 0; k < 4; ++k) S.m[4 * r + k] = __ldg(c + 4 * k + r);
  }
}

__global__ void k_sampler_fifo(const double* sup34, const double* sup16, const uint32_t* active,
                               uint64_t m, const uint64_t* seg_first,
                               const uint64_t* seg_draw, int nseg, uint64_t state0,
                               const SbRegionTri* tris, const double* cum, int nt, double* pos) {
  const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  int lo = 0, hi = nseg - 1;  // last segment with seg_first <= j
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(seg_first + mid) <= j) lo = mid;
    else hi = mid - 1;
  }
  Pcg r{state0};
  r.advance(6ull * (__ldg(seg_draw + lo) + (j - __ldg(seg_first + lo))));
  const double u = r.next_double(), r1 = r.next_double(), r2 = r.next_double();
  double lx, ly;
  sbp::draw_point(tris, cum, nt, u, r1, r2, lx, ly);
  M34 S;
  support_of(sup34, sup16, active, j, S);
  double px, py, pz;
  xform(S, lx, ly, 0.0, px, py, pz);  // transform_point(support_world[inst], (x, y, 0))
  pos[3 * j] = px;
  pos[3 * j + 1] = py;
  pos[3 * j + 2] = pz;
}

// Per-instance regions (sampler.cpp:101-126): one draw from instance inst's own table on
// make_stream(run_seed, {salt, "fall", inst, attempt}); an empty table -> not placeable.
__global__ void k_sampler_fallback(const double* sup34, const double* sup16,
                                   const uint32_t* active, uint64_t m,
                                   uint64_t run_seed, uint64_t salt, uint64_t attempt,
                                   const uint32_t* inst_tab, const int32_t* inst_n, int cap,
                                   const SbRegionTri* tris, const double* cum, double* pos,
                                   uint8_t* placeable) {
  const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  const uint32_t inst = __ldg(active + j);
  uint32_t o0, nt;
  if (inst_tab) {
    o0 = __ldg(inst_tab + 2 * inst);
    nt = __ldg(inst_tab + 2 * inst + 1);
  } else {  // relation tables, [n][cap] (k_relation_regions layout)
    o0 = inst * (uint32_t)cap;
    nt = (uint32_t)__ldg(inst_n + inst);
  }
  double px = 0.0, py = 0.0, pz = 0.0;
  if (nt > 0) {
    Pcg r = Pcg::seeded(stream_seed4(run_seed, salt, kFallbackSalt, inst, attempt));
    const double u = r.next_double(), r1 = r.next_double(), r2 = r.next_double();
    double lx, ly;
    sbp::draw_point(tris + o0, cum + o0, (int)nt, u, r1, r2, lx, ly);
    M34 S;
    support_of(sup34, sup16, active, j, S);
    xform(S, lx, ly, 0.0, px, py, pz);
  }
  pos[3 * j] = px;
  pos[3 * j + 1] = py;
  pos[3 * j + 2] = pz;
  placeable[j] = nt > 0 ? 1 : 0;
}

// sample_orientations (sampler.cpp:129-156): kind 1 = uniform_yaw on
// make_stream(run_seed, {salt, "yaw!", inst, attempt}); kind 2 = face_to_yaw
// (relationships.cpp:232-239) toward face_xy[inst] with the correctly rounded atan2.
__global__ void k_orientations(int kind, const uint32_t* active, uint64_t m, const double* pos,
                               const double* face_xy, uint64_t run_seed, uint64_t salt,
                               uint64_t attempt, double* yaws) {
  const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  const uint32_t inst = __ldg(active + j);
  double yaw = 0.0;
  if (kind == SB_ORIENT_UNIFORM_YAW) {
    Pcg r = Pcg::seeded(stream_seed4(run_seed, salt, kYawSalt, inst, attempt));
    const double two_pi = 2.0 * 3.14159265358979323846;
    yaw = 0.0 + (two_pi - 0.0) * r.next_double();
  } else if (kind == SB_ORIENT_FACE_TO) {
    const double dx = __ldg(face_xy + 2 * inst) - __ldg(pos + 3 * j);
    const double dy = __ldg(face_xy + 2 * inst + 1) - __ldg(pos + 3 * j + 1);
    yaw = sqrt(dx * dx + dy * dy) < 1e-12 ? 0.0 : sbg::atan2(dy, dx);
  }
  yaws[j] = yaw;
}

}  // namespace

namespace sbk {

void debug_math(int fn, const double* in, uint64_t n, double* out, sb_stream_t s) {
  if (n == 0) return;
  k_debug_math<<<grid_for(n), kBlock, 0, s>>>(fn, in, n, out);
  check_launch("debug_math");
}

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
  const size_t smem = (kBlock / 32) * sizeof(WarpScratch);
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute((const void*)k_check_batch, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      throw std::runtime_error("check_batch: cudaFuncSetAttribute failed");
    attr = true;
  }
  k_check_batch<<<grid_for(m), kBlock, smem, s>>>(w, geom, poses16, active, m, free_out,
                                                  contact_out, counters);
  check_launch("check_batch");
}
void narrow_profile_check(unsigned long long out[8], bool reset) {
  if (cudaMemcpyFromSymbol(out, g_nprof, 8 * sizeof(unsigned long long)) != cudaSuccess)
    throw std::runtime_error("narrow_profile_check");
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (cudaMemcpyToSymbol(g_nprof, z, sizeof z) != cudaSuccess)
      throw std::runtime_error("narrow_profile_check reset");
  }
}
void engine_reset(const SbWorldView& w, int32_t first_obj, int32_t n_obj, uint8_t* valid,
                  int16_t* accepted, int32_t n_place, sb_stream_t s) {
  k_engine_reset<<<grid_for(w.n), kBlock, 0, s>>>(w, first_obj, n_obj, valid, accepted, n_place);
  check_launch("engine_reset");
}
void unaccepted_fixup(const SbWorldView& w, int32_t first_obj, int32_t n_place,
                      const int16_t* accepted, sb_stream_t s) {
  k_unaccepted_fixup<<<grid_for(w.n), kBlock, 0, s>>>(w, first_obj, n_place, accepted);
  check_launch("unaccepted_fixup");
}
void support_frames(const SbWorldView& w, int32_t obj, const double frame[12], double* S,
                    double* inv, sb_stream_t s) {
  M34 F;
  for (int k = 0; k < 12; ++k) F.m[k] = frame[k];
  k_support_frames<<<grid_for(w.n), kBlock, 0, s>>>(w, obj, F, S, inv);
  check_launch("support_frames");
}
void out16_fixup(uint64_t n, const int16_t* accepted, double* out16, sb_stream_t s) {
  k_out16_fixup<<<grid_for(n), kBlock, 0, s>>>(n, accepted, out16);
  check_launch("out16_fixup");
}
void cells_reset(const SbWorldView& w, const SbCellGrid& g, int32_t first_obj, sb_stream_t s) {
  if (g.words <= 8 && std::getenv("SB_CELLS_MEMSET") == nullptr) {
    const uint64_t total = w.n * (uint64_t)(g.g * g.g);
    k_cells_init<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(w, g, first_obj);
    check_launch("cells_init");
    return;
  }
  const cudaError_t e = cudaMemsetAsync(g.cells, 0, w.n * (uint64_t)(g.g * g.g) * g.words * sizeof(uint32_t),
                                        reinterpret_cast<cudaStream_t>(s));
  if (e != cudaSuccess) throw std::runtime_error(std::string("cells memset: ") + cudaGetErrorString(e));
  k_cells_insert_fixed<<<grid_for(w.n), kBlock, 0, s>>>(w, g, first_obj);
  check_launch("cells_reset");
}
void anchor_states(const SbWorldView& w, int32_t anchor_obj, const double inv_support[12],
                   const double* inv_inst, double* out, sb_stream_t s) {
  M34 inv;
  for (int k = 0; k < 12; ++k) inv.m[k] = inv_support[k];
  k_anchor_states<<<grid_for(w.n), kBlock, 0, s>>>(w, anchor_obj, inv, inv_inst, out);
  check_launch("anchor_states");
}
void download_poses(const SbWorldView& w, int32_t obj, double* out16, sb_stream_t s) {
  k_pose_colmajor<<<grid_for(w.n), kBlock, 0, s>>>(w, obj, out16);
  check_launch("download_poses");
}

void sampler_fifo(const double* sup34, const double* sup16, const uint32_t* active, uint64_t m,
                  const uint64_t* seg_first, const uint64_t* seg_draw, int nseg, uint64_t state0,
                  const SbRegionTri* tris, const double* cum, int nt, double* pos, sb_stream_t s) {
  if (m == 0) return;
  k_sampler_fifo<<<grid_for(m, 256), 256, 0, s>>>(sup34, sup16, active, m, seg_first, seg_draw,
                                                  nseg, state0, tris, cum, nt, pos);
  check_launch("sampler_fifo");
}
void sampler_fallback(const double* sup34, const double* sup16, const uint32_t* active,
                      uint64_t m, uint64_t run_seed,
                      uint64_t salt, uint64_t attempt, const uint32_t* inst_tab,
                      const int32_t* inst_n, int cap, const SbRegionTri* tris, const double* cum,
                      double* pos, uint8_t* placeable, sb_stream_t s) {
  if (m == 0) return;
  k_sampler_fallback<<<grid_for(m, 256), 256, 0, s>>>(sup34, sup16, active, m, run_seed, salt,
                                                      attempt,
                                                      inst_tab, inst_n, cap, tris, cum, pos,
                                                      placeable);
  check_launch("sampler_fallback");
}
void orientations(int kind, const uint32_t* active, uint64_t m, const double* pos,
                  const double* face_xy, uint64_t run_seed, uint64_t salt, uint64_t attempt,
                  double* yaws, sb_stream_t s) {
  if (m == 0) return;
  k_orientations<<<grid_for(m, 256), 256, 0, s>>>(kind, active, m, pos, face_xy, run_seed, salt,
                                                  attempt, yaws);
  check_launch("orientations");
}

}  // namespace sbk
