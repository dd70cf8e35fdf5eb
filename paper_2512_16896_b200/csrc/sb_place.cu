// Tiled placement engine (see sb_place.h). sm_100a, -fmad=false.
#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>

#include <climits>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "../../include/scenebatch_b200.h"
#include "sb_crmath.cuh"
#include "sb_glibcm.cuh"
#include "sb_dev.cuh"
#include "sb_pdl.cuh"
#include "sb_place.h"
#include "sb_reachdev.cuh"
#include "sb_poly.h"
#include "sb_warp.cuh"

#ifndef SB_WIDE_SAMPLE_MINB
#define SB_WIDE_SAMPLE_MINB 3  // CTAs per SM k_wide_sample's register budget is sized for
#endif
#ifndef SB_WIDE_NARROW_MINB
#define SB_WIDE_NARROW_MINB 3  // same for k_wide_narrow
#endif
#ifndef SB_PLACE_MIN_BLOCKS
#define SB_PLACE_MIN_BLOCKS (512 / SB_PLACE_BLOCK)  // CTAs per SM the register budget is sized for
#endif

namespace cg = cooperative_groups;
using namespace sbd;

namespace sbk {
namespace {

constexpr int kB = kPlaceBlock;
constexpr int kWarps = kB / 32;
constexpr int32_t kFree = INT32_MAX;
constexpr int kCand = 512;    // broad-phase items per chunk (grid mode)
constexpr int kQueue = 1024;  // narrow pairs (grid mode: <= one per item of a chunk)
constexpr uint8_t kSlotChecked = 1, kSlotUnplaceable = 2, kSlotEnumerated = 4;
constexpr int kGW = 8;  // enable words the broad phase keeps in registers (<= 256 objects)
constexpr int kPrefixItems = 8;  // tile counts per thread per prefix-scan chunk
constexpr uint64_t kSoloFlag = 1ull << 63;

enum Ctrl { kRounds = 2, kErr = 3, kTileCtr = 4 /* kTotal0 = 5, kTotal1 = 6 */ };

using BlockScan = cub::BlockScan<uint32_t, kB>;


// Per-round candidate state of the CTA's tile (dynamic shared memory).
struct Tile {
  double* box;       // [kB][6]  candidate world AABB per slot
  uint32_t* ovm;     // [words][kB] broad-phase overlap bits per slot
  uint32_t* enw;     // [words][kB] enable words per tile entry
  uint32_t* list;    // [kB] tile's active instances (ascending)
  uint32_t* queue;   // [kQueue] narrow pairs (slot << 24 | object)
  uint32_t* cand;    // [kCand] broad-phase items (slot << 24 | object)
  int32_t* contact;  // [kB] min colliding object per slot
  uint32_t* rem;     // [kB] queued, not yet tested pairs per slot
  int32_t* minfree;  // [kB] per tile entry: lowest slot (attempt offset) confirmed free, W = none
  uint8_t* sflag;    // [kB]
  unsigned char* ws; // [kWarps][ws_bytes]
  int4* ogeo;        // [n_objects] narrow-record descriptor of each object's geometry
};

struct Fixed {  // static shared memory
  PlaceGeomCache gc;
  typename BlockScan::TempStorage scan;
  uint32_t prefix[kPlaceMaxOwnedTiles];  // fast path: draw offset of each owned tile
  uint32_t cnt[kPlaceMaxOwnedTiles];     // fast path: its survivors entering this round
  uint32_t qn;
  uint32_t dq, dt;  // debug: pairs queued / tested this tile round
  uint32_t qhead;   // narrow-phase claim counter
  uint32_t total;
  uint32_t tile;
  int32_t used;     // rounds a tile round consumed (FIFO speculation, phase C)
  uint64_t seed;    // run seed (from p.seed_dev when set: graph-replayable launches)
  uint64_t state0;  // Pcg32(make_stream(seed, {salt, "cach"})) after its constructor
  unsigned long long tclk;  // block 0 / thread 0 phase clock
  unsigned long long acc[8];  // its per-slot sums, written to p.prof once at the end
  unsigned long long ta, tb, t0;  // every block: A1 / A2+B ns of the current round (debug)
};

__device__ __forceinline__ Tile carve(unsigned char* d, int words, int ws_bytes) {
  Tile t;
  t.box = reinterpret_cast<double*>(d);
  t.ovm = reinterpret_cast<uint32_t*>(t.box + 6 * kB);
  t.enw = t.ovm + words * kB;
  t.list = t.enw + words * kB;
  t.queue = t.list + kB;
  t.cand = t.queue + kQueue;
  t.contact = reinterpret_cast<int32_t*>(t.cand + kCand);
  t.rem = reinterpret_cast<uint32_t*>(t.contact + kB);
  t.minfree = reinterpret_cast<int32_t*>(t.rem + kB);
  t.sflag = reinterpret_cast<uint8_t*>(t.minfree + kB);
  t.ws = t.sflag + kB;
  t.ogeo = reinterpret_cast<int4*>(t.ws + kWarps * ws_bytes);
  return t;
}

__host__ __device__ constexpr size_t tile_bytes(int words) {
  return 6 * 8 * (size_t)kB + 2 * (size_t)words * kB * 4 + (size_t)kB * 4 +
         (size_t)(kQueue + kCand) * 4 + 3 * (size_t)kB * 4 + kB;
}

struct Local {  // per-thread counters, flushed once at kernel end
  unsigned checked = 0, sampled = 0, accepted = 0;
  CheckCounters cnt{0, 0, 0, 0};
};

__device__ __forceinline__ void flush(const PlaceParams& p, const Local& l) {
  auto add = [&](int k, unsigned v) {
    unsigned s = __reduce_add_sync(kFull, v);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(p.counters + k, (unsigned long long)s);
  };
  add(0, l.checked);
  add(1, l.cnt.narrow);
  add(2, l.cnt.pairs);
  add(3, l.sampled);
  add(4, l.cnt.broad);
  add(5, l.cnt.nodes);
  add(6, l.accepted);
}

// Sampling source of the placement, resolved on the device when the host left the
// fast-path/per-instance decision to the variation flag.
struct Sampling {
  int fast;
  const SbRegionTri* tris;
  const double* cum;
  int n;
};

__device__ __forceinline__ Sampling resolve_sampling(const PlaceParams& p) {
  Sampling s{p.fast, p.canon_tris, p.canon_cum, p.canon_n};
  if (p.vary_flag) {
    const bool vary = __ldcg(p.vary_flag) != 0;
    s.fast = vary ? 0 : 1;
    if (!vary) {
      s.tris = p.inst_tris;
      s.cum = p.inst_cum;
      s.n = __ldcg(p.inst_n);
    }
  }
  return s;
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Phase clock (block 0, thread 0; device globaltimer) into p.prof[slot] (ns):
// 0 setup + tile init, 1 fast-path prefix scan, 2 A1 sample/compose, 3 A2+B broad/narrow,
// 4 C accept + compaction, 5 grid barrier, 6 per-instance path (whole), 7 fast rounds.
__device__ __forceinline__ void dbg_mark(const PlaceParams& p, Fixed& F, unsigned long long& acc) {
  if ((p.dbg || p.dbg_inst) && threadIdx.x == 0) {
    const unsigned long long now = global_ns();
    acc += now - F.t0;
    F.t0 = now;
  }
}

__device__ __forceinline__ void lap(const PlaceParams& p, Fixed& F, int slot) {
  if (p.prof && blockIdx.x == 0 && threadIdx.x == 0) {
    const unsigned long long now = global_ns();
    F.acc[slot] += now - F.tclk;
    F.tclk = now;
  }
}

// A1 core for one slot (sampler.cpp:70-156 + the driver's pose compose): the position
// (FIFO draw `draw`, or the counter stream make_stream(run_seed, {salt, "fall", inst, at}))
// mapped through the support frame, the yaw, and pose = translation(p + z_off z) *
// rotation_z(yaw) in the shim's operation order. Returns false when the region is empty
// (placeable = 0: a failed attempt).
__device__ __forceinline__ bool compose_candidate(const PlaceParams& p, const Sampling& S,
                                                  uint64_t seed, uint64_t state0, uint32_t inst,
                                                  int32_t at, uint64_t draw, M34& pose,
                                                  double* rec = nullptr) {
  const WorldView& w = p.w;
  const SbPlacementDev& pl = p.pl;
  const uint64_t gid = p.global_begin + inst;
  double lx = 0.0, ly = 0.0;
  if (S.fast) {
    if (S.n == 0) return false;
    // j-th drained point = j-th draw (sampler.cpp:30-43): 6j PCG steps in
    Pcg r{pcg_jump_draws(p.jump, state0, draw)};
    double u = r.next_double(), r1 = r.next_double(), r2 = r.next_double();
    sbp::draw_point(S.tris, S.cum, S.n, u, r1, r2, lx, ly);
  } else {
    const int nti = __ldg(p.inst_n + inst);
    if (nti == 0) return false;
    // make_stream(run_seed, {salt, "fall", inst, attempt}) (sampler.cpp:117)
    Pcg r = Pcg::seeded(stream_seed4(seed, pl.salt, kFallbackSalt, gid, static_cast<uint64_t>(at)));
    double u = r.next_double(), r1 = r.next_double(), r2 = r.next_double();
    const uint64_t off = (uint64_t)inst * p.inst_cap;
    sbp::draw_point(p.inst_tris + off, p.inst_cum + off, nti, u, r1, r2, lx, ly);
  }
  M34 Sp;  // support_world[inst]
  if (pl.support_inst) {
    const double2* sp = reinterpret_cast<const double2*>(pl.support_inst + (size_t)inst * 12);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const double2 v = __ldcg(sp + k);
      Sp.m[2 * k] = v.x;
      Sp.m[2 * k + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 12; ++k) Sp.m[k] = pl.support[k];
  }
  double px, py, pz;
  xform(Sp, lx, ly, 0.0, px, py, pz);  // transform_point(support_world, (x, y, 0))
  double yaw = 0.0;
  if (pl.orientation == SB_ORIENT_UNIFORM_YAW) {  // sampler.cpp:140-141
    Pcg r = Pcg::seeded(stream_seed4(seed, pl.salt, kYawSalt, gid, static_cast<uint64_t>(at)));
    const double two_pi = 2.0 * 3.14159265358979323846;
    yaw = 0.0 + (two_pi - 0.0) * r.next_double();
  } else if (pl.orientation == SB_ORIENT_FACE_TO) {  // relationships.cpp:232-239
    const double* tp = w.pose + sb_pose_off(w, pl.face_object, inst);
    double dx = tp[3] - px, dy = tp[7] - py;
    yaw = sqrt(dx * dx + dy * dy) < 1e-12 ? 0.0 : sbg::atan2(dy, dx);
  }
  double c, s;
  sbg::sincos(yaw, &s, &c);  // rotation_z: std::cos / std::sin (transform.hpp:47)
  M34 Tr, Rz;  // translation(p + z_off z) * rotation_z(yaw)
#pragma unroll
  for (int k = 0; k < 12; ++k) Tr.m[k] = Rz.m[k] = 0.0;
  Tr.m[0] = Tr.m[5] = Tr.m[10] = 1.0;
  Rz.m[10] = 1.0;
  Tr.m[3] = px + 0.0;
  Tr.m[7] = py + 0.0;
  Tr.m[11] = pz + pl.z_off;
  Rz.m[0] = c;
  Rz.m[1] = -s;
  Rz.m[4] = s;
  Rz.m[5] = c;
  mul34(Tr, Rz, pose);
  if (rec) {
    rec[0] = Tr.m[3];
    rec[1] = Tr.m[7];
    rec[2] = Tr.m[11];
    rec[3] = c;
    rec[4] = s;
    rec[5] = 0.0;
  }
  return true;
}

// The candidate pose from its compact record {tx, ty, tz, cos, sin, 0} (48 B, what
// compose_candidate wrote): translation * rotation_z rebuilt and multiplied with the same
// operations, so the result is bit-identical to compose_candidate's pose.
__device__ __forceinline__ void pose_from_rec(const double* rec, M34& pose) {
  M34 Tr, Rz;
#pragma unroll
  for (int k = 0; k < 12; ++k) Tr.m[k] = Rz.m[k] = 0.0;
  Tr.m[0] = Tr.m[5] = Tr.m[10] = 1.0;
  Rz.m[10] = 1.0;
  Tr.m[3] = rec[0];
  Tr.m[7] = rec[1];
  Tr.m[11] = rec[2];
  Rz.m[0] = rec[3];
  Rz.m[1] = -rec[4];
  Rz.m[4] = rec[4];
  Rz.m[5] = rec[3];
  mul34(Tr, Rz, pose);
}
__device__ __forceinline__ void load_rec(const double* g, double rec[6]) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double2 v = __ldcg(reinterpret_cast<const double2*>(g) + k);
    rec[2 * k] = v.x;
    rec[2 * k + 1] = v.y;
  }
}

// Fused placement_filter (reachability.cpp:164-190): the candidate frame's origin in the
// instance's robot base frame must hit occ_any; an unreachable candidate is a failed
// attempt that is not collision-checked (Appendix C item 8).
__device__ __forceinline__ bool reach_ok(const PlaceParams& p, uint32_t inst, const M34& pose) {
  M34 Bs, Bi;
  const double* bp = p.reach_base + (size_t)inst * 12;
#pragma unroll
  for (int k = 0; k < 12; ++k) Bs.m[k] = __ldg(bp + k);
  inverse_rigid(Bs, Bi);
  double rx, ry, rz;
  xform(Bi, pose.m[3], pose.m[7], pose.m[11], rx, ry, rz);
  uint64_t ir, iz;
  return reach_bin(p.reach_grid, rx, ry, rz, ir, iz) &&
         reach_bit(p.reach_any, ir * p.reach_grid.nz + iz);
}

// Accept (update_transform, collision.cpp:408-412, + set_enabled): the candidate pose q
// (row-major 3x4 as 6 double2) and its world box (min xyz, max xyz) become instance inst's
// record of the placement's object; the attempt index and (optionally) the column-major
// result pose are written.
template <bool kGrid>
__device__ __forceinline__ void accept_candidate(const PlaceParams& p, uint32_t inst, const double2 q[6],
                                                 const double* box, int32_t attempt) {
  const WorldView& w = p.w;
  const SbPlacementDev& pl = p.pl;
  double2* pp = reinterpret_cast<double2*>(w.pose + sb_pose_off(w, pl.object, inst));
#pragma unroll
  for (int k = 0; k < 6; ++k) pp[k] = q[k];
  if (p.out16) {  // the result pose, column-major Mat4 (k_pose_colmajor layout)
    const double* m = reinterpret_cast<const double*>(q);
    double2* o = reinterpret_cast<double2*>(p.out16 + (size_t)inst * 16);
    o[0] = make_double2(m[0], m[4]);
    o[1] = make_double2(m[8], 0.0);
    o[2] = make_double2(m[1], m[5]);
    o[3] = make_double2(m[9], 0.0);
    o[4] = make_double2(m[2], m[6]);
    o[5] = make_double2(m[10], 0.0);
    o[6] = make_double2(m[3], m[7]);
    o[7] = make_double2(m[11], 1.0);
  }
  double2* bp = reinterpret_cast<double2*>(w.box + sb_box_off(w, pl.object, inst));
#pragma unroll
  for (int k = 0; k < 3; ++k) bp[k] = make_double2(box[2 * k], box[2 * k + 1]);
  w.enabled[sb_word_off(w, pl.object >> 5, inst)] |= 1u << (pl.object & 31);
  if (kGrid) cell_insert(p.grid, inst, pl.object, box, box + 3);
  p.accepted[inst] = (int16_t)attempt;
}

// Leaf-box filter of one (candidate, object) pair, thread-level: warp_collide's step 2 on
// its own. other_in_cand = inv(cand) * pose(ob) and B's leaf boxes moved into A's frame
// are computed with the very operations warp_collide uses, so "no leaf pair's boxes
// overlap" here is exactly warp_collide returning false at step 2 (a miss). inv / pose:
// row-major 3x4 (global memory); gr = obj_grec of the object.
template <bool kCandRec = false>
__device__ __forceinline__ bool leaf_filter(const WorldView& w, const PlaceGeomCache& gc,
                                            const double* inv, const double* pose, int4 gr) {
  double I[12], P[12];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const double2 b = __ldcg(reinterpret_cast<const double2*>(pose) + k);
    P[2 * k] = b.x;
    P[2 * k + 1] = b.y;
  }
  if constexpr (kCandRec) {  // `inv` is the candidate's compact record: pose, then inverse
    double rec[6];
    load_rec(inv, rec);
    M34 C, Ci;
    pose_from_rec(rec, C);
    inverse_rigid(C, Ci);
#pragma unroll
    for (int k = 0; k < 12; ++k) I[k] = Ci.m[k];
  } else {
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const double2 a = __ldcg(reinterpret_cast<const double2*>(inv) + k);
      I[2 * k] = a.x;
      I[2 * k + 1] = a.y;
    }
  }
  M34 M;  // warp_collide's other_in_cand, entry by entry (shim order)
#pragma unroll
  for (int e = 0; e < 12; ++e) {
    const int i = e >> 2, j = e & 3;
    double s = I[4 * i + 0] * P[j];
    s = s + I[4 * i + 1] * P[4 + j];
    s = s + I[4 * i + 2] * P[8 + j];
    s = s + I[4 * i + 3] * (j == 3 ? 1.0 : 0.0);
    M.m[e] = s;
  }
  const unsigned char* rec = reinterpret_cast<const unsigned char*>(w.brec) + 16 * (size_t)gr.x;
  const int nB = gr.z, nA = gc.n_leaves;
  const uint32_t* info = reinterpret_cast<const uint32_t*>(rec + 48 * nB);
  for (int b = 0; b < nB; ++b) {
    if ((__ldg(info + 2 * b) & 0xffu) != 0xffu) continue;  // B leaf nodes only
    const double* nbox = reinterpret_cast<const double*>(rec) + 6 * b;
    double c[3], h[3], bmn[3], bmx[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      c[k] = __ldg(nbox + k);
      h[k] = __ldg(nbox + 3 + k);
    }
    xform_aabb(M, c, h, bmn, bmx);
    for (int l = 0; l < nA; ++l) {
      const int a = gc.leaves[l];
      if (gc.bmin[a][0] <= bmx[0] && bmn[0] <= gc.bmax[a][0] && gc.bmin[a][1] <= bmx[1] &&
          bmn[1] <= gc.bmax[a][1] && gc.bmin[a][2] <= bmx[2] && bmn[2] <= gc.bmax[a][2])
        return true;
    }
  }
  return false;
}

constexpr uint32_t kQueueDone = 0xffffffffu;  // queue entry settled by the leaf filter

// ---------------- B: warp per queued pair (warp w takes entries w, w + 8, ...). Pairs
// behind a lower hit of their slot, or of a slot beyond their instance's lowest
// confirmed-free attempt, are skipped before any data is staged; the next eligible pair's
// pose and geometry record are copied into the warp's other staging buffer (cp.async)
// while the current one is tested. All threads of the CTA call it.
__device__ __forceinline__ void narrow_drain(const PlaceParams& p, Tile& T, Fixed& F, uint32_t nt, uint32_t qn,
                             Local& L) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const WorldView& w = p.w;
  const WarpScratchView ws = carve_scratch(T.ws + warp * p.ws_bytes, p.max_tris, p.max_nodes);
  unsigned char* wsb = T.ws + warp * p.ws_bytes;
  auto skippable = [&](int v, int ob) {
    return *((volatile int32_t*)T.contact + v) < ob ||
           v / (int)nt > *((volatile int32_t*)T.minfree + v % (int)nt);
  };
  // Pairs are claimed one at a time from a shared counter (F.qhead, zeroed by the caller),
  // so a warp that drew cheap pairs (skips, early exits) takes more of them.
  // Thread per queued pair: the leaf-box filter settles most pairs as misses (the same
  // bookkeeping as a warp-tested miss below) before any warp stages one.
  for (uint32_t q = threadIdx.x; q < qn; q += kB) {
    const uint32_t ent = T.queue[q];
    const int v = (int)(ent >> 24), ob = (int)(ent & 0xffffffu);
    if (skippable(v, ob)) continue;
    if (!leaf_filter(w, F.gc, p.cinv + ((size_t)blockIdx.x * kB + v) * 12,
                     w.pose + sb_pose_off(w, ob, T.list[v % (int)nt]), T.ogeo[ob])) {
      T.queue[q] = kQueueDone;
      if (atomicSub(T.rem + v, 1u) == 1u &&
          (*((volatile uint8_t*)T.sflag + v) & kSlotEnumerated) &&
          *((volatile int32_t*)T.contact + v) == kFree)
        atomicMin(T.minfree + v % (int)nt, v / (int)nt);
    }
  }
  __syncthreads();
  auto claim = [&]() -> uint32_t {  // next non-skippable queue index, or qn
    for (;;) {
      uint32_t q = 0;
      if (lane == 0) q = atomicAdd(&F.qhead, 1u);
      q = __shfl_sync(kFull, q, 0);
      if (q >= qn) return qn;
      const uint32_t ent = T.queue[q];
      if (ent != kQueueDone && !skippable((int)(ent >> 24), (int)(ent & 0xffffffu))) return q;
    }
  };
  auto stage = [&](uint32_t ent, int buf) {
    const int v = (int)(ent >> 24), ob = (int)(ent & 0xffffffu);
    warp_stage(w, T.ogeo[ob], ob, T.list[v % (int)nt], p.cinv + ((size_t)blockIdx.x * kB + v) * 12,
               stage_buf(wsb, p.max_tris, p.max_nodes, buf));
  };
  int cur = 0;
  uint32_t q = claim();
  if (q < qn) stage(T.queue[q], cur);
  while (q < qn) {
    const uint32_t ent_cur = T.queue[q];
    const uint32_t q2 = claim();
    if (q2 < qn) {
      stage(T.queue[q2], cur ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const int v = (int)(ent_cur >> 24), ob = (int)(ent_cur & 0xffffffu);
    if (!skippable(v, ob)) {
      const int e = v % (int)nt, sl = v / (int)nt;
      const bool hit = warp_collide(F.gc, stage_buf(wsb, p.max_tris, p.max_nodes, cur),
                                    T.ogeo[ob].z, T.ogeo[ob].w, ws, L.cnt);
      if (p.dbg_inst && lane == 0) atomicAdd(&F.dt, 1u);
      if (lane == 0) {
        if (hit) {
          atomicMin(T.contact + v, ob);
        } else if (atomicSub(T.rem + v, 1u) == 1u &&
                   (*((volatile uint8_t*)T.sflag + v) & kSlotEnumerated) &&
                   *((volatile int32_t*)T.contact + v) == kFree) {
          atomicMin(T.minfree + e, sl);
        }
      }
    }
    __syncwarp();
    q = q2;
    cur ^= 1;
  }
}

// ------------------------------------------------------------------ one tile round
// Evaluates attempts [a, a + W) of the tile's nt active instances (T.list) and compacts the
// survivors in place. Slots are attempt-major (slot v = s * nt + e is attempt a + s of entry
// e), so the narrow queue lists every instance's first attempt before any second one and
// an instance's later attempts are mostly skipped once a lower one is confirmed free.
// Returns the survivor count. All threads of the CTA call it.
template <bool kGrid, bool kReach>
__device__ uint32_t tile_round(const PlaceParams& p, const Sampling& S, const SbGeom& gA,
                               Tile& T, Fixed& F, uint32_t nt, int32_t a, int W,
                               uint64_t draw_base, Local& L) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const WorldView& w = p.w;
  const SbPlacementDev& pl = p.pl;
  const int words = w.n_words, nobj = w.n_objects;
  const int nslots = (int)nt * W;

  // enable words of the tile's instances (independent loads, consumed in A2)
  for (int i = tid; i < (int)nt * words; i += kB) {
    const int wd = i / (int)nt, e = i - wd * (int)nt;
    T.enw[wd * kB + e] = __ldcg(w.enabled + sb_word_off(w, wd, T.list[e]));
  }
  // ---------------- A1: thread per slot
  if (tid < nslots) {
    const int v = tid;
    const int e = v % (int)nt;  // attempt-major slots: v = s * nt + e
    const int32_t at = a + v / (int)nt;
    const uint32_t inst = T.list[e];
    // slot v = s * nt + e is round a + s, rank e: FIFO draw draw_base + s * nt + e =
    // draw_base + v while nobody accepts before round a + s (speculation, resolved in C)
    M34 pose;
    const bool placeable = compose_candidate(p, S, F.seed, F.state0, inst, at,
                                             draw_base + (uint64_t)v, pose);
    T.contact[v] = kFree;
    T.rem[v] = 0u;
    if (v < (int)nt) T.minfree[e] = W;
    for (int wd = 0; wd < words; ++wd) T.ovm[wd * kB + v] = 0u;
    if (!placeable) {
      T.sflag[v] = kSlotUnplaceable;
    } else {
      double cmn[3], cmx[3];
      xform_aabb(pose, gA.box_c, gA.box_h, cmn, cmx);
      M34 inv;
      inverse_rigid(pose, inv);
      double2* cp = reinterpret_cast<double2*>(p.cpose + ((size_t)blockIdx.x * kB + v) * 12);
#pragma unroll
      for (int k = 0; k < 6; ++k) cp[k] = make_double2(pose.m[2 * k], pose.m[2 * k + 1]);
#pragma unroll
      for (int k = 0; k < 6; ++k)
        reinterpret_cast<double2*>(p.cinv + ((size_t)blockIdx.x * kB + v) * 12)[k] =
            make_double2(inv.m[2 * k], inv.m[2 * k + 1]);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        T.box[6 * v + k] = cmn[k];
        T.box[6 * v + 3 + k] = cmx[k];
      }
      T.sflag[v] = kSlotChecked;
      if constexpr (kReach) {
        if (!reach_ok(p, inst, pose)) T.sflag[v] = kSlotUnplaceable;
      }
    }
  }
  if (tid == 0) {
    F.qn = 0;
    F.qhead = 0;
    F.dq = F.dt = 0;
  }
  __syncthreads();
  lap(p, F, 2);
  dbg_mark(p, F, F.ta);

  if constexpr (!kGrid) {
    // ---------------- A2 (broad phase) + B, few objects: item per (slot, enabled object),
    // four box loads in flight per thread (aabb.hpp:29-33, collision.cpp:439-443); the
    // queue (queue + cand storage, kQueue + kCand entries) is drained when nearly full.
    constexpr int kU = 4;
    constexpr uint32_t kQD = kQueue + kCand;
    const int items = nslots * nobj;
    for (int it0 = 0; it0 < items; it0 += kB * kU) {
      bool ov[kU];
      int vs[kU], obs[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int it = it0 + u * kB + tid;
        ov[u] = false;
        vs[u] = 0;
        obs[u] = 0;
        if (it < items) {
          const int v = it / nobj;
          const int ob = it - v * nobj;
          vs[u] = v;
          obs[u] = ob;
          if (T.sflag[v] == kSlotChecked &&
              ((T.enw[(ob >> 5) * kB + v % (int)nt] >> (ob & 31)) & 1u)) {
            ++L.cnt.broad;
            const double2* bp =
                reinterpret_cast<const double2*>(w.box + sb_box_off(w, ob, T.list[v % (int)nt]));
            const double2 b0 = __ldcg(bp), b1 = __ldcg(bp + 1), b2 = __ldcg(bp + 2);
            const double* cb = T.box + 6 * v;
            ov[u] = cb[0] <= b1.y && b0.x <= cb[3] && cb[1] <= b2.x && b0.y <= cb[4] &&
                    cb[2] <= b2.y && b1.x <= cb[5];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint32_t mask = __ballot_sync(kFull, ov[u]);
        if (!mask) continue;
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&F.qn, (uint32_t)__popc(mask));
        base = __shfl_sync(kFull, base, 0);
        if (ov[u]) {
          atomicOr(T.ovm + (obs[u] >> 5) * kB + vs[u], 1u << (obs[u] & 31));
          atomicAdd(T.rem + vs[u], 1u);
          T.queue[base + __popc(mask & ((1u << lane) - 1u))] = ((uint32_t)vs[u] << 24) | (uint32_t)obs[u];
        }
      }
      __syncthreads();
      // slots whose items are now all enumerated: free if no queued pair is pending
      const bool last = it0 + kB * kU >= items;
      const int vdone = last ? nslots : (it0 + kB * kU) / nobj;
      const int vprev = it0 / nobj;
      for (int v = vprev + tid; v < vdone; v += kB)
        if (T.sflag[v] == kSlotChecked) {
          T.sflag[v] = kSlotChecked | kSlotEnumerated;
          if (T.rem[v] == 0u && T.contact[v] == kFree) atomicMin(T.minfree + v % (int)nt, v / (int)nt);
        }
      __syncthreads();
      const uint32_t qn = F.qn;
      if (last || qn > kQD - kB * kU) {
        if (p.dbg_inst && tid == 0) F.dq += qn;
        narrow_drain(p, T, F, nt, qn, L);
        __syncthreads();
        if (tid == 0) {
          F.qn = 0;
          F.qhead = 0;
        }
        __syncthreads();
      }
    }
    if (items == 0) __syncthreads();
  } else {
  // ---------------- A2 (broad phase) + B (narrow phase). The candidate objects of a slot are
  // the OR of the occupancy-grid cells its box meets (only enabled objects are ever in a
  // cell). Slots' candidates are expanded into a shared item list (block scan), then
  // tested item-parallel against the world AABBs (aabb.hpp:29-33, collision.cpp:439-443),
  // kCand items per chunk; the chunk's overlapping pairs go to the queue, which B drains.
  uint32_t pend[kGW];
  uint32_t cnt = 0;
  {
    const bool mine = tid < nslots && T.sflag[tid] == kSlotChecked;
#pragma unroll
    for (int wd = 0; wd < kGW; ++wd) pend[wd] = 0u;
    if (mine) {
      const SbCellGrid& G = p.grid;
      int cx0, cx1, cy0, cy1;
      cell_range(G, T.box + 6 * tid, T.box + 6 * tid + 3, cx0, cx1, cy0, cy1);
      const uint32_t* cb = G.cells + (uint64_t)T.list[tid % (int)nt] * (uint64_t)(G.g * G.g) * words;
      for (int cy = cy0; cy <= cy1; ++cy)
        for (int cx = cx0; cx <= cx1; ++cx) {
          const uint32_t* c = cb + (uint64_t)(cy * G.g + cx) * words;
          if (words == 4) {  // the cell's words in one 16-byte load
            const uint4 v = __ldcg(reinterpret_cast<const uint4*>(c));
            pend[0] |= v.x;
            pend[1] |= v.y;
            pend[2] |= v.z;
            pend[3] |= v.w;
            continue;
          }
#pragma unroll
          for (int wd = 0; wd < kGW; ++wd)
            if (wd < words) pend[wd] |= __ldcg(c + wd);
        }
#pragma unroll
      for (int wd = 0; wd < kGW; ++wd) cnt += __popc(pend[wd]);
    }
  }
  uint32_t off, ncand;
  BlockScan(F.scan).ExclusiveSum(cnt, off, ncand);
  __syncthreads();
  for (uint32_t c0 = 0; c0 < ncand || c0 == 0; c0 += kCand) {
    const uint32_t nitems = ncand - c0 < (uint32_t)kCand ? ncand - c0 : (uint32_t)kCand;
    if (cnt && off < c0 + nitems && off + cnt > c0) {  // this slot's items in the chunk
      uint32_t idx = off;
#pragma unroll
      for (int wd = 0; wd < kGW; ++wd) {
        uint32_t m = pend[wd];
        while (m) {
          const int ob = 32 * wd + __ffs(m) - 1;
          m &= m - 1u;
          if (idx >= c0 && idx < c0 + nitems) T.cand[idx - c0] = ((uint32_t)tid << 24) | (uint32_t)ob;
          ++idx;
        }
      }
    }
    if (tid == 0) {
          F.qn = 0;
          F.qhead = 0;
        }
    __syncthreads();
    {  // item-parallel AABB tests, two box loads in flight per thread
      constexpr int kI = kCand / kB;
#pragma unroll 1
      for (int u0 = 0; u0 < kI; u0 += 2) {
        double2 bx[2][3];
        uint32_t ent[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint32_t i = (u0 + u) * kB + tid;
          ent[u] = i < nitems ? T.cand[i] : 0xffffffffu;
          if (i < nitems) {
            const int v = (int)(ent[u] >> 24), ob = (int)(ent[u] & 0xffffffu);
            const double2* bp =
                reinterpret_cast<const double2*>(w.box + sb_box_off(w, ob, T.list[v % (int)nt]));
            bx[u][0] = __ldcg(bp);
            bx[u][1] = __ldcg(bp + 1);
            bx[u][2] = __ldcg(bp + 2);
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          bool ov = false;
          int v = 0, ob = 0;
          if (ent[u] != 0xffffffffu) {
            v = (int)(ent[u] >> 24);
            ob = (int)(ent[u] & 0xffffffu);
            ++L.cnt.broad;
            const double* cb = T.box + 6 * v;
            const double2 b0 = bx[u][0], b1 = bx[u][1], b2 = bx[u][2];
            ov = cb[0] <= b1.y && b0.x <= cb[3] && cb[1] <= b2.x && b0.y <= cb[4] &&
                 cb[2] <= b2.y && b1.x <= cb[5];
          }
          const uint32_t mask = __ballot_sync(kFull, ov);
          if (!mask) continue;
          uint32_t base = 0;
          if (lane == 0) base = atomicAdd(&F.qn, (uint32_t)__popc(mask));
          base = __shfl_sync(kFull, base, 0);
          if (ov) {
            atomicOr(T.ovm + (ob >> 5) * kB + v, 1u << (ob & 31));
            atomicAdd(T.rem + v, 1u);
            T.queue[base + __popc(mask & ((1u << lane) - 1u))] = ((uint32_t)v << 24) | (uint32_t)ob;
          }
        }
      }
    }
    __syncthreads();
    // slots whose candidates are now all enumerated: free if no queued pair is pending
    if (tid < nslots && T.sflag[tid] == kSlotChecked && off + cnt <= c0 + nitems) {
      T.sflag[tid] = kSlotChecked | kSlotEnumerated;
      if (T.rem[tid] == 0u && T.contact[tid] == kFree)
        atomicMin(T.minfree + tid % (int)nt, tid / (int)nt);
    }
    __syncthreads();
    const uint32_t qn = F.qn;
    if (p.dbg_inst && tid == 0) F.dq += qn;
    if (qn > 0) {
      narrow_drain(p, T, F, nt, qn, L);
    }
    __syncthreads();
    if (ncand == 0) break;
  }
  }
  lap(p, F, 3);
  dbg_mark(p, F, F.tb);

  // ---------------- C: thread per instance; first free slot is accepted (Appendix C.5)
  // FIFO speculation (S.fast, W > 1): rounds a .. a + slim are exact, where slim = the first
  // round in which any instance is free (ranks shift after an accept); later slots are
  // discarded and F.used = rounds consumed. Per-instance streams: every slot is exact.
  int lim = W - 1;
  if (S.fast && W > 1) {
    if (tid == 0) F.used = W;
    __syncthreads();
    if (tid < (int)nt && T.minfree[tid] < W) atomicMin(&F.used, T.minfree[tid]);
    __syncthreads();
    if (F.used < W) lim = F.used;
    __syncthreads();
    if (tid == 0) F.used = lim + 1;
  } else if (tid == 0) {
    F.used = W;
  }
  uint32_t keep = 0, inst = 0;
  if (tid < (int)nt) {
    const int e = tid;
    inst = T.list[e];
    int32_t last = a;  // last attempt this instance made in the sequential loop
    bool ok = false;
    for (int s = 0; s <= lim && !ok; ++s) {
      const int v = s * (int)nt + e;
      last = a + s;
      ++L.sampled;
      if (!(T.sflag[v] & kSlotChecked)) continue;  // placeable == 0 -> failed attempt
      ++L.checked;
      const int32_t c = T.contact[v];
      for (int wd = 0; wd < words; ++wd) {  // narrow tests up to the first hit
        uint32_t mk = T.ovm[wd * kB + v];
        if (c != kFree) {
          const int lim = c - 32 * wd;  // keep objects <= c
          if (lim < 0) mk = 0;
          else if (lim < 31) mk &= (2u << lim) - 1u;
        }
        L.cnt.narrow += __popc(mk);
      }
      if (c == kFree) {  // update_transform (collision.cpp:408-412) + set_enabled
        double2 q[6];
#pragma unroll
        for (int k = 0; k < 6; ++k)
          q[k] = __ldcg(reinterpret_cast<const double2*>(p.cpose + ((size_t)blockIdx.x * kB + v) * 12) + k);
        accept_candidate<kGrid>(p, inst, q, T.box + 6 * v, a + s);
        ++L.accepted;
        ok = true;
      }
    }
    atomicMax(p.ctrl + kRounds, (uint32_t)(last + 1));  // reference round count
    keep = ok ? 0u : 1u;
  }
  uint32_t rank, total;
  BlockScan(F.scan).ExclusiveSum(keep, rank, total);
  __syncthreads();  // every thread has read T.list[tid]
  if (keep) T.list[rank] = inst;
  __syncthreads();
  lap(p, F, 4);
  return total;
}

// Stable compaction of the valid instances of tile t into T.list; returns the count.
__device__ uint32_t tile_load_valid(const PlaceParams& p, Tile& T, Fixed& F, uint32_t t,
                                    uint32_t ti) {
  const uint64_t i = (uint64_t)t * ti + threadIdx.x;
  const uint32_t f = (threadIdx.x < ti && i < p.w.n && p.valid[i] != 0) ? 1u : 0u;
  uint32_t rank, total;
  BlockScan(F.scan).ExclusiveSum(f, rank, total);
  if (f) T.list[rank] = (uint32_t)i;
  __syncthreads();
  return total;
}

__device__ __forceinline__ void mark_invalid(const PlaceParams& p, const Tile& T, uint32_t nt) {
  for (uint32_t e = threadIdx.x; e < nt; e += kB) p.valid[T.list[e]] = 0;  // mark_invalid
}

// Fast path: exclusive prefix of the per-tile survivor counts for the CTA's tiles
// (t = blockIdx.x + k * gridDim.x) into F.prefix / F.cnt; returns the round total.
// Tiles of the fast path's current lists: all of them, or those k_wide_spread filled.
__device__ __forceinline__ uint32_t tiles_in_use(const PlaceParams& p) {
  return p.ntiles_dev ? (uint32_t)__ldcg(p.ntiles_dev) : p.ntiles;
}

__device__ uint64_t tile_prefix(const PlaceParams& p, const uint32_t* cnt, Fixed& F) {
  const uint32_t G = gridDim.x, b = blockIdx.x, nt = tiles_in_use(p);
  uint64_t running = 0;
  for (uint32_t c0 = 0; c0 < nt; c0 += kB * kPrefixItems) {
    uint32_t x[kPrefixItems], ex[kPrefixItems], agg;
#pragma unroll
    for (int j = 0; j < kPrefixItems; ++j) {
      const uint32_t idx = c0 + threadIdx.x * kPrefixItems + j;
      x[j] = idx < nt ? __ldcg(cnt + idx) : 0u;
    }
    BlockScan(F.scan).ExclusiveSum(x, ex, agg);
#pragma unroll
    for (int j = 0; j < kPrefixItems; ++j) {
      const uint32_t idx = c0 + threadIdx.x * kPrefixItems + j;
      if (idx < nt && idx % G == b) {
        F.prefix[idx / G] = (uint32_t)running + ex[j];
        F.cnt[idx / G] = x[j];
      }
    }
    running += agg;
    __syncthreads();
  }
  return running;
}

__device__ __forceinline__ void load_list(const PlaceParams& p, Tile& T, uint32_t t, uint32_t n) {
  const uint32_t* src = p.tile_list + (uint64_t)t * p.tile_inst;
  for (uint32_t e = threadIdx.x; e < n; e += kB) T.list[e] = __ldcg(src + e);
  __syncthreads();
}

__device__ __forceinline__ void store_list(const PlaceParams& p, const Tile& T, uint32_t t,
                                           uint32_t n, uint32_t* cnt_out) {
  uint32_t* dst = p.tile_list + (uint64_t)t * p.tile_inst;
  for (uint32_t e = threadIdx.x; e < n; e += kB) dst[e] = T.list[e];
  if (threadIdx.x == 0) cnt_out[t] = n;
}

// One fast-path round over the CTA's tiles: survivors of round a -> counts of round a+1.
template <bool kGrid, bool kReach>
// `resident`: the CTA owns at most one tile and T.list still holds its survivors from the
// previous round (persistent kernel), so the list is not reloaded.
__device__ uint64_t fast_round(const PlaceParams& p, const Sampling& S, const SbGeom& gA,
                               Tile& T, Fixed& F, int32_t a, uint64_t draws, Local& L,
                               uint32_t* total_word, bool resident,
                               unsigned long long* total_word64 = nullptr) {
  const uint32_t* cin = p.tile_cnt + (size_t)(a & 1) * p.cnt_stride;
  uint32_t* cout = p.tile_cnt + (size_t)((a + 1) & 1) * p.cnt_stride;
  const uint64_t total = tile_prefix(p, cin, F);
  lap(p, F, 1);
  if (total == 0) return 0;
  if (total <= (uint64_t)p.solo_max) return total | kSoloFlag;  // caller runs solo rounds
  uint32_t k = 0, mine = 0;
  const uint32_t ntu = tiles_in_use(p);
  for (uint32_t t = blockIdx.x; t < ntu; t += gridDim.x, ++k) {
    const uint32_t n = F.cnt[k];
    if (n == 0) {
      if (threadIdx.x == 0) cout[t] = 0;
      continue;
    }
    if (!resident) load_list(p, T, t, n);
    lap(p, F, 1);
    if (p.dbg && threadIdx.x == 0) F.t0 = global_ns();
    const uint32_t ns = tile_round<kGrid, kReach>(p, S, gA, T, F, n, a, 1, draws + F.prefix[k], L);
    store_list(p, T, t, ns, cout);
    mine += ns;
    __syncthreads();
  }
  if (total_word && threadIdx.x == 0 && mine) atomicAdd(total_word, mine);
  if (total_word64 && threadIdx.x == 0 && mine) atomicAdd(total_word64, (unsigned long long)mine);
  return total;
}

// Fast rounds without a grid barrier (p.lb_board). Round a of tile t needs the draws before
// round a (D_a = D_{a-1} + N_{a-1}: every tile's count of round a - 1, i.e. every tile done
// with round a - 2) and the counts of round a of the tiles below t (those tiles done with
// round a - 1). Each tile publishes its survivor count to the board with a release store;
// readers spin on the entry's epoch. So a tile may run one round ahead of the slowest tile
// instead of waiting for it at a grid barrier. Tile t stays with CTA t % gridDim, which alone
// reads and writes its list; only the counts cross CTAs. The draws (and so every result) are
// those of the barrier version. All CTAs are co-resident (cooperative launch).
__device__ __forceinline__ uint32_t lb_get(const PlaceParams& p, int32_t a, uint32_t t) {
  const unsigned long long* e = p.lb_board + (size_t)a * p.lb_stride + t;
  unsigned long long v;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(e) : "memory");
    if ((uint32_t)(v >> 32) == p.lb_epoch) return (uint32_t)v;
    if (p.lb_sleep) __nanosleep(p.lb_sleep);
  }
}

__device__ __forceinline__ void lb_put(const PlaceParams& p, int32_t a, uint32_t t, uint32_t n) {
  unsigned long long* e = p.lb_board + (size_t)a * p.lb_stride + t;
  const unsigned long long v = ((unsigned long long)p.lb_epoch << 32) | n;
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(e), "l"(v) : "memory");
}

// Counts of round a: from the launch's input buffer for the first round, else the board.
__device__ __forceinline__ uint32_t lb_count(const PlaceParams& p, int32_t a, uint32_t t) {
  return a == p.start_round ? __ldcg(p.tile_cnt + (size_t)(a & 1) * p.cnt_stride + t) : lb_get(p, a, t);
}

template <bool kGrid, bool kReach>
__device__ void lookback_rounds(const PlaceParams& p, const Sampling& S, const SbGeom& gA,
                                Tile& T, Fixed& F, int32_t a, uint64_t draws, Local& L) {
  const uint32_t G = gridDim.x, b = blockIdx.x, ntu = tiles_in_use(p);
  const bool resident = ntu <= G;
  uint64_t n_prev = 0;  // N_{a-1}
  for (; a < p.attempts; ++a) {
    if (a > p.start_round) {  // D_a = D_{a-1} + N_{a-1}
      uint32_t part = 0, ex, tot;
      for (uint32_t t = threadIdx.x; t < ntu; t += kB) part += lb_count(p, a - 1, t);
      BlockScan(F.scan).ExclusiveSum(part, ex, tot);
      __syncthreads();
      n_prev = tot;
      draws += n_prev;
      if (n_prev == 0) return;  // round a - 1 had no active instance: all placed
    }
    // exclusive prefix of round a's counts over the tiles below each of this CTA's tiles
    uint32_t running = 0, k = 0;
    for (uint32_t t = b; t < ntu; t += G, ++k) {
      // tiles (t - G, t): the ones up to t - G are in `running` already
      uint32_t part = 0, ex, s;
      for (uint32_t u = (t >= G ? t - G + 1 : 0) + threadIdx.x; u < t; u += kB) part += lb_count(p, a, u);
      BlockScan(F.scan).ExclusiveSum(part, ex, s);
      __syncthreads();
      running += s;
      const uint32_t n = lb_count(p, a, t);  // own tile: published by this CTA (or the input)
      if (n == 0) {
        if (threadIdx.x == 0) lb_put(p, a + 1, t, 0u);
      } else {
        if (!resident || a == p.start_round) load_list(p, T, t, n);
        const uint32_t ns = tile_round<kGrid, kReach>(p, S, gA, T, F, n, a, 1, draws + running, L);
        if (!resident) {
          uint32_t* dst = p.tile_list + (uint64_t)t * p.tile_inst;
          for (uint32_t e = threadIdx.x; e < ns; e += kB) dst[e] = T.list[e];
        }
        __syncthreads();
        if (threadIdx.x == 0) lb_put(p, a + 1, t, ns);
      }
      running += n;  // the next own tile's prefix continues from here
      __syncthreads();
    }
  }
  // K attempts exhausted: the survivors of this CTA's tiles are invalid
  for (uint32_t t = b; t < ntu; t += G) {
    const uint32_t n = lb_count(p, a, t);
    if (n == 0) continue;
    if (!resident || a == p.start_round) load_list(p, T, t, n);  // no round ran: not loaded
    mark_invalid(p, T, n);
    __syncthreads();
  }
}

// Fast path tail: once at most p.solo_max instances remain, CTA 0 gathers them in global
// active order (tile order, then position) and runs the remaining rounds alone -- no grid
// barrier, no prefix scan; draw j of round a is draws + position, as in the grid rounds.
template <bool kGrid, bool kReach>
__device__ void solo_rounds(const PlaceParams& p, const Sampling& S, const SbGeom& gA, Tile& T,
                            Fixed& F, int32_t a, uint64_t draws, Local& L) {
  const uint32_t* cin = p.tile_cnt + (size_t)(a & 1) * p.cnt_stride;
  uint32_t base = 0;
  const uint32_t ntu = tiles_in_use(p);
  for (uint32_t t0 = 0; t0 < ntu; t0 += kB) {
    const uint32_t t = t0 + threadIdx.x;
    const uint32_t c = t < ntu ? __ldcg(cin + t) : 0u;
    uint32_t off, tot;
    BlockScan(F.scan).ExclusiveSum(c, off, tot);
    const uint32_t* src = p.tile_list + (uint64_t)t * p.tile_inst;
    for (uint32_t e = 0; e < c; ++e) T.list[base + off + e] = __ldcg(src + e);
    base += tot;
    __syncthreads();
  }
  uint32_t nt = base;
  while (nt > 0 && a < p.attempts) {
    // W speculative rounds at once (see tile_round phase C): round a + s of rank e is
    // draw draws + s * nt + e as long as nobody accepts before it
    int W = p.solo_spec / (int)nt;
    if (W < 1) W = 1;
    if (W > kB / (int)nt) W = kB / (int)nt;
    if (W > p.attempts - a) W = p.attempts - a;
    const uint32_t ns = tile_round<kGrid, kReach>(p, S, gA, T, F, nt, a, W, draws, L);
    const int used = F.used;
    draws += (uint64_t)used * nt;
    a += used;
    nt = ns;
  }
  if (a == p.attempts) mark_invalid(p, T, nt);
}

// Per-instance path: tiles are independent; each is run to completion by one CTA.
template <bool kGrid, bool kReach>
__device__ void instance_tiles(const PlaceParams& p, const Sampling& S, const SbGeom& gA,
                               Tile& T, Fixed& F, Local& L) {
  for (;;) {
    if (threadIdx.x == 0) F.tile = atomicAdd(p.ctrl + kTileCtr, 1u);
    __syncthreads();
    const uint32_t c = F.tile;
    __syncthreads();
    if (c >= p.ntiles_pi) break;
    // claim order -> tile: the previous run's slowest tiles first (longest processing time
    // first, so a straggler does not start in the last wave); results do not depend on it
    const uint32_t t = p.tile_perm ? __ldg(p.tile_perm + c) : c;
    uint32_t nt = tile_load_valid(p, T, F, t, p.tile_inst_pi);
    int32_t a = 0;
    unsigned rounds = 0;
    const unsigned long long tt0 = (p.dbg_inst || p.tile_ns) && threadIdx.x == 0 ? global_ns() : 0;
    while (nt > 0 && a < p.attempts) {
      ++rounds;
      int W = p.spec_target / (int)nt;
      if (W < 1) W = 1;
      if (W > kB / (int)nt) W = kB / (int)nt;
      if (W > p.attempts - a) W = p.attempts - a;
      if (p.dbg_inst && threadIdx.x == 0) {
        F.ta = F.tb = 0;
        F.t0 = global_ns();
      }
      const unsigned nslots_dbg = nt * W;
      nt = tile_round<kGrid, kReach>(p, S, gA, T, F, nt, a, W, 0, L);
      a += W;
      if (p.dbg_inst && threadIdx.x == 0) {  // A1 / A2+B / C sums (us) and A2+B max (ns)
        atomicAdd(p.dbg_inst + 5, (unsigned)(F.ta / 1000));
        atomicAdd(p.dbg_inst + 6, (unsigned)(F.tb / 1000));
        atomicAdd(p.dbg_inst + 7, (unsigned)((global_ns() - F.t0) / 1000));
        atomicMax(p.dbg_inst + 8, (unsigned)F.tb);
        atomicAdd(p.dbg_inst + 9, nslots_dbg);
        atomicAdd(p.dbg_inst + 10, F.dq);
        atomicAdd(p.dbg_inst + 11, F.dt);
        atomicMax(p.dbg_inst + 12, F.dq);
        atomicMax(p.dbg_inst + 13, F.dt);
      }
    }
    mark_invalid(p, T, nt);
    if (p.tile_ns && threadIdx.x == 0) {
      const unsigned long long d = global_ns() - tt0;
      p.tile_ns[t] = d < 0xffffffffull ? (uint32_t)d : 0xffffffffu;
    }
    if (p.dbg_inst && threadIdx.x == 0) {  // per-tile debug: max / sum of ns and rounds
      const unsigned dt = (unsigned)(global_ns() - tt0);
      atomicMax(p.dbg_inst + 0, dt);
      atomicAdd(p.dbg_inst + 1, dt / 1000u);
      atomicMax(p.dbg_inst + 2, rounds);
      atomicAdd(p.dbg_inst + 3, rounds);
      atomicAdd(p.dbg_inst + 4, 1u);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ void block_setup(const PlaceParams& p, Fixed& F, Tile& T, SbGeom& gA) {
  if (threadIdx.x == 0) {  // the run seed from device memory (CUDA-graph replays) or the params
    const uint64_t seed = p.seed_dev ? *p.seed_dev : p.run_seed;
    F.seed = seed;
    F.state0 = p.seed_dev ? Pcg::seeded(stream_seed2(seed, p.pl.salt, kCacheSalt)).state
                          : p.fast_state0;
  }
  gA = p.w.geoms[p.pl.geom];
  load_geom_cache(p.w, gA, F.gc);
  for (int ob = threadIdx.x; ob < p.w.n_objects; ob += kB) T.ogeo[ob] = obj_grec(p.w, ob);
  __syncthreads();
}

extern __shared__ __align__(16) unsigned char g_dsm[];

// kMinB: CTAs per SM the register budget is sized for -- 2 (128 registers, spills) by
// default, 1 (no spills, half the warps) for the FIFO placements with SB_PLACE1.
template <bool kGrid, bool kReach, int kMinB = SB_PLACE_MIN_BLOCKS>
__global__ void __launch_bounds__(kB, kMinB) k_place(PlaceParams p) {
  pdl_enter();
  __shared__ Fixed F;
  Tile T = carve(g_dsm, p.w.n_words, p.ws_bytes);
  const bool timer = p.prof && blockIdx.x == 0 && threadIdx.x == 0;
  if (timer) {
    for (int k = 0; k < 8; ++k) F.acc[k] = 0;
    F.tclk = global_ns();
  }
  SbGeom gA;
  block_setup(p, F, T, gA);
  Local L;
  const Sampling S = resolve_sampling(p);
  if (!S.fast) {
    if (p.vary_flag && blockIdx.x == 0 && threadIdx.x == 0)
      atomicAdd(p.counters + 7, 1ull);  // per-instance placement
    const unsigned long long t6 = timer ? global_ns() : 0;
    instance_tiles<kGrid, kReach>(p, S, gA, T, F, L);
    if (timer) F.acc[6] += global_ns() - t6;
  } else {
    cg::grid_group grid = cg::this_grid();
    uint64_t draws = 0;
    int32_t a = 0;
    if (p.start_round == 0) {
      for (uint32_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        const uint32_t n = tile_load_valid(p, T, F, t, p.tile_inst);
        store_list(p, T, t, n, p.tile_cnt);
        __syncthreads();
      }
      lap(p, F, 0);
      grid.sync();
      lap(p, F, 5);
    } else {  // rounds < start_round ran in k_wide_*: their draws precede this round's
      a = p.start_round;
      draws = __ldcg(p.start_draws);
    }
    if (p.lb_board && p.solo_max == 0 && !p.dbg) {
      lookback_rounds<kGrid, kReach>(p, S, gA, T, F, a, draws, L);
      a = -1;  // survivors of exhausted instances marked inside
    }
    for (; a >= 0 && a < p.attempts; ++a) {
      unsigned long long r0 = 0;
      if (p.dbg && threadIdx.x == 0) {
        r0 = global_ns();
        F.ta = F.tb = 0;
      }
      uint64_t total = fast_round<kGrid, kReach>(p, S, gA, T, F, a, draws, L, nullptr,
                                                 tiles_in_use(p) <= gridDim.x && a > p.start_round);
      if (total & kSoloFlag) {
        if (blockIdx.x == 0) solo_rounds<kGrid, kReach>(p, S, gA, T, F, a, draws, L);
        a = -1;  // tail done by CTA 0
        break;
      }
      if (total == 0) break;
      draws += total;
      if (p.dbg && threadIdx.x == 0) {  // per-round maxima over CTAs: work, A1, A2+B
        atomicMax(p.dbg + 3 * a, (unsigned)(global_ns() - r0));
        atomicMax(p.dbg + 3 * a + 1, (unsigned)F.ta);
        atomicMax(p.dbg + 3 * a + 2, (unsigned)F.tb);
        atomicAdd(p.dbg_inst + 14, (unsigned)((global_ns() - r0) / 1000));  // sum of work (us)
        atomicAdd(p.dbg_inst + 15, (unsigned)(F.tb / 1000));                // sum of A2+B (us)
      }
      lap(p, F, 1);
      grid.sync();
      lap(p, F, 5);
      if (timer) F.acc[7] += 1;
    }
    if (a == p.attempts) {  // K attempts exhausted: survivors are invalid
      const uint32_t* cin = p.tile_cnt + (size_t)(a & 1) * p.cnt_stride;
      const uint32_t ntu = tiles_in_use(p);
      for (uint32_t t = blockIdx.x; t < ntu; t += gridDim.x) {
        const uint32_t n = __ldcg(cin + t);
        if (n == 0) continue;
        load_list(p, T, t, n);
        mark_invalid(p, T, n);
        __syncthreads();
      }
    }
  }
  if (timer)
    for (int k = 0; k < 8; ++k) p.prof[k] += F.acc[k];
  flush(p, L);
}

// Sharded building blocks (no grid barrier inside a launch).
template <bool kGrid, bool kReach>
__global__ void __launch_bounds__(kB, SB_PLACE_MIN_BLOCKS) k_place_instances(PlaceParams p) {
  pdl_enter();
  __shared__ Fixed F;
  Tile T = carve(g_dsm, p.w.n_words, p.ws_bytes);
  SbGeom gA;
  if (p.shard_vary && __ldcg(p.shard_vary) == 0) return;  // canonical: the FIFO rounds place it
  block_setup(p, F, T, gA);
  Local L;
  Sampling S{0, nullptr, nullptr, 0};
  instance_tiles<kGrid, kReach>(p, S, gA, T, F, L);
  flush(p, L);
}

__global__ void __launch_bounds__(kB, SB_PLACE_MIN_BLOCKS) k_fast_init(PlaceParams p) {
  pdl_enter();
  __shared__ Fixed F;
  Tile T = carve(g_dsm, p.w.n_words, p.ws_bytes);
  if (p.shard_vary && __ldcg(p.shard_vary) != 0) return;  // per-instance: no FIFO rounds
  uint32_t mine = 0;
  for (uint32_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
    const uint32_t n = tile_load_valid(p, T, F, t, p.tile_inst);
    store_list(p, T, t, n, p.tile_cnt);
    mine += n;
    __syncthreads();
  }
  if (threadIdx.x == 0 && mine) {
    if (p.xcount) atomicAdd(p.xcount, (unsigned long long)mine);
    else atomicAdd(p.ctrl + place_total_word(0), mine);
  }
}

template <bool kGrid, bool kReach>
__global__ void __launch_bounds__(kB, SB_PLACE_MIN_BLOCKS) k_fast_round(PlaceParams p, int32_t a) {
  pdl_enter();
  __shared__ Fixed F;
  Tile T = carve(g_dsm, p.w.n_words, p.ws_bytes);
  SbGeom gA;
  if (p.xrecv) {  // rounds enqueued past the placement's last one: return before any setup
    unsigned long long tot = 0;
    for (int r = 0; r < p.xworld; ++r) tot += __ldcg(p.xrecv + (size_t)a * p.xworld + r);
    if (tot == 0) return;
  }
  block_setup(p, F, T, gA);
  Local L;
  const int32_t canon_n = p.canon_n_dev ? __ldcg(p.canon_n_dev) : p.canon_n;
  Sampling S{1, p.canon_tris, p.canon_cum, canon_n};
  if (p.xrecv) {  // device-side exchange: this round's offsets from the gathered counts
    unsigned long long tot = 0, before = 0;
    for (int r = 0; r < p.xworld; ++r) {
      const unsigned long long v = __ldcg(p.xrecv + (size_t)a * p.xworld + r);
      tot += v;
      if (r < p.xrank) before += v;
    }
    if (tot == 0) return;  // every rank is done: a no-op round
    const unsigned long long draws = __ldcg(p.xdraws + a);
    if (blockIdx.x == 0 && threadIdx.x == 0)
      p.xdraws[a + 1] = draws + (canon_n > 0 ? tot : 0ull);  // cache drained only if sampled
    // this rank has no survivors left: idle, but keep its tile counts maintained (the
    // round-(a+1) buffer still holds round a-1's counts, which k_fast_finish would read)
    if (__ldcg(p.xrecv + (size_t)a * p.xworld + p.xrank) == 0) {
      uint32_t* cout = p.tile_cnt + (size_t)((a + 1) & 1) * p.cnt_stride;
      for (uint32_t t = blockIdx.x * kB + threadIdx.x; t < p.ntiles; t += gridDim.x * kB) cout[t] = 0;
      return;
    }
    fast_round<kGrid, kReach>(p, S, gA, T, F, a, draws + before, L, nullptr, false,
                              p.xcount + a + 1);
  } else {
    fast_round<kGrid, kReach>(p, S, gA, T, F, a, p.draw_base, L, p.ctrl + place_total_word(a + 1),
                              false);
  }
  flush(p, L);
}

__global__ void __launch_bounds__(kB) k_fast_finish(PlaceParams p, int32_t a) {
  pdl_enter();
  const uint32_t* cin = p.tile_cnt + (size_t)(a & 1) * p.cnt_stride;
  for (uint32_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
    const uint32_t n = __ldcg(cin + t);
    const uint32_t* src = p.tile_list + (uint64_t)t * p.tile_inst;
    for (uint32_t e = threadIdx.x; e < n; e += kB) p.valid[src[e]] = 0;
  }
}

// ---------------------------------------------------------------- wide round 0
// The first attempt round of a FIFO placement carries every valid instance (C4: 262,144),
// and nearly all of them accept there. It runs as three grid-wide kernels with no CTA
// barrier between the phases and no grid barrier at all; the persistent kernel then takes
// the survivors from round 1 on (k_place with start_round = 1). Slot of a round-0 entry:
// tile * kB + position in the tile's (ascending) list, the tiles of k_fast_init.
constexpr uint8_t kWideDone = 8;  // accepted in k_wide_sample: no object overlaps its box
constexpr int kWideChunk = 0;  // narrow pairs a warp claims at a time; 0 = adaptive (1, or up to 4
                               // when every warp has > 64 pairs: C4 1/2/4/8 = 31.0/31.2/32.5/35.6
                               // ms, C5 x 100 1/4/8 = 342.7/334.3/336.0 ms)
static_assert(kWideRec == 6, "compact candidate record: tx, ty, tz, cos, sin, pad");

// A set of object ids < 32 * kW held in 64-bit registers with explicit members (no
// dynamically indexed array, which nvcc places in local memory).
template <int kW>
struct ObjSet {
  static constexpr int kQ = (kW + 1) / 2;  // 64-bit quads
  static_assert(kQ >= 1 && kQ <= 4, "at most 256 objects");
  unsigned long long q0 = 0, q1 = 0, q2 = 0, q3 = 0;
  __device__ __forceinline__ unsigned long long& quad(int k) {  // k compile-time after unrolling
    return k == 0 ? q0 : k == 1 ? q1 : k == 2 ? q2 : q3;
  }
  __device__ __forceinline__ unsigned long long quad_c(int k) const {
    return k == 0 ? q0 : k == 1 ? q1 : k == 2 ? q2 : q3;
  }
  __device__ __forceinline__ void or_word(int wd, uint32_t v) {  // wd compile-time
    quad(wd >> 1) |= (unsigned long long)v << (32 * (wd & 1));
  }
  __device__ __forceinline__ uint32_t word(int wd) const {  // wd compile-time
    return (uint32_t)(quad_c(wd >> 1) >> (32 * (wd & 1)));
  }
  __device__ __forceinline__ void set(int ob) {  // ob at run time: branches, no indexing
    const unsigned long long b = 1ull << (ob & 63);
    if (kQ == 1 || ob < 64) q0 |= b;
    else if (kQ == 2 || ob < 128) q1 |= b;
    else if (kQ == 3 || ob < 192) q2 |= b;
    else q3 |= b;
  }
  __device__ __forceinline__ int pop_lowest() {  // lowest id, removed; -1 when empty
    if (q0) { const int i = __ffsll(q0) - 1; q0 &= q0 - 1ull; return i; }
    if (kQ > 1 && q1) { const int i = __ffsll(q1) - 1; q1 &= q1 - 1ull; return 64 + i; }
    if (kQ > 2 && q2) { const int i = __ffsll(q2) - 1; q2 &= q2 - 1ull; return 128 + i; }
    if (kQ > 3 && q3) { const int i = __ffsll(q3) - 1; q3 &= q3 - 1ull; return 192 + i; }
    return -1;
  }
  __device__ __forceinline__ int count() const {
    return __popcll(q0) + (kQ > 1 ? __popcll(q1) : 0) + (kQ > 2 ? __popcll(q2) : 0) +
           (kQ > 3 ? __popcll(q3) : 0);
  }
};

// Exclusive prefix of the round-0 tile counts = each tile's first FIFO draw; resets the
// pair counters. One block of kWideScanThreads.
constexpr int kWideScanThreads = 1024;
// buf 0: round 0's counts (draw offsets, pair counters reset); buf 1: round 1's survivors
// (offsets for k_wide_spread, total S into w_ctl[5]).
// post = 0, before round a's sample: offsets of the round's actives (count buffer a & 1),
// pair counters reset, w_ctl[9] = D_a (draws before round a), w_ctl[4] = D_a + actives.
// post = 1, after its accept: offsets of the survivors (buffer (a + 1) & 1) for k_wide_spread,
// their total into w_ctl[5] (and w_surv[a] when the engine records it).
__global__ void __launch_bounds__(kWideScanThreads) k_wide_scan(PlaceParams p, int post) {
  pdl_enter();
  using Scan = cub::BlockScan<uint32_t, kWideScanThreads>;
  __shared__ typename Scan::TempStorage scan;
  const int32_t a = p.wide_round;
  const int buf = (a + post) & 1;
  uint32_t running = 0;
  for (uint32_t c0 = 0; c0 < p.ntiles; c0 += kWideScanThreads) {
    const uint32_t t = c0 + threadIdx.x;
    const uint32_t x = t < p.ntiles ? __ldcg(p.tile_cnt + (size_t)buf * p.cnt_stride + t) : 0u;
    uint32_t ex, agg;
    Scan(scan).ExclusiveSum(x, ex, agg);
    if (t < p.ntiles) p.w_toff[t] = running + ex;
    running += agg;
    __syncthreads();
  }
  if (!post) {
    if (threadIdx.x < 4) p.w_ctl[threadIdx.x] = 0ull;
    if (threadIdx.x == 0) {
      const unsigned long long d_a = a ? p.w_ctl[4] : 0ull;
      p.w_ctl[9] = d_a;
      p.w_ctl[4] = d_a + running;  // draws before round a + 1 (k_place: start_draws)
    }
  } else if (threadIdx.x == 0) {
    p.w_ctl[5] = running;  // round a + 1's active instances
    if (p.w_surv && a < kWideSurvRounds) p.w_surv[a] = running;
    if (p.xcount) p.xcount[1] = running;  // sharded: this rank's count for the exchange
  }
}

// Thread per round-0 entry: sample + compose (A1), candidate box, broad phase over the
// instance's enabled objects (the occupancy grid narrows them when kGrid). A candidate
// that overlaps no object is free (collision.cpp:439-448 finds nothing) and is accepted
// here; the others keep their pose / inverse / box / overlap bits in the slot scratch and
// append one (slot, object) pair per overlap, ascending objects, for k_wide_narrow.
template <bool kGrid, bool kReach, int kW>
__global__ void __launch_bounds__(kB, SB_WIDE_SAMPLE_MINB) k_wide_sample(PlaceParams p) {
  pdl_enter();
  static_assert(kW <= kGW && kGW % kW == 0, "enable words");
  constexpr int kWC = kW < 4 ? kW : 4;  // words of a cell loaded per batch
  const uint32_t t = blockIdx.x;
  const int e = threadIdx.x, lane = e & 31;
  const WorldView& w = p.w;
  const int32_t a = p.wide_round;  // this wide round's attempt (0, or later dense rounds)
  const uint32_t n = __ldcg(p.tile_cnt + (size_t)(a & 1) * p.cnt_stride + t);
  const uint64_t seed = p.seed_dev ? __ldg(p.seed_dev) : p.run_seed;
  const uint64_t state0 =
      p.seed_dev ? Pcg::seeded(stream_seed2(seed, p.pl.salt, kCacheSalt)).state : p.fast_state0;
  const Sampling S = resolve_sampling(p);
  const int words = w.n_words;
  // sharded (device exchange): round 0's draws start after the lower ranks' instances,
  // and round 1's draw offset is published as k_fast_round does for its rounds
  uint64_t draw_base = 0;
  if (p.xrecv) {
    unsigned long long tot = 0;
    for (int r = 0; r < p.xworld; ++r) {
      const unsigned long long v = __ldcg(p.xrecv + r);
      tot += v;
      if (r < p.xrank) draw_base += v;
    }
    draw_base += __ldcg(p.xdraws);
    if (t == 0 && threadIdx.x == 0) p.xdraws[1] = __ldcg(p.xdraws) + (S.n > 0 ? tot : 0ull);
  }
  Local L;
  ObjSet<kW> ov;
  uint32_t npairs = 0;
  const size_t slot = (size_t)t * kB + e;
  if (e < (int)n) {
    const uint32_t inst = __ldcg(p.tile_list + (uint64_t)t * p.tile_inst + e);
    M34 pose;
    double rec[6];
    // FIFO draw of round a: the draws of the earlier rounds (w_ctl[9]) + this entry's rank
    const uint64_t d_a = a ? __ldcg(p.w_ctl + 9) : 0ull;
    bool placeable = compose_candidate(p, S, seed, state0, inst, a,
                                       draw_base + d_a + (uint64_t)__ldcg(p.w_toff + t) + (uint64_t)e,
                                       pose, rec);
    if constexpr (kReach) {
      if (placeable) placeable = reach_ok(p, inst, pose);
    }
    ++L.sampled;
    uint8_t flag = kSlotUnplaceable;
    if (placeable) {
      ++L.checked;
      const SbGeom* gA = p.w.geoms + p.pl.geom;
      double box[6];
      {
        double c[3], h[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          c[k] = __ldg(gA->box_c + k);
          h[k] = __ldg(gA->box_h + k);
        }
        xform_aabb(pose, c, h, box, box + 3);
      }
      ObjSet<kW> cand;
      if constexpr (kGrid) {  // OR of the cells the candidate box meets, 4 cells' loads at once
        const SbCellGrid& G = p.grid;
        int cx0, cx1, cy0, cy1;
        cell_range(G, box, box + 3, cx0, cx1, cy0, cy1);
        const int ncell = (cx1 - cx0 + 1) * (cy1 - cy0 + 1);
        const uint32_t* cb = G.cells + (uint64_t)inst * (uint64_t)(G.g * G.g) * words;
        int wx = cx0, wy = cy0;  // cells walked row by row (no division per cell)
        for (int c0 = 0; c0 < ncell; c0 += 4) {
          const uint32_t* cp[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            cp[u] = cb + (uint64_t)(wy * G.g + wx) * words;
            if (++wx > cx1) {
              wx = cx0;
              ++wy;
            }
          }
          if (kW == 4 && words == 4) {  // a cell's 4 words in one 16-byte load
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              v[u] = c0 + u < ncell ? __ldcg(reinterpret_cast<const uint4*>(cp[u])) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              cand.or_word(0, v[u].x);
              cand.or_word(1, v[u].y);
              cand.or_word(2, v[u].z);
              cand.or_word(3, v[u].w);
            }
            continue;
          }
#pragma unroll
          for (int wg = 0; wg < kW; wg += kWC) {  // words [wg, wg + kWC) of 4 cells
            if (wg >= words) break;
            uint32_t v[4][kWC];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int j = 0; j < kWC; ++j)
                v[u][j] = (c0 + u < ncell && wg + j < words) ? __ldcg(cp[u] + wg + j) : 0u;
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int j = 0; j < kWC; ++j) cand.or_word(wg + j, v[u][j]);
          }
        }
      } else {  // every enabled object
#pragma unroll
        for (int wd = 0; wd < kW; ++wd)
          if (wd < words) cand.or_word(wd, __ldcg(w.enabled + sb_word_off(w, wd, inst)));
      }
      // AABB tests (aabb.hpp:29-33, margin 0), four box loads in flight. The next set bit is
      // found by a select chain over the (unrolled) words, so cand[] / ov[] stay in
      // registers (no dynamically indexed local arrays).
      {
        for (;;) {
          int obs[4];
          int k = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            obs[u] = cand.pop_lowest();
            k += obs[u] >= 0;
          }
          if (k == 0) break;
          double2 bx[4][3];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < k) {
              const double2* bp = reinterpret_cast<const double2*>(w.box + sb_box_off(w, obs[u], inst));
              bx[u][0] = __ldcg(bp);
              bx[u][1] = __ldcg(bp + 1);
              bx[u][2] = __ldcg(bp + 2);
            }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < k) {
              ++L.cnt.broad;
              const double2 a0 = bx[u][0], a1 = bx[u][1], a2 = bx[u][2];
              if (box[0] <= a1.y && a0.x <= box[3] && box[1] <= a2.x && a0.y <= box[4] &&
                  box[2] <= a2.y && a1.x <= box[5])
                ov.set(obs[u]);
            }
          if (k < 4) break;
        }
      }
      npairs = ov.count();
      if (npairs == 0) {  // free: accept now (the pose rebuilt from the record, bit-identical)
        M34 P;
        pose_from_rec(rec, P);
        double2 q[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) q[k] = make_double2(P.m[2 * k], P.m[2 * k + 1]);
        accept_candidate<kGrid>(p, inst, q, box, a);
        ++L.accepted;
        flag = kWideDone;
      } else {
        // only the compact record (translation, cos, sin: 48 B) is kept; the pose, its
        // inverse (k_wide_filter / k_wide_narrow) and the world box (k_wide_accept) are
        // recomputed from it with the same operations, bit for bit
        double2* cp = reinterpret_cast<double2*>(p.w_pose + slot * kWideRec);
#pragma unroll
        for (int k = 0; k < 3; ++k) cp[k] = make_double2(rec[2 * k], rec[2 * k + 1]);
        if (kW == 4 && words == 4) {
          *reinterpret_cast<uint4*>(p.w_ovm + slot * kGW) =
              make_uint4(ov.word(0), ov.word(1), ov.word(2), ov.word(3));
        } else {
#pragma unroll
          for (int wd = 0; wd < kW; ++wd)
            if (wd < words) p.w_ovm[slot * kGW + wd] = ov.word(wd);
        }
        p.w_contact[slot] = kFree;
        flag = kSlotChecked;
      }
    }
    p.w_flag[slot] = flag;
  }
  // warp-aggregated append of the pairs (slot << 8 | object), each entry's in ascending order
  uint32_t incl = npairs;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += y;
  }
  const uint32_t wtotal = __shfl_sync(kFull, incl, 31);
  unsigned long long base = 0;
  if (lane == 31 && wtotal) base = atomicAdd(p.w_ctl, (unsigned long long)wtotal);
  base = __shfl_sync(kFull, base, 31);
  if (npairs) {
    uint64_t q = base + incl - npairs;
#pragma unroll
    for (int ob = ov.pop_lowest(); ob >= 0; ob = ov.pop_lowest())
      p.w_pairs[q++] = ((uint32_t)slot << 8) | (uint32_t)ob;
  }
  if (threadIdx.x == 0 && n) atomicMax(p.ctrl + kRounds, (uint32_t)(a + 1));  // reference rounds
  flush(p, L);
}

// Thread per (slot, object) pair: the leaf-box filter of the narrow phase (warp_collide
// step 2) on its own. other_in_cand = inv(cand) * pose(ob) and B's leaf boxes moved into
// A's frame are computed with the very operations warp_collide uses, so "no leaf pair's
// boxes overlap" here is exactly the case in which warp_collide returns false at step 2
// -- such pairs never reach k_wide_narrow. Survivors are appended to the second list.
// Pairs behind a lower hit of their slot cannot matter and are dropped as well.
__global__ void __launch_bounds__(kB) k_wide_filter(PlaceParams p) {
  pdl_enter();
  __shared__ PlaceGeomCache gc;
  const WorldView& w = p.w;
  const int lane = threadIdx.x & 31;
  load_geom_cache(w, p.w.geoms[p.pl.geom], gc);
  __syncthreads();
  const uint64_t np = __ldcg(p.w_ctl);
  Local L;
  for (uint64_t q0 = (uint64_t)blockIdx.x * kB; q0 < np; q0 += (uint64_t)gridDim.x * kB) {
    const uint64_t q = q0 + threadIdx.x;
    bool pass = false;
    uint32_t ent = 0, inst = 0;
    if (q < np) {
      ent = __ldcg(p.w_pairs + q);
      const uint32_t sl = ent >> 8;
      const int32_t ob = (int32_t)(ent & 0xffu);
      if (*((volatile int32_t*)p.w_contact + sl) >= ob) {
        inst = __ldcg(p.tile_list + (uint64_t)(sl / kB) * p.tile_inst + sl % kB);
        pass = leaf_filter<true>(w, gc, p.w_pose + (size_t)sl * kWideRec, w.pose + sb_pose_off(w, ob, inst),
                                 obj_grec(w, ob));
      }
    }
    // warp-aggregated append of the survivors (order within the list is free: the narrow
    // verdict is a min over objects)
    const uint32_t m = __ballot_sync(kFull, pass);
    unsigned long long base = 0;
    if (lane == 0 && m) base = atomicAdd(p.w_ctl + 2, (unsigned long long)__popc(m));
    base = __shfl_sync(kFull, base, 0);
    if (pass) {
      const unsigned long long k = base + __popc(m & ((1u << lane) - 1u));
      p.w_pairs2[k] = ent;
      p.w_pinst2[k] = inst;
    }
  }
  flush(p, L);
}

// Warp per (slot, object) pair over the whole grid: the exact narrow phase (sb_warp.cuh)
// with the pair's pose + geometry record staged one pair ahead; a pair behind a lower
// hit of its slot is skipped (the reference stops at the first colliding object).
// kBulk: pairs staged by cp.async.bulk + an mbarrier per staging buffer (one lane issues
// three copies) instead of per-lane 16-byte cp.async (default; SB_BULK_STAGE=0 for the
// cp.async variant; DESIGN 3.3).
template <bool kBulk, int kMinB = SB_WIDE_NARROW_MINB>
__global__ void __launch_bounds__(kB, kMinB) k_wide_narrow(PlaceParams p, int chunk, int claim_ahead) {
  pdl_enter();
  __shared__ PlaceGeomCache gc;
  __shared__ __align__(8) uint64_t bars[kWarps][2];
  __shared__ int4 ogeo[kGW * 32];  // obj_grec of every object (no dependent load per pair)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const WorldView& w = p.w;
  load_geom_cache(w, p.w.geoms[p.pl.geom], gc);
  for (int ob = threadIdx.x; ob < w.n_objects; ob += kB) ogeo[ob] = obj_grec(w, ob);
  if constexpr (kBulk) {
    if (lane == 0) {
      mbar_init(&bars[warp][0], 1);
      mbar_init(&bars[warp][1], 1);
      mbar_init_fence();
    }
  }
  unsigned phase_bits = 0u;  // bit b: the parity staging buffer b's barrier completes next
  __syncthreads();
  unsigned char* wsb = g_dsm + warp * p.ws_bytes;
  const WarpScratchView ws = carve_scratch(wsb, p.max_tris, p.max_nodes);
  const uint64_t np = __ldcg(p.w_ctl + 2);  // pairs past k_wide_filter
  Local L;
  auto skippable = [&](uint32_t ent) {
    return *((volatile int32_t*)p.w_contact + (ent >> 8)) < (int32_t)(ent & 0xffu);
  };
  auto stage = [&](uint64_t q, int buf) {  // pair q's records into staging buffer `buf`
    const uint32_t ent = __ldcg(p.w_pairs2 + q), inst = __ldcg(p.w_pinst2 + q);
    const uint32_t sl = ent >> 8, ob = ent & 0xffu;
    if constexpr (kBulk)
      warp_stage_bulk(w, ogeo[ob], (int32_t)ob, inst, p.w_pose + (size_t)sl * kWideRec,
                      8u * kWideRec, stage_buf(wsb, p.max_tris, p.max_nodes, buf), &bars[warp][buf]);
    else
      warp_stage(w, ogeo[ob], (int32_t)ob, inst, p.w_pose + (size_t)sl * kWideRec,
                 stage_buf(wsb, p.max_tris, p.max_nodes, buf), 3);  // candidate RECORD at +96
  };
  auto wait_stage = [&](int buf, int pending) {  // buffer `buf` staged and visible
    if constexpr (kBulk) {
      while (!mbar_try_wait(&bars[warp][buf], (phase_bits >> buf) & 1u)) {
      }
      phase_bits ^= 1u << buf;
    } else {
      if (pending) cp_async_wait<1>();
      else cp_async_wait<0>();
    }
  };
  // One continuous stream of pairs per warp: chunks of kWideChunk claimed dynamically, the
  // next chunk claimed one chunk ahead (lane 0's atomic is only waited for at the chunk
  // boundary), so staging stays one pair ahead across chunk boundaries.
  constexpr uint64_t kEnd = ~0ull;
  // chunk 0 = adaptive: one pair per claim unless every warp has > 64 pairs on average
  // (dense launches: larger chunks keep the claim counter from becoming the bottleneck)
  unsigned long long ck = (unsigned long long)chunk;
  if (chunk == 0) {
    const unsigned long long per_warp = np / ((unsigned long long)gridDim.x * kWarps);
    ck = per_warp > 64 ? (per_warp / 64 < 4 ? per_warp / 64 : 4) : 1;
  }
  unsigned long long ahead = 0;  // lane 0: start of the chunk claimed ahead (in flight)
  if (lane == 0 && claim_ahead) ahead = atomicAdd(p.w_ctl + 3, ck);
  uint64_t qe = 0;  // end of the current chunk
  auto advance = [&](uint64_t q) -> uint64_t {  // next non-skippable pair at or after q
    for (;;) {
      while (q < qe && skippable(__ldcg(p.w_pairs2 + q))) ++q;
      if (q < qe) return q;
      if (lane == 0 && !claim_ahead) ahead = atomicAdd(p.w_ctl + 3, ck);
      const unsigned long long c = __shfl_sync(kFull, ahead, 0);
      if (c >= np) return kEnd;
      if (lane == 0 && claim_ahead) ahead = atomicAdd(p.w_ctl + 3, ck);
      q = c;
      qe = c + ck < np ? c + ck : np;
    }
  };
  int cur = 0;
  uint64_t q = advance(0);
  if (q != kEnd) stage(q, cur);
  while (q != kEnd) {
    const uint32_t ent = __ldcg(p.w_pairs2 + q);
    const uint64_t q2 = advance(q + 1);
    if (q2 != kEnd) stage(q2, cur ^ 1);
    wait_stage(cur, q2 != kEnd);
    __syncwarp();
    if (__shfl_sync(kFull, (int)!skippable(ent), 0)) {  // one verdict for the whole warp
      const int32_t ob = (int32_t)(ent & 0xffu);
      const int4 gr = ogeo[ob];
      unsigned char* st = stage_buf(wsb, p.max_tris, p.max_nodes, cur);
      {  // the staged record -> the candidate's inverse pose, lane per entry
        double* R = reinterpret_cast<double*>(st + 96);
        double v = 0.0;
        if (lane < 12) {
          double rec[6];
#pragma unroll
          for (int k = 0; k < 6; ++k) rec[k] = R[k];
          M34 C, Ci;
          pose_from_rec(rec, C);
          inverse_rigid(C, Ci);
          v = Ci.m[0];
#pragma unroll
          for (int k = 1; k < 12; ++k)
            if (lane == k) v = Ci.m[k];
        }
        __syncwarp();
        if (lane < 12) R[lane] = v;
        __syncwarp();
      }
      const bool hit = warp_collide(gc, st, gr.z, gr.w, ws, L.cnt);
      if (hit && lane == 0) atomicMin(p.w_contact + (ent >> 8), ob);
    }
    __syncwarp();
    q = q2;
    cur ^= 1;
  }
  flush(p, L);
}

// Thread per round-0 entry: first-valid accept of the slots that had pairs (contact still
// free), the reference's narrow-test count up to the first hit, and the survivors
// compacted in place into the tile's list with round 1's count (tile_cnt buffer 1).
template <bool kGrid>
__global__ void __launch_bounds__(kB) k_wide_accept(PlaceParams p) {
  pdl_enter();
  __shared__ typename BlockScan::TempStorage scan;
  const uint32_t t = blockIdx.x;
  const int e = threadIdx.x;
  const int32_t a = p.wide_round;
  const uint32_t n = __ldcg(p.tile_cnt + (size_t)(a & 1) * p.cnt_stride + t);
  const int words = p.w.n_words;
  Local L;
  uint32_t keep = 0, inst = 0;
  if (e < (int)n) {
    const size_t slot = (size_t)t * kB + e;
    inst = __ldcg(p.tile_list + (uint64_t)t * p.tile_inst + e);
    const uint8_t flag = __ldcg(p.w_flag + slot);
    if (flag == kSlotUnplaceable) {
      keep = 1;
    } else if (flag == kSlotChecked) {
      const int32_t c = __ldcg(p.w_contact + slot);
      uint4 m4 = make_uint4(0, 0, 0, 0);
      if (words == 4) m4 = __ldcg(reinterpret_cast<const uint4*>(p.w_ovm + slot * kGW));
      for (int wd = 0; wd < words; ++wd) {  // narrow tests up to the first hit
        uint32_t mk = words == 4 ? (wd == 0 ? m4.x : wd == 1 ? m4.y : wd == 2 ? m4.z : m4.w)
                                 : __ldcg(p.w_ovm + slot * kGW + wd);
        if (c != kFree) {
          const int lim = c - 32 * wd;  // keep objects <= c
          if (lim < 0) mk = 0;
          else if (lim < 31) mk &= (2u << lim) - 1u;
        }
        L.cnt.narrow += __popc(mk);
      }
      if (c == kFree) {
        double2 q[6];
        double box[6];
        {  // the candidate's pose and world box, as k_wide_sample computed them
          double rec[6];
          load_rec(p.w_pose + slot * kWideRec, rec);
          M34 pose;
          pose_from_rec(rec, pose);
#pragma unroll
          for (int k = 0; k < 6; ++k) q[k] = make_double2(pose.m[2 * k], pose.m[2 * k + 1]);
          const SbGeom* gA = p.w.geoms + p.pl.geom;
          double c[3], h[3];
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            c[k] = __ldg(gA->box_c + k);
            h[k] = __ldg(gA->box_h + k);
          }
          xform_aabb(pose, c, h, box, box + 3);
        }
        accept_candidate<kGrid>(p, inst, q, box, a);
        ++L.accepted;
      } else {
        keep = 1;
      }
    }
  }
  uint32_t rank, total;
  BlockScan(scan).ExclusiveSum(keep, rank, total);
  __syncthreads();  // every entry of the list has been read
  if (keep) p.tile_list[(uint64_t)t * p.tile_inst + rank] = inst;
  if (e == 0) p.tile_cnt[(size_t)((a + 1) & 1) * p.cnt_stride + t] = total;
  flush(p, L);
}

// Round 1's survivors (S, ascending in tile order) re-dealt over `gridDim` tiles of
// q = min(ceil(S / min(grid, ntiles)), tile_inst) consecutive entries each, so every CTA of the persistent kernel
// gets a share (rounds >= 1 are few instances; one CTA's narrow phase is serial per warp):
// survivor of old tile t at position e has global rank toff[t] + e and goes to tile
// rank / q, entry rank % q (tile_list2, tile_cnt2 buffer 1). Block per old tile; the
// counts of all new tiles are written by a grid-stride loop.
__global__ void __launch_bounds__(kB) k_wide_spread(PlaceParams p, unsigned grid) {
  pdl_enter();
  const unsigned long long S = __ldcg(p.w_ctl + 5);
  if (grid > p.ntiles) grid = p.ntiles;  // S / q tiles must exist
  unsigned long long q = S ? (S + grid - 1) / grid : 1;  // at most one tile's capacity
  if (q > (unsigned long long)p.tile_inst) q = p.tile_inst;
  const uint32_t t = blockIdx.x;
  const size_t ob = (size_t)((p.wide_round + 1) & 1) * p.cnt_stride;  // the survivors' buffer
  const uint32_t n = __ldcg(p.tile_cnt + ob + t);
  const unsigned long long off = __ldcg(p.w_toff + t);
  for (uint32_t e = threadIdx.x; e < n; e += kB) {
    const unsigned long long r = off + e;
    p.w_list2[(r / q) * p.tile_inst + r % q] = __ldcg(p.tile_list + (uint64_t)t * p.tile_inst + e);
  }
  for (uint32_t k = blockIdx.x * kB + threadIdx.x; k < p.ntiles; k += gridDim.x * kB) {
    const unsigned long long lo = (unsigned long long)k * q;
    p.w_cnt2[ob + k] = S > lo ? (uint32_t)(S - lo < q ? S - lo : q) : 0u;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) p.w_ctl[6] = (S + q - 1) / q;  // tiles in use
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

void set_smem(const void* fn, size_t smem) {
  check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
        "cudaFuncSetAttribute(smem)");
}


}  // namespace

int place_ws_bytes(int max_tris, int max_nodes) { return warp_scratch_bytes(max_tris, max_nodes); }

size_t place_smem_bytes(int n_words, int ws_bytes, int n_objects) {
  return tile_bytes(n_words) + (size_t)kWarps * ws_bytes + 16 * (size_t)n_objects;
}

void narrow_profile(unsigned long long out[8], bool reset) {
  check(cudaMemcpyFromSymbol(out, g_nprof, 8 * sizeof(unsigned long long)), "narrow_profile");
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    check(cudaMemcpyToSymbol(g_nprof, z, sizeof z), "narrow_profile reset");
  }
}

namespace {
// kernel variant by (occupancy grid, fused reachability filter)
const void* place_fn(const PlaceParams& p, bool one = false) {
  const bool g = p.grid.g != 0, r = p.reach_any != nullptr;
  if (one)
    return g ? (r ? (const void*)k_place<true, true, 1> : (const void*)k_place<true, false, 1>)
             : (r ? (const void*)k_place<false, true, 1> : (const void*)k_place<false, false, 1>);
  return g ? (r ? (const void*)k_place<true, true> : (const void*)k_place<true, false>)
           : (r ? (const void*)k_place<false, true> : (const void*)k_place<false, false>);
}
}  // namespace

int place_grid(int num_sms, size_t smem, bool one) {
  const void* fns[4] = {place_fn(PlaceParams{}, one), nullptr, nullptr, nullptr};
  {
    PlaceParams q = {};
    q.grid.g = 1;
    fns[1] = place_fn(q, one);
    q.reach_any = reinterpret_cast<const unsigned long long*>(1);
    fns[3] = place_fn(q, one);
    q.grid.g = 0;
    fns[2] = place_fn(q, one);
  }
  int per = 1 << 30;
  for (const void* fn : fns) {
    set_smem(fn, smem);
    int v = 0;
    check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, fn, kB, smem), "occupancy");
    if (v < per) per = v;
  }
  return per * num_sms;
}

bool place_persistent(const PlaceParams& p, unsigned grid, size_t smem, sb_stream_t s, bool one) {
  if (grid == 0) return false;
  PlaceParams q = p;
  void* args[] = {&q};
  static const bool pdl = [] {  // SB_PDL_COOP=0: plain cooperative launch
    const char* e = std::getenv("SB_PDL_COOP");
    return pdl_on() && (!e || std::atoi(e) != 0);
  }();
  if (!pdl) {
    check(cudaLaunchCooperativeKernel(place_fn(p, one), dim3(grid), dim3(kB), args, smem,
                                      reinterpret_cast<cudaStream_t>(s)),
          "cudaLaunchCooperativeKernel(k_place)");
    return true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kB);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = reinterpret_cast<cudaStream_t>(s);
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  check(cudaLaunchKernelExC(&cfg, place_fn(p, one), args), "cudaLaunchKernelEx(k_place, cooperative)");
  return true;
}

template <bool kGrid, bool kReach>
void launch_instances(const PlaceParams& p, unsigned grid, size_t smem, sb_stream_t s) {
  set_smem((const void*)k_place_instances<kGrid, kReach>, smem);
  launch_pdl(k_place_instances<kGrid, kReach>, grid, kB, smem, reinterpret_cast<cudaStream_t>(s), p);
}

void place_instances(const PlaceParams& p, unsigned grid, size_t smem, sb_stream_t s) {
  const bool r = p.reach_any != nullptr;
  if (p.grid.g) r ? launch_instances<true, true>(p, grid, smem, s) : launch_instances<true, false>(p, grid, smem, s);
  else r ? launch_instances<false, true>(p, grid, smem, s) : launch_instances<false, false>(p, grid, smem, s);
  check(cudaGetLastError(), "k_place_instances");
}

void place_fast_init(const PlaceParams& p, unsigned grid, size_t smem, sb_stream_t s) {
  set_smem((const void*)k_fast_init, smem);
  launch_pdl(k_fast_init, grid, kB, smem, reinterpret_cast<cudaStream_t>(s), p);
  check(cudaGetLastError(), "k_fast_init");
}

template <bool kGrid, bool kReach>
void launch_fast_round(const PlaceParams& p, int32_t attempt, unsigned grid, size_t smem,
                       sb_stream_t s) {
  set_smem((const void*)k_fast_round<kGrid, kReach>, smem);
  launch_pdl(k_fast_round<kGrid, kReach>, grid, kB, smem, reinterpret_cast<cudaStream_t>(s), p, attempt);
}

void place_fast_round(const PlaceParams& p, int32_t attempt, unsigned grid, size_t smem,
                      sb_stream_t s) {
  const bool r = p.reach_any != nullptr;
  if (p.grid.g) r ? launch_fast_round<true, true>(p, attempt, grid, smem, s) : launch_fast_round<true, false>(p, attempt, grid, smem, s);
  else r ? launch_fast_round<false, true>(p, attempt, grid, smem, s) : launch_fast_round<false, false>(p, attempt, grid, smem, s);
  check(cudaGetLastError(), "k_fast_round");
}

template <bool kGrid, bool kReach>
void launch_wide_sample(const PlaceParams& p, int nw, cudaStream_t st) {
  if (nw <= 1) launch_pdl(k_wide_sample<kGrid, kReach, 1>, p.ntiles, kB, 0, st, p);
  else if (nw <= 2) launch_pdl(k_wide_sample<kGrid, kReach, 2>, p.ntiles, kB, 0, st, p);
  else if (nw <= 4) launch_pdl(k_wide_sample<kGrid, kReach, 4>, p.ntiles, kB, 0, st, p);
  else launch_pdl(k_wide_sample<kGrid, kReach, kGW>, p.ntiles, kB, 0, st, p);
}

size_t wide_narrow_smem(int ws_bytes) { return (size_t)kWarps * ws_bytes; }

int place_wide_round0(const PlaceParams& p, unsigned init_grid, size_t init_smem, int num_sms,
                      sb_stream_t s, unsigned spread_grid) {
  place_fast_init(p, init_grid, init_smem, s);
  return 1 + place_wide_round0_rest(p, init_grid, num_sms, s, spread_grid, true);
}

int place_wide_round0_a(const PlaceParams& p, int num_sms, sb_stream_t s) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
  launch_pdl(k_wide_scan, 1, kWideScanThreads, 0, st, p, 0);
  check(cudaGetLastError(), "k_wide_scan");
  const bool g = p.grid.g != 0, r = p.reach_any != nullptr;
  // register footprint sized by the enable words in use (cand / ov stay in registers)
  const int nw = p.w.n_words;
  if (g) r ? launch_wide_sample<true, true>(p, nw, st) : launch_wide_sample<true, false>(p, nw, st);
  else r ? launch_wide_sample<false, true>(p, nw, st) : launch_wide_sample<false, false>(p, nw, st);
  check(cudaGetLastError(), "k_wide_sample");
  {
    int per = 0;
    check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, (const void*)k_wide_filter, kB, 0), "occupancy");
    launch_pdl(k_wide_filter, (unsigned)(per > 0 ? per : 1) * num_sms, kB, 0, st, p);
    check(cudaGetLastError(), "k_wide_filter");
  }
  const size_t smem = wide_narrow_smem(p.ws_bytes);
  static const bool bulk = [] {  // measured: C4 37.41 -> 37.28 ms (SB_BULK_STAGE=0: cp.async)
    const char* e = std::getenv("SB_BULK_STAGE");
    return !e || std::atoi(e) != 0;
  }();
  static const int minb = [] {  // experiment: SB_NARROW_MINB=4 (64-register cap)
    const char* e = std::getenv("SB_NARROW_MINB");
    return e && std::atoi(e) == 4 ? 4 : SB_WIDE_NARROW_MINB;
  }();
  const void* nfn = !bulk ? (const void*)k_wide_narrow<false>
                    : minb == 4 ? (const void*)k_wide_narrow<true, 4> : (const void*)k_wide_narrow<true>;
  set_smem(nfn, smem);
  int per = 0;
  check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, nfn, kB, smem), "occupancy");
  const unsigned ngrid = (unsigned)(per > 0 ? per : 1) * num_sms;
  static const int chunk = [] {  // pairs a warp claims at a time (SB_NARROW_CHUNK)
    const char* e = std::getenv("SB_NARROW_CHUNK");
    return e && std::atoi(e) >= 0 ? std::atoi(e) : kWideChunk;
  }();
  static const int ahead = [] {  // claim the next chunk one chunk ahead (SB_NARROW_AHEAD)
    const char* e = std::getenv("SB_NARROW_AHEAD");
    return e ? std::atoi(e) : 0;
  }();
  if (!bulk) launch_pdl(k_wide_narrow<false>, ngrid, kB, smem, st, p, chunk, ahead);
  else if (minb == 4) launch_pdl(k_wide_narrow<true, 4>, ngrid, kB, smem, st, p, chunk, ahead);
  else launch_pdl(k_wide_narrow<true>, ngrid, kB, smem, st, p, chunk, ahead);
  check(cudaGetLastError(), "k_wide_narrow");
  return 4;
}

int place_wide_round0_c(const PlaceParams& p, unsigned init_grid, sb_stream_t s,
                        unsigned spread_grid, bool spread) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
  const bool g = p.grid.g != 0;
  if (g) launch_pdl(k_wide_accept<true>, p.ntiles, kB, 0, st, p);
  else launch_pdl(k_wide_accept<false>, p.ntiles, kB, 0, st, p);
  check(cudaGetLastError(), "k_wide_accept");
  launch_pdl(k_wide_scan, 1, kWideScanThreads, 0, st, p, 1);
  check(cudaGetLastError(), "k_wide_scan");
  if (!spread) return 2;  // sharded: rounds >= 1 read the compacted tiles in place
  // round 1's survivors over the persistent kernel's grid (SB_SPREAD=0: full tiles instead)
  unsigned sg = spread_grid ? spread_grid : init_grid;
  if (const char* e = std::getenv("SB_SPREAD")) sg = std::atoi(e) ? sg : 1u;
  launch_pdl(k_wide_spread, p.ntiles, kB, 0, st, p, sg);
  check(cudaGetLastError(), "k_wide_spread");
  return 3;
}

int place_wide_round0_rest(const PlaceParams& p, unsigned init_grid, int num_sms, sb_stream_t s,
                           unsigned spread_grid, bool spread) {
  return place_wide_round0_a(p, num_sms, s) + place_wide_round0_c(p, init_grid, s, spread_grid, spread);
}

void place_fast_finish(const PlaceParams& p, int32_t attempt, unsigned grid, sb_stream_t s) {
  launch_pdl(k_fast_finish, grid, kB, 0, reinterpret_cast<cudaStream_t>(s), p, attempt);
  check(cudaGetLastError(), "k_fast_finish");
}

}  // namespace sbk
