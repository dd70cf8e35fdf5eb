// Phased placement engine (see sb_place.h). sm_100a, -fmad=false.
#include <cooperative_groups.h>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <climits>
#include <stdexcept>
#include <string>

#include "../../include/scenebatch_b200.h"
#include "sb_crmath.cuh"
#include "sb_dev.cuh"
#include "sb_place.h"
#include "sb_poly.h"
#include "sb_warp.cuh"

namespace cg = cooperative_groups;
using namespace sbd;

namespace sbk {
namespace {

constexpr int kB = kPlaceBlock;
constexpr int kWarps = kB / 32;
constexpr int32_t kFree = INT32_MAX;
constexpr uint8_t kSlotVoid = 0, kSlotChecked = 1, kSlotUnplaceable = 2;

enum Ctrl { kM = 0, kPairs = 1, kRounds = 2, kErr = 3, kCur = 4 };

// Phase A tile (one slot per thread) and phase B warp scratch share the same bytes.
struct TileA {
  double box[kB][6];   // candidate world AABB per slot of the tile
  uint32_t inst[kB];
  uint8_t ok[kB];      // slot holds a placeable candidate
};
struct Shared {
  union {
    WarpScratch ws[kWarps];
    TileA ta;
  } u;
  GeomCache gc;
};

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

__device__ __forceinline__ uint32_t* act_list(const PlaceParams& p, int which) {
  return which ? p.act1 : p.act0;
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

// Attempts evaluated per remaining instance this round (1 on the FIFO fast path).
__device__ __forceinline__ int spec_width(const PlaceParams& p, int fast, uint64_t m,
                                          int32_t attempt) {
  if (fast || m == 0) return 1;
  uint64_t w = p.spec_budget / m;
  const uint64_t cap = p.slot_cap / m;
  if (w > cap) w = cap;
  if (w > (uint64_t)(p.attempts - attempt)) w = (uint64_t)(p.attempts - attempt);
  return w < 1 ? 1 : (int)w;
}

// ------------------------------------------------------------------ compaction
// Stable compaction in chunks of kB entries: count pass, then (after a grid barrier) a
// scatter pass that derives each chunk's output offset from the chunk counts.
template <class Flag>
__device__ void compact_count(const PlaceParams& p, uint64_t m, Flag flag) {
  const uint64_t nc = (m + kB - 1) / kB;
  for (uint64_t ch = blockIdx.x; ch < nc; ch += gridDim.x) {
    const uint64_t e = ch * kB + threadIdx.x;
    const int f = e < m ? flag(e) : 0;
    const int c = __syncthreads_count(f);
    if (threadIdx.x == 0) p.chunk_cnt[ch] = (uint32_t)c;
  }
}

template <class Flag, class Src>
__device__ void compact_scatter(const PlaceParams& p, uint64_t m, Flag flag, Src src,
                                uint32_t* dst) {
  using BR = cub::BlockReduce<uint32_t, kB>;
  using BS = cub::BlockScan<uint32_t, kB>;
  __shared__ union {
    typename BR::TempStorage r;
    typename BS::TempStorage s;
  } tmp;
  __shared__ uint32_t s_off;
  const uint64_t nc = (m + kB - 1) / kB;
  uint64_t done = 0;  // chunks [0, done) already summed into off
  uint32_t off = 0;
  for (uint64_t ch = blockIdx.x; ch < nc; ch += gridDim.x) {
    uint32_t part = 0;
    for (uint64_t c = done + threadIdx.x; c < ch; c += kB) part += __ldcg(p.chunk_cnt + c);
    uint32_t sum = BR(tmp.r).Sum(part);
    if (threadIdx.x == 0) s_off = off + sum;
    __syncthreads();
    off = s_off;
    done = ch;
    const uint64_t e = ch * kB + threadIdx.x;
    const uint32_t f = e < m ? (uint32_t)flag(e) : 0u;
    uint32_t rank;
    BS(tmp.s).ExclusiveSum(f, rank);
    if (f) dst[off + rank] = src(e);
    __syncthreads();
  }
  if (blockIdx.x == 0) {  // total -> next M
    uint32_t part = 0;
    for (uint64_t c = threadIdx.x; c < nc; c += kB) part += __ldcg(p.chunk_cnt + c);
    uint32_t sum = BR(tmp.r).Sum(part);
    if (threadIdx.x == 0) p.ctrl[kM] = sum;
  }
}

// ------------------------------------------------------------------ phase A
// Tiles of kB virtual slots per block; slot v = e * W + s is instance act[e] at attempt
// `attempt + s`.
// A1 (thread per slot): sample -> yaw -> compose -> candidate AABB + inverse; pose and
//    inverse to global, AABB to shared memory.
// A2 (thread per (slot, object) item): AABB broad phase (collision.cpp:439-443) over the
//    enabled objects; consecutive threads read consecutive object records of one instance
//    (instance-major layout), so the loads are contiguous and independent. Overlaps set
//    the slot's ovmask bit and append (slot, object) to the pair queue.
__device__ void phase_a(const PlaceParams& p, const Sampling& S, const SbGeom& gA,
                        Shared& sh, const uint32_t* act, uint64_t m, int W,
                        uint64_t draw_base, int32_t attempt, Local& L) {
  const int lane = threadIdx.x & 31;
  const SbPlacementDev& pl = p.pl;
  const WorldView& w = p.w;
  TileA& ta = sh.u.ta;
  const uint64_t nslots = m * (uint64_t)W;
  const int nobj = w.n_objects;
  // tile size: kB slots, or fewer so that small rounds still spread over every block
  uint64_t T = (nslots + gridDim.x - 1) / gridDim.x;
  T = T < 32 ? 32 : ((T + 31) / 32) * 32;
  if (T > (uint64_t)kB) T = kB;
  for (uint64_t t0 = (uint64_t)blockIdx.x * T; t0 < nslots; t0 += (uint64_t)gridDim.x * T) {
    // ---------------- A1
    const uint64_t v = t0 + threadIdx.x;
    bool ok = false;
    uint32_t inst = 0;
    if (threadIdx.x < T && v < nslots) {
      const uint64_t e = v / W;
      const int32_t at = attempt + (int32_t)(v - e * W);
      inst = act[e];
      const uint64_t gid = p.global_begin + inst;
      bool placeable = true;
      double lx = 0.0, ly = 0.0;
      if (S.fast) {
        if (S.n == 0) {
          placeable = false;
        } else {
          Pcg r{p.fast_state0};
          r.advance(6ull * (draw_base + e));  // j-th drained point = j-th draw (sampler.cpp:30-43)
          double u = r.next_double(), r1 = r.next_double(), r2 = r.next_double();
          sbp::draw_point(S.tris, S.cum, S.n, u, r1, r2, lx, ly);
        }
      } else {
        const int nt = p.inst_n[inst];
        if (nt == 0) {
          placeable = false;
        } else {  // make_stream(run_seed, {salt, "fall", inst, attempt}) (sampler.cpp:117)
          Pcg r = Pcg::seeded(stream_seed4(p.run_seed, pl.salt, kFallbackSalt, gid,
                                           static_cast<uint64_t>(at)));
          double u = r.next_double(), r1 = r.next_double(), r2 = r.next_double();
          const uint64_t off = (uint64_t)inst * p.inst_cap;
          sbp::draw_point(p.inst_tris + off, p.inst_cum + off, nt, u, r1, r2, lx, ly);
        }
      }
      p.contact[v] = kFree;
      for (int wd = 0; wd < w.n_words; ++wd) p.ovmask[(uint64_t)wd * p.slot_cap + v] = 0u;
      if (!placeable) {
        p.cflag[v] = kSlotUnplaceable;
      } else {
        M34 Sp;
#pragma unroll
        for (int k = 0; k < 12; ++k) Sp.m[k] = pl.support[k];
        double px, py, pz;
        xform(Sp, lx, ly, 0.0, px, py, pz);  // transform_point(support_world, (x, y, 0))
        double yaw = 0.0;
        if (pl.orientation == SB_ORIENT_UNIFORM_YAW) {  // sampler.cpp:140-141
          Pcg r = Pcg::seeded(
              stream_seed4(p.run_seed, pl.salt, kYawSalt, gid, static_cast<uint64_t>(at)));
          const double two_pi = 2.0 * 3.14159265358979323846;
          yaw = 0.0 + (two_pi - 0.0) * r.next_double();
        } else if (pl.orientation == SB_ORIENT_FACE_TO) {  // relationships.cpp:232-239
          const double* tp = w.pose + sb_pose_off(w, pl.face_object, inst);
          double dx = tp[3] - px, dy = tp[7] - py;
          yaw = sqrt(dx * dx + dy * dy) < 1e-12 ? 0.0 : sbm::atan2_cr(dy, dx);
        }
        double c, s;
        sbm::sincos_cr(yaw, &s, &c);  // rotation_z: std::cos / std::sin (transform.hpp:47)
        M34 T, Rz, pose;  // translation(p + z_off z) * rotation_z(yaw)
#pragma unroll
        for (int k = 0; k < 12; ++k) T.m[k] = Rz.m[k] = 0.0;
        T.m[0] = T.m[5] = T.m[10] = 1.0;
        Rz.m[10] = 1.0;
        T.m[3] = px + 0.0;
        T.m[7] = py + 0.0;
        T.m[11] = pz + pl.z_off;
        Rz.m[0] = c;
        Rz.m[1] = -s;
        Rz.m[4] = s;
        Rz.m[5] = c;
        mul34(T, Rz, pose);
        double cmn[3], cmx[3];
        xform_aabb(pose, gA.box_c, gA.box_h, cmn, cmx);
        M34 inv;
        inverse_rigid(pose, inv);
        double2* cp = reinterpret_cast<double2*>(p.cpose + v * 12);
        double2* ci = reinterpret_cast<double2*>(p.cinv + v * 12);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          cp[k] = make_double2(pose.m[2 * k], pose.m[2 * k + 1]);
          ci[k] = make_double2(inv.m[2 * k], inv.m[2 * k + 1]);
        }
        p.cflag[v] = kSlotChecked;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          ta.box[threadIdx.x][k] = cmn[k];
          ta.box[threadIdx.x][3 + k] = cmx[k];
        }
        ok = true;
      }
    }
    ta.inst[threadIdx.x] = inst;
    ta.ok[threadIdx.x] = ok ? 1 : 0;
    __syncthreads();
    // ---------------- A2 (4 items per thread in flight: loads first, then ballots)
    const uint64_t tile_n = (nslots - t0) < T ? (nslots - t0) : T;
    const uint64_t items = tile_n * (uint64_t)nobj;
    constexpr int U = 4;
    for (uint64_t it0 = 0; it0 < items; it0 += (uint64_t)kB * U) {
      bool ov[U];
      uint32_t tt[U];
      int obs[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t it = it0 + (uint64_t)u * kB + threadIdx.x;
        ov[u] = false;
        tt[u] = 0;
        obs[u] = 0;
        if (it < items) {
          const uint32_t t = (uint32_t)(it / nobj);
          const int ob = (int)(it - (uint64_t)t * nobj);
          tt[u] = t;
          obs[u] = ob;
          if (ta.ok[t]) {
            const uint32_t in = ta.inst[t];
            const uint32_t bits = w.enabled[sb_word_off(w, ob >> 5, in)];
            if ((bits >> (ob & 31)) & 1u) {
              ++L.cnt.broad;
              const double2* bp =
                  reinterpret_cast<const double2*>(w.box + sb_box_off(w, ob, in));
              const double2 b0 = bp[0], b1 = bp[1], b2 = bp[2];
              const double* cb = ta.box[t];
              ov[u] = cb[0] <= b1.y && b0.x <= cb[3] && cb[1] <= b2.x && b0.y <= cb[4] &&
                      cb[2] <= b2.y && b1.x <= cb[5];
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t mask = __ballot_sync(kFull, ov[u]);
        if (!mask) continue;
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(p.ctrl + kPairs, (uint32_t)__popc(mask));
        base = __shfl_sync(kFull, base, 0);
        if (ov[u]) {
          const uint64_t vv = t0 + tt[u];
          const int ob = obs[u];
          atomicOr(p.ovmask + (uint64_t)(ob >> 5) * p.slot_cap + vv, 1u << (ob & 31));
          const uint64_t idx = base + __popc(mask & ((1u << lane) - 1u));
          if (idx < p.pair_cap) p.pairs[idx] = (vv << 32) | (uint32_t)ob;
          else atomicOr(p.ctrl + kErr, 1u);
        }
      }
    }
    __syncthreads();  // tile buffers are reused by the next tile
  }
}

// ------------------------------------------------------------------ phase B
__device__ void phase_b(const PlaceParams& p, Shared& sh, const uint32_t* act, int W,
                        Local& L) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  uint64_t np = __ldcg(p.ctrl + kPairs);
  if (np > p.pair_cap) np = p.pair_cap;
  WarpScratch& ws = sh.u.ws[threadIdx.x >> 5];
  for (uint64_t q = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); q < np; q += nwarps) {
    const uint64_t pr = p.pairs[q];
    const uint64_t v = pr >> 32;
    const int32_t ob = (int32_t)(pr & 0xffffffffu);
    const bool hit = warp_collide(p.w, sh.gc, ob, act[v / W], p.cinv + 12 * v, ws, L.cnt);
    if (hit && lane == 0) atomicMin(p.contact + v, ob);
    __syncwarp();
  }
}

// ------------------------------------------------------------------ phase C
// Thread per remaining instance: first free attempt among its W slots is accepted
// (update_transform + set_enabled, Appendix C.5); counters follow the sequential loop.
__device__ void phase_c(const PlaceParams& p, const uint32_t* act, uint64_t m, int W,
                        int32_t attempt, Local& L) {
  const WorldView& w = p.w;
  const int words = w.n_words;
  compact_count(p, m, [&](uint64_t e) -> int {
    int32_t last = attempt;  // last attempt this instance made in the sequential loop
    bool ok = false;
    for (int s = 0; s < W && !ok; ++s) {
      const uint64_t v = e * W + s;
      last = attempt + s;
      ++L.sampled;
      if (p.cflag[v] != kSlotChecked) continue;  // placeable == 0 -> failed attempt
      ++L.checked;
      const int32_t c = __ldcg(p.contact + v);
      for (int wd = 0; wd < words; ++wd) {  // narrow tests up to the first hit
        uint32_t mk = p.ovmask[(uint64_t)wd * p.slot_cap + v];
        if (c != kFree) {
          const int lim = c - 32 * wd;  // keep objects <= c
          if (lim < 0) mk = 0;
          else if (lim < 31) mk &= (2u << lim) - 1u;
        }
        L.cnt.narrow += __popc(mk);
      }
      if (c == kFree) {
        const uint32_t inst = act[e];
        M34 P;
#pragma unroll
        for (int k = 0; k < 12; ++k) P.m[k] = p.cpose[v * 12 + k];
        store_pose(w, p.pl.object, inst, P);
        w.enabled[sb_word_off(w, p.pl.object >> 5, inst)] |= 1u << (p.pl.object & 31);
        p.accepted[inst] = (int16_t)(attempt + s);
        ++L.accepted;
        ok = true;
      }
    }
    atomicMax(p.ctrl + kRounds, (uint32_t)(last + 1));  // reference round count
    p.failflag[e] = ok ? 0 : 1;
    return ok ? 0 : 1;
  });
  if (blockIdx.x == 0 && threadIdx.x == 0) p.ctrl[kPairs] = 0;  // phase B is done reading it
}

// ------------------------------------------------------------------ kernels
__device__ __forceinline__ void block_setup(const PlaceParams& p, Shared& sh, SbGeom& gA) {
  gA = p.w.geoms[p.pl.geom];
  load_geom_cache(p.w, gA, sh.gc);
  __syncthreads();
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Phase timer: block 0 / thread 0 accumulates wall time between grid barriers into
// p.prof[slot] (ns): 0 init, 1 A, 2 B, 3 C, 4 D; prof[5] counts rounds.
struct PhaseClock {
  uint64_t* prof;
  uint64_t t;
  __device__ PhaseClock(uint64_t* pr) : prof(pr), t(0) {
    if (prof && blockIdx.x == 0 && threadIdx.x == 0) t = global_ns();
  }
  __device__ void lap(int slot) {
    if (prof && blockIdx.x == 0 && threadIdx.x == 0) {
      uint64_t now = global_ns();
      prof[slot] += now - t;
      t = now;
    }
  }
};

__global__ void __launch_bounds__(kB, 2) k_place(PlaceParams p) {
  __shared__ Shared sh;
  cg::grid_group grid = cg::this_grid();
  PhaseClock clk(p.prof);
  SbGeom gA;
  block_setup(p, sh, gA);
  Local L;
  const uint64_t n = p.w.n;
  compact_count(p, n, [&](uint64_t i) -> int { return p.valid[i] != 0; });
  grid.sync();
  compact_scatter(p, n, [&](uint64_t i) -> int { return p.valid[i] != 0; },
                  [&](uint64_t i) -> uint32_t { return (uint32_t)i; }, p.act0);
  grid.sync();
  clk.lap(0);
  const Sampling S = resolve_sampling(p);
  if (p.vary_flag && !S.fast && blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(p.counters + 7, 1ull);  // per-instance placement
  uint64_t draws = 0;
  int cur = 0;
  for (int32_t a = 0; a < p.attempts;) {
    const uint64_t m = __ldcg(p.ctrl + kM);
    if (m == 0) break;
    const int W = spec_width(p, S.fast, m, a);
    const uint32_t* act = act_list(p, cur);
    phase_a(p, S, gA, sh, act, m, W, draws, a, L);
    grid.sync();
    clk.lap(1);
    phase_b(p, sh, act, W, L);
    grid.sync();
    clk.lap(2);
    phase_c(p, act, m, W, a, L);
    grid.sync();
    clk.lap(3);
    compact_scatter(p, m, [&](uint64_t e) -> int { return p.failflag[e]; },
                    [&](uint64_t e) -> uint32_t { return act[e]; }, act_list(p, cur ^ 1));
    grid.sync();
    clk.lap(4);
    if (p.prof && blockIdx.x == 0 && threadIdx.x == 0) p.prof[5] += 1;
    if (S.fast) draws += m;
    cur ^= 1;
    a += W;
  }
  const uint64_t m = __ldcg(p.ctrl + kM);
  const uint32_t* act = act_list(p, cur);
  for (uint64_t e = blockIdx.x * (uint64_t)kB + threadIdx.x; e < m; e += (uint64_t)gridDim.x * kB)
    p.valid[act[e]] = 0;  // K attempts exhausted: mark_invalid
  if (blockIdx.x == 0 && threadIdx.x == 0) p.ctrl[kCur] = cur;
  flush(p, L);
}

// Host-loop variants (sharded runs: the rank exchange happens between rounds).
__global__ void __launch_bounds__(kB) k_init_count(PlaceParams p) {
  compact_count(p, p.w.n, [&](uint64_t i) -> int { return p.valid[i] != 0; });
}
__global__ void __launch_bounds__(kB) k_init_scatter(PlaceParams p) {
  compact_scatter(p, p.w.n, [&](uint64_t i) -> int { return p.valid[i] != 0; },
                  [&](uint64_t i) -> uint32_t { return (uint32_t)i; }, p.act0);
}
__global__ void __launch_bounds__(kB) k_phase_a(PlaceParams p, int32_t attempt, int cur) {
  SbGeom gA = p.w.geoms[p.pl.geom];
  const uint64_t m = __ldcg(p.ctrl + kM);
  __shared__ Shared sh;
  Local L;
  const Sampling S = resolve_sampling(p);
  phase_a(p, S, gA, sh, act_list(p, cur), m, p.spec_width, p.draw_base, attempt, L);
  flush(p, L);
}
__global__ void __launch_bounds__(kB) k_phase_b(PlaceParams p, int cur) {
  __shared__ Shared sh;
  SbGeom gA;
  block_setup(p, sh, gA);
  Local L;
  phase_b(p, sh, act_list(p, cur), p.spec_width, L);
  flush(p, L);
}
__global__ void __launch_bounds__(kB) k_phase_c(PlaceParams p, int32_t attempt, int cur) {
  Local L;
  const uint64_t m = __ldcg(p.ctrl + kM);
  phase_c(p, act_list(p, cur), m, p.spec_width, attempt, L);
  flush(p, L);
}
__global__ void __launch_bounds__(kB) k_phase_d(PlaceParams p, int cur) {
  const uint64_t m = __ldcg(p.ctrl + kM);
  const uint32_t* act = act_list(p, cur);
  compact_scatter(p, m, [&](uint64_t e) -> int { return p.failflag[e]; },
                  [&](uint64_t e) -> uint32_t { return act[e]; }, act_list(p, cur ^ 1));
}
__global__ void __launch_bounds__(kB) k_finish(PlaceParams p, int cur) {
  const uint64_t m = __ldcg(p.ctrl + kM);
  const uint32_t* act = act_list(p, cur);
  for (uint64_t e = blockIdx.x * (uint64_t)kB + threadIdx.x; e < m; e += (uint64_t)gridDim.x * kB)
    p.valid[act[e]] = 0;
}

int g_coop_blocks = -1;

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

unsigned host_grid() {
  static unsigned g = 0;
  if (g == 0) {
    int dev = 0, sms = 0, per = 0;
    check(cudaGetDevice(&dev), "cudaGetDevice");
    check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_phase_b, kB, 0), "occupancy");
    g = (unsigned)(sms * (per > 0 ? per : 1));
  }
  return g;
}

}  // namespace

void narrow_profile(unsigned long long out[8], bool reset) {
  check(cudaMemcpyFromSymbol(out, g_nprof, 8 * sizeof(unsigned long long)), "narrow_profile");
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    check(cudaMemcpyToSymbol(g_nprof, z, sizeof z), "narrow_profile reset");
  }
}

int place_grid_warps(int num_sms) {
  if (g_coop_blocks < 0) {
    int per = 0;
    check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_place, kB, 0), "occupancy");
    g_coop_blocks = per * num_sms;
  }
  return g_coop_blocks * kWarps;
}

bool place_persistent(const PlaceParams& p, int num_sms, sb_stream_t s) {
  if (place_grid_warps(num_sms) <= 0) return false;
  unsigned grid = (unsigned)g_coop_blocks;
  PlaceParams q = p;
  void* args[] = {&q};
  check(cudaLaunchCooperativeKernel((void*)k_place, dim3(grid), dim3(kB), args, 0,
                                    reinterpret_cast<cudaStream_t>(s)),
        "cudaLaunchCooperativeKernel(k_place)");
  return true;
}

void place_init(const PlaceParams& p, sb_stream_t s) {
  unsigned g = host_grid();
  k_init_count<<<g, kB, 0, s>>>(p);
  k_init_scatter<<<g, kB, 0, s>>>(p);
  check(cudaGetLastError(), "place_init");
}

void place_round(const PlaceParams& p, int32_t attempt, int cur, sb_stream_t s) {
  unsigned g = host_grid();
  k_phase_a<<<g, kB, 0, s>>>(p, attempt, cur);
  k_phase_b<<<g, kB, 0, s>>>(p, cur);
  k_phase_c<<<g, kB, 0, s>>>(p, attempt, cur);
  k_phase_d<<<g, kB, 0, s>>>(p, cur);
  check(cudaGetLastError(), "place_round");
}

void place_finish(const PlaceParams& p, int cur, sb_stream_t s) {
  k_finish<<<host_grid(), kB, 0, s>>>(p, cur);
  check(cudaGetLastError(), "place_finish");
}

}  // namespace sbk
