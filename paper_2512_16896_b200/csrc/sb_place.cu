// Tiled placement engine (see sb_place.h). sm_100a, -fmad=false.
#include <cooperative_groups.h>
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
constexpr int kQueue = 2048;  // shared-memory narrow-phase queue (slot << 24 | object)
constexpr int kU = 4;         // broad-phase items per thread per batch (loads in flight)
constexpr uint8_t kSlotChecked = 1, kSlotUnplaceable = 2;
constexpr int kPrefixItems = 8;  // tile counts per thread per prefix-scan chunk

enum Ctrl { kRounds = 2, kErr = 3, kTileCtr = 4 /* kTotal0 = 5, kTotal1 = 6 */ };

using BlockScan = cub::BlockScan<uint32_t, kB>;

// Per-round candidate state of the CTA's tile (dynamic shared memory).
struct Tile {
  double* inv;       // [kB][12] inverse pose per slot
  double* box;       // [kB][6]  candidate world AABB per slot
  uint32_t* ovm;     // [words][kB] broad-phase overlap bits per slot
  uint32_t* enw;     // [words][kB] enable words per tile entry
  uint32_t* list;    // [kB] tile's active instances (ascending)
  uint32_t* queue;   // [kQueue]
  int32_t* contact;  // [kB] min colliding object per slot
  uint32_t* rem;     // [kB] queued, not yet tested pairs per slot
  int32_t* minfree;  // [kB] per tile entry: lowest slot (attempt offset) confirmed free, W = none
  uint8_t* sflag;    // [kB]
  unsigned char* ws; // [kWarps][ws_bytes]
  int4* ogeo;        // [n_objects] narrow-record descriptor of each object's geometry
};

struct Fixed {  // static shared memory
  GeomCache gc;
  typename BlockScan::TempStorage scan;
  uint32_t prefix[kPlaceMaxOwnedTiles];  // fast path: draw offset of each owned tile
  uint32_t cnt[kPlaceMaxOwnedTiles];     // fast path: its survivors entering this round
  uint32_t qn;
  uint32_t vdone;  // slots whose broad-phase items are all enumerated
  uint32_t total;
  uint32_t tile;
  unsigned long long tclk;  // block 0 / thread 0 phase clock
  unsigned long long acc[8];  // its per-slot sums, written to p.prof once at the end
  unsigned long long ta, tb, t0;  // every block: A1 / A2+B ns of the current round (debug)
};

__device__ __forceinline__ Tile carve(unsigned char* d, int words, int ws_bytes) {
  Tile t;
  t.inv = reinterpret_cast<double*>(d);
  t.box = t.inv + 12 * kB;
  t.ovm = reinterpret_cast<uint32_t*>(t.box + 6 * kB);
  t.enw = t.ovm + words * kB;
  t.list = t.enw + words * kB;
  t.queue = t.list + kB;
  t.contact = reinterpret_cast<int32_t*>(t.queue + kQueue);
  t.rem = reinterpret_cast<uint32_t*>(t.contact + kB);
  t.minfree = reinterpret_cast<int32_t*>(t.rem + kB);
  t.sflag = reinterpret_cast<uint8_t*>(t.minfree + kB);
  t.ws = t.sflag + kB;
  t.ogeo = reinterpret_cast<int4*>(t.ws + kWarps * ws_bytes);
  return t;
}

__host__ __device__ constexpr size_t tile_bytes(int words) {
  return (12 + 6) * 8 * (size_t)kB + 2 * (size_t)words * kB * 4 + (size_t)kB * 4 +
         (size_t)kQueue * 4 + 3 * (size_t)kB * 4 + kB;
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

// ------------------------------------------------------------------ one tile round
// Evaluates attempts [a, a + W) of the tile's nt active instances (T.list) and compacts the
// survivors in place. Returns the survivor count. All threads of the CTA call it.
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
    const int e = v / W;
    const int32_t at = a + (v - e * W);
    const uint32_t inst = T.list[e];
    const uint64_t gid = p.global_begin + inst;
    bool placeable = true;
    double lx = 0.0, ly = 0.0;
    if (S.fast) {
      if (S.n == 0) {
        placeable = false;
      } else {
        Pcg r{p.fast_state0};
        r.advance(6ull * (draw_base + (uint64_t)e));  // j-th drained point = j-th draw (sampler.cpp:30-43)
        double u = r.next_double(), r1 = r.next_double(), r2 = r.next_double();
        sbp::draw_point(S.tris, S.cum, S.n, u, r1, r2, lx, ly);
      }
    } else {
      const int nti = __ldg(p.inst_n + inst);
      if (nti == 0) {
        placeable = false;
      } else {  // make_stream(run_seed, {salt, "fall", inst, attempt}) (sampler.cpp:117)
        Pcg r = Pcg::seeded(stream_seed4(p.run_seed, pl.salt, kFallbackSalt, gid,
                                         static_cast<uint64_t>(at)));
        double u = r.next_double(), r1 = r.next_double(), r2 = r.next_double();
        const uint64_t off = (uint64_t)inst * p.inst_cap;
        sbp::draw_point(p.inst_tris + off, p.inst_cum + off, nti, u, r1, r2, lx, ly);
      }
    }
    T.contact[v] = kFree;
    T.rem[v] = 0u;
    if (v - e * W == 0) T.minfree[e] = W;
    for (int wd = 0; wd < words; ++wd) T.ovm[wd * kB + v] = 0u;
    if (!placeable) {
      T.sflag[v] = kSlotUnplaceable;
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
      M34 Tr, Rz, pose;  // translation(p + z_off z) * rotation_z(yaw)
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
      double cmn[3], cmx[3];
      xform_aabb(pose, gA.box_c, gA.box_h, cmn, cmx);
      M34 inv;
      inverse_rigid(pose, inv);
      double2* cp = reinterpret_cast<double2*>(p.cpose + ((size_t)blockIdx.x * kB + v) * 12);
#pragma unroll
      for (int k = 0; k < 6; ++k) cp[k] = make_double2(pose.m[2 * k], pose.m[2 * k + 1]);
#pragma unroll
      for (int k = 0; k < 12; ++k) T.inv[12 * v + k] = inv.m[k];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        T.box[6 * v + k] = cmn[k];
        T.box[6 * v + 3 + k] = cmx[k];
      }
      T.sflag[v] = kSlotChecked;
    }
  }
  if (tid == 0) {
    F.qn = 0;
    F.vdone = 0;
  }
  __syncthreads();
  lap(p, F, 2);
  dbg_mark(p, F, F.ta);

  // ---------------- A2 (broad phase) interleaved with B (narrow phase) in queue batches
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
            ((T.enw[(ob >> 5) * kB + v / W] >> (ob & 31)) & 1u)) {
          ++L.cnt.broad;
          const double2* bp = reinterpret_cast<const double2*>(w.box + sb_box_off(w, ob, T.list[v / W]));
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
    // Slots whose items are now all enumerated and whose queued pairs are all tested
    // without a hit are free: the instance's lowest such attempt bounds the useful work.
    const int vdone_old = (int)F.vdone;
    int vdone = (it0 + kB * kU >= items) ? nslots : (it0 + kB * kU) / nobj;
    for (int v = vdone_old + tid; v < vdone; v += kB)
      if (T.sflag[v] == kSlotChecked && T.rem[v] == 0u && T.contact[v] == kFree)
        atomicMin(T.minfree + v / W, v - (v / W) * W);
    __syncthreads();
    if (tid == 0) F.vdone = (uint32_t)vdone;
    const uint32_t qn = F.qn;
    if (it0 + kB * kU >= items || qn > (uint32_t)(kQueue - kB * kU)) {
      // ---------------- B: warp per queued pair; skip pairs behind a lower hit
      const WarpScratchView ws = carve_scratch(T.ws + warp * p.ws_bytes, p.max_tris, p.max_nodes);
      // software-pipelined: the next pair's pose and geometry record are copied into the
      // warp's other staging buffer (cp.async) while the current pair is tested
      unsigned char* wsb = T.ws + warp * p.ws_bytes;
      uint32_t q = warp;
      int v = 0, ob = 0, cur = 0;
      int4 gr = make_int4(0, 0, 0, 0);
      auto fetch = [&](uint32_t qq, int& v_, int& ob_, int4& g_, int buf) {
        const uint32_t ent = T.queue[qq];
        v_ = (int)(ent >> 24);
        ob_ = (int)(ent & 0xffffffu);
        g_ = T.ogeo[ob_];
        warp_stage(w, g_, ob_, T.list[v_ / W], stage_buf(wsb, p.max_tris, p.max_nodes, buf));
      };
      if (q < qn) fetch(q, v, ob, gr, 0);
      while (q < qn) {
        const uint32_t qn2 = q + kWarps;
        int v2 = 0, ob2 = 0;
        int4 gr2 = make_int4(0, 0, 0, 0);
        if (qn2 < qn) {
          fetch(qn2, v2, ob2, gr2, cur ^ 1);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncwarp();
        // skip pairs behind a lower hit of their slot, or of a slot beyond the instance's
        // lowest confirmed-free attempt (neither can change the first-valid result)
        const int e = v / W;
        if (*((volatile int32_t*)T.contact + v) >= ob &&
            v - e * W <= *((volatile int32_t*)T.minfree + e)) {
          const bool hit = warp_collide(F.gc, stage_buf(wsb, p.max_tris, p.max_nodes, cur), gr.z,
                                        gr.w, T.inv + 12 * v, ws, L.cnt);
          if (lane == 0) {
            if (hit) {
              atomicMin(T.contact + v, ob);
            } else if (atomicSub(T.rem + v, 1u) == 1u && v < vdone &&
                       *((volatile int32_t*)T.contact + v) == kFree) {
              atomicMin(T.minfree + e, v - e * W);
            }
          }
        }
        __syncwarp();
        q = qn2;
        v = v2;
        ob = ob2;
        gr = gr2;
        cur ^= 1;
      }
      __syncthreads();
      if (tid == 0) F.qn = 0;
      __syncthreads();
    }
  }
  if (items == 0) __syncthreads();
  lap(p, F, 3);
  dbg_mark(p, F, F.tb);

  // ---------------- C: thread per instance; first free slot is accepted (Appendix C.5)
  uint32_t keep = 0, inst = 0;
  if (tid < (int)nt) {
    const int e = tid;
    inst = T.list[e];
    int32_t last = a;  // last attempt this instance made in the sequential loop
    bool ok = false;
    for (int s = 0; s < W && !ok; ++s) {
      const int v = e * W + s;
      last = a + s;
      ++L.sampled;
      if (T.sflag[v] != kSlotChecked) continue;  // placeable == 0 -> failed attempt
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
        double2* pp = reinterpret_cast<double2*>(w.pose + sb_pose_off(w, pl.object, inst));
#pragma unroll
        for (int k = 0; k < 6; ++k) pp[k] = __ldcg(reinterpret_cast<const double2*>(p.cpose + ((size_t)blockIdx.x * kB + v) * 12) + k);
        double2* bp = reinterpret_cast<double2*>(w.box + sb_box_off(w, pl.object, inst));
#pragma unroll
        for (int k = 0; k < 3; ++k) bp[k] = make_double2(T.box[6 * v + 2 * k], T.box[6 * v + 2 * k + 1]);
        w.enabled[sb_word_off(w, pl.object >> 5, inst)] |= 1u << (pl.object & 31);
        p.accepted[inst] = (int16_t)(a + s);
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
__device__ uint32_t tile_load_valid(const PlaceParams& p, Tile& T, Fixed& F, uint32_t t) {
  const uint64_t i = (uint64_t)t * p.tile_inst + threadIdx.x;
  const uint32_t f = (threadIdx.x < p.tile_inst && i < p.w.n && p.valid[i] != 0) ? 1u : 0u;
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
__device__ uint64_t tile_prefix(const PlaceParams& p, const uint32_t* cnt, Fixed& F) {
  const uint32_t G = gridDim.x, b = blockIdx.x, nt = p.ntiles;
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
__device__ uint64_t fast_round(const PlaceParams& p, const Sampling& S, const SbGeom& gA,
                               Tile& T, Fixed& F, int32_t a, uint64_t draws, Local& L,
                               uint32_t* total_word) {
  const uint32_t* cin = p.tile_cnt + (size_t)(a & 1) * p.cnt_stride;
  uint32_t* cout = p.tile_cnt + (size_t)((a + 1) & 1) * p.cnt_stride;
  const uint64_t total = tile_prefix(p, cin, F);
  lap(p, F, 1);
  if (total == 0) return 0;
  uint32_t k = 0, mine = 0;
  for (uint32_t t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++k) {
    const uint32_t n = F.cnt[k];
    if (n == 0) {
      if (threadIdx.x == 0) cout[t] = 0;
      continue;
    }
    load_list(p, T, t, n);
    lap(p, F, 1);
    if (p.dbg && threadIdx.x == 0) F.t0 = global_ns();
    const uint32_t ns = tile_round(p, S, gA, T, F, n, a, 1, draws + F.prefix[k], L);
    store_list(p, T, t, ns, cout);
    mine += ns;
    __syncthreads();
  }
  if (total_word && threadIdx.x == 0 && mine) atomicAdd(total_word, mine);
  return total;
}

// Per-instance path: tiles are independent; each is run to completion by one CTA.
__device__ void instance_tiles(const PlaceParams& p, const Sampling& S, const SbGeom& gA,
                               Tile& T, Fixed& F, Local& L) {
  for (;;) {
    if (threadIdx.x == 0) F.tile = atomicAdd(p.ctrl + kTileCtr, 1u);
    __syncthreads();
    const uint32_t t = F.tile;
    __syncthreads();
    if (t >= p.ntiles) break;
    uint32_t nt = tile_load_valid(p, T, F, t);
    int32_t a = 0;
    unsigned rounds = 0;
    const unsigned long long tt0 = p.dbg_inst && threadIdx.x == 0 ? global_ns() : 0;
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
      nt = tile_round(p, S, gA, T, F, nt, a, W, 0, L);
      a += W;
      if (p.dbg_inst && threadIdx.x == 0) {  // A1 / A2+B / C sums (us) and A2+B max (ns)
        atomicAdd(p.dbg_inst + 5, (unsigned)(F.ta / 1000));
        atomicAdd(p.dbg_inst + 6, (unsigned)(F.tb / 1000));
        atomicAdd(p.dbg_inst + 7, (unsigned)((global_ns() - F.t0) / 1000));
        atomicMax(p.dbg_inst + 8, (unsigned)F.tb);
        atomicAdd(p.dbg_inst + 9, nslots_dbg);
      }
    }
    mark_invalid(p, T, nt);
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
  gA = p.w.geoms[p.pl.geom];
  load_geom_cache(p.w, gA, F.gc);
  for (int ob = threadIdx.x; ob < p.w.n_objects; ob += kB) T.ogeo[ob] = obj_grec(p.w, ob);
  __syncthreads();
}

extern __shared__ __align__(16) unsigned char g_dsm[];

__global__ void __launch_bounds__(kB, 2) k_place(PlaceParams p) {
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
    instance_tiles(p, S, gA, T, F, L);
    if (timer) F.acc[6] += global_ns() - t6;
  } else {
    cg::grid_group grid = cg::this_grid();
    for (uint32_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
      const uint32_t n = tile_load_valid(p, T, F, t);
      store_list(p, T, t, n, p.tile_cnt);
      __syncthreads();
    }
    lap(p, F, 0);
    grid.sync();
    lap(p, F, 5);
    uint64_t draws = 0;
    int32_t a = 0;
    for (; a < p.attempts; ++a) {
      unsigned long long r0 = 0;
      if (p.dbg && threadIdx.x == 0) {
        r0 = global_ns();
        F.ta = F.tb = 0;
      }
      const uint64_t total = fast_round(p, S, gA, T, F, a, draws, L, nullptr);
      if (total == 0) break;
      draws += total;
      if (p.dbg && threadIdx.x == 0) {  // per-round maxima over CTAs: work, A1, A2+B
        atomicMax(p.dbg + 3 * a, (unsigned)(global_ns() - r0));
        atomicMax(p.dbg + 3 * a + 1, (unsigned)F.ta);
        atomicMax(p.dbg + 3 * a + 2, (unsigned)F.tb);
      }
      lap(p, F, 1);
      grid.sync();
      lap(p, F, 5);
      if (timer) F.acc[7] += 1;
    }
    if (a == p.attempts) {  // K attempts exhausted: survivors are invalid
      const uint32_t* cin = p.tile_cnt + (size_t)(a & 1) * p.cnt_stride;
      for (uint32_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
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
__global__ void __launch_bounds__(kB, 2) k_place_instances(PlaceParams p) {
  __shared__ Fixed F;
  Tile T = carve(g_dsm, p.w.n_words, p.ws_bytes);
  SbGeom gA;
  block_setup(p, F, T, gA);
  Local L;
  Sampling S{0, nullptr, nullptr, 0};
  instance_tiles(p, S, gA, T, F, L);
  flush(p, L);
}

__global__ void __launch_bounds__(kB, 2) k_fast_init(PlaceParams p) {
  __shared__ Fixed F;
  Tile T = carve(g_dsm, p.w.n_words, p.ws_bytes);
  uint32_t mine = 0;
  for (uint32_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
    const uint32_t n = tile_load_valid(p, T, F, t);
    store_list(p, T, t, n, p.tile_cnt);
    mine += n;
    __syncthreads();
  }
  if (threadIdx.x == 0 && mine) atomicAdd(p.ctrl + place_total_word(0), mine);
}

__global__ void __launch_bounds__(kB, 2) k_fast_round(PlaceParams p, int32_t a) {
  __shared__ Fixed F;
  Tile T = carve(g_dsm, p.w.n_words, p.ws_bytes);
  SbGeom gA;
  block_setup(p, F, T, gA);
  Local L;
  Sampling S{1, p.canon_tris, p.canon_cum, p.canon_n};
  fast_round(p, S, gA, T, F, a, p.draw_base, L, p.ctrl + place_total_word(a + 1));
  flush(p, L);
}

__global__ void __launch_bounds__(kB) k_fast_finish(PlaceParams p, int32_t a) {
  const uint32_t* cin = p.tile_cnt + (size_t)(a & 1) * p.cnt_stride;
  for (uint32_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
    const uint32_t n = __ldcg(cin + t);
    const uint32_t* src = p.tile_list + (uint64_t)t * p.tile_inst;
    for (uint32_t e = threadIdx.x; e < n; e += kB) p.valid[src[e]] = 0;
  }
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

int place_grid(int num_sms, size_t smem) {
  set_smem((const void*)k_place, smem);
  int per = 0;
  check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_place, kB, smem), "occupancy");
  return per * num_sms;
}

bool place_persistent(const PlaceParams& p, unsigned grid, size_t smem, sb_stream_t s) {
  if (grid == 0) return false;
  PlaceParams q = p;
  void* args[] = {&q};
  check(cudaLaunchCooperativeKernel((void*)k_place, dim3(grid), dim3(kB), args, smem,
                                    reinterpret_cast<cudaStream_t>(s)),
        "cudaLaunchCooperativeKernel(k_place)");
  return true;
}

void place_instances(const PlaceParams& p, unsigned grid, size_t smem, sb_stream_t s) {
  set_smem((const void*)k_place_instances, smem);
  k_place_instances<<<grid, kB, smem, s>>>(p);
  check(cudaGetLastError(), "k_place_instances");
}

void place_fast_init(const PlaceParams& p, unsigned grid, size_t smem, sb_stream_t s) {
  set_smem((const void*)k_fast_init, smem);
  k_fast_init<<<grid, kB, smem, s>>>(p);
  check(cudaGetLastError(), "k_fast_init");
}

void place_fast_round(const PlaceParams& p, int32_t attempt, unsigned grid, size_t smem,
                      sb_stream_t s) {
  set_smem((const void*)k_fast_round, smem);
  k_fast_round<<<grid, kB, smem, s>>>(p, attempt);
  check(cudaGetLastError(), "k_fast_round");
}

void place_fast_finish(const PlaceParams& p, int32_t attempt, unsigned grid, sb_stream_t s) {
  k_fast_finish<<<grid, kB, 0, s>>>(p, attempt);
  check(cudaGetLastError(), "k_fast_finish");
}

}  // namespace sbk
