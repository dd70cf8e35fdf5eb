// Warp-pooled candidate check with an exact, parallel BVH-vs-BVH narrow phase.
//
// Lane i owns candidate i of the warp for everything uniform per candidate (sampling,
// pose compose, candidate AABB, inverse pose, AABB broad phase over enabled objects).
// Narrow-phase pairs (candidate, object) are pooled: the whole warp takes one pair at a
// time.
//
// Narrow phase = MeshBvh::collide (collision.cpp:285-329) restated for 32 lanes:
//  1. lane b transforms B's effective node b into A's frame (transform_aabb is independent
//     of the A node it is tested against);
//  2. for every A node a, one ballot yields pass(a, .) = na.box.overlaps(nb_in_a) and one
//     the descend rule desc(a, .) = leaf(nb) || (!leaf(na) && ext2(na) >= ext2(nb_in_a));
//  3. a bitmask walk of the pair DAG from (0,0) -- the reference's stack traversal with
//     children read as {left, left+1}, each pair visited once -- marks the leaf pairs the
//     reference would reach with every box test on the way passing;
//  4. the triangle pairs of those leaf pairs are tested in parallel.
// The verdict is "some reached leaf pair has an intersecting triangle pair": exactly the
// reference's (its early exit and repeated visits do not change an existential).
// Objects of a candidate are visited in ascending id order with an early exit at the first
// hit, so contact_object matches collision.cpp:439-448.
#pragma once

#include "sb_dev.cuh"

namespace sbd {

constexpr unsigned kFull = 0xffffffffu;

// Optional cycle breakdown of the narrow phase (build with -DSB_NARROW_PROF):
// [0] M, [1] B triangle transform + planes, [2] node transform + node-pair tests (hits
// only), [3] DAG walk, [4] reached-hit check, [5] pairs, [6] filter 1, [7] filter 2 + rest.
static __device__ unsigned long long g_nprof[8];
#ifdef SB_NARROW_PROF
#define SB_NP_MARK(var) const long long var = clock64()
#define SB_NP_ADD(k, a, b) \
  if ((threadIdx.x & 31) == 0) atomicAdd(&g_nprof[k], (unsigned long long)((b) - (a)))
#else
#define SB_NP_MARK(var)
#define SB_NP_ADD(k, a, b)
#endif
constexpr int kMaxEffTris = SB_MAX_EFF_TRIS;  // host-checked at registration
constexpr int kMaxNodes = SB_MAX_NODES_PER_GEOM;

// ---------------------------------------------------------------- async staging
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
// L2-only variant for data written earlier in the same kernel (no stale L1 line).
__device__ __forceinline__ void cp_async16_cg(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Bytes of one pair's staging buffer: the placed object's pose (row-major 3x4, 96 B), the
// candidate's inverse pose (96 B) and the compact record of its geometry (sb_layout.h).
__host__ __device__ constexpr int stage_bytes(int maxT, int maxN) {
  return 192 + sb_brec_bytes(maxN, maxT);
}

// The whole warp issues the asynchronous copies of pair (ob, inst) into `dst` (one commit
// group per lane); gr = grec[geometry of ob]; inv = the candidate's inverse pose in global
// memory (12 doubles, 16-byte aligned) or null when the caller fills dst + 96 itself.
__device__ __forceinline__ void warp_stage(const WorldView& w, const int4 gr, int32_t ob,
                                           uint64_t inst, const double* inv, unsigned char* dst,
                                           int inv_chunks = 6) {
  const int lane = threadIdx.x & 31;
  const unsigned char* pose = reinterpret_cast<const unsigned char*>(w.pose + sb_pose_off(w, ob, inst));
  const unsigned char* rec = reinterpret_cast<const unsigned char*>(w.brec) + 16 * (size_t)gr.x;
  for (int c = lane; c < 12 + gr.y; c += 32) {
    if (c < 6) cp_async16_cg(dst + 16 * c, pose + 16 * c);
    else if (c < 12) {
      if (inv && c - 6 < inv_chunks)
        cp_async16_cg(dst + 16 * c, reinterpret_cast<const unsigned char*>(inv) + 16 * (c - 6));
    } else cp_async16(dst + 16 * c, rec + 16 * (c - 12));
  }
  cp_async_commit();
}

// ---------------------------------------------------------------- bulk-copy staging
// The same staging with the Blackwell copy engine: one lane arms an mbarrier with the byte
// count and issues cp.async.bulk (global -> shared, no register or LSU round trip per 16 B;
// SASS UBLKCP + SYNCS), the warp waits on the barrier's phase.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned phase) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// generic-proxy writes to shared memory before later async-proxy (bulk) writes to it
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Lane 0 stages pair (ob, inst) into dst with bulk copies completing on `bar`: the placed
// pose (96 B), `cand_bytes` of candidate data at +96, the geometry record at +192.
__device__ __forceinline__ void warp_stage_bulk(const WorldView& w, const int4 gr, int32_t ob,
                                                uint64_t inst, const double* cand,
                                                unsigned cand_bytes, unsigned char* dst,
                                                uint64_t* bar) {
  if ((threadIdx.x & 31) == 0) {
    fence_proxy_async_smem();
    const unsigned rec_bytes = 16u * (unsigned)gr.y;
    mbar_expect_tx(bar, 96u + cand_bytes + rec_bytes);
    bulk_g2s(dst, w.pose + sb_pose_off(w, ob, inst), 96u, bar);
    bulk_g2s(dst + 96, cand, cand_bytes, bar);
    bulk_g2s(dst + 192, reinterpret_cast<const unsigned char*>(w.brec) + 16 * (size_t)gr.x, rec_bytes, bar);
  }
}

// {record offset, record length (16 B units), n_nodes, n_tris} of object ob's geometry.
__device__ __forceinline__ int4 obj_grec(const WorldView& w, int32_t ob) {
  return __ldg(reinterpret_cast<const int4*>(w.grec) + __ldg(w.obj_geom + ob));
}

// Per-warp narrow-phase scratch, as pointers into shared memory so a kernel can size it
// by the world's largest effective geometry (place_ws_bytes) or use the fixed-size
// WarpScratch below.
struct WarpScratchView {
  double* M;           // [12] other_in_self of the pair under test
  double* qb;          // [maxT][9] B's effective triangles moved into A's frame
  double* pb;          // [maxT][5] their planes: n xyz, dc, tol (TriPlane)
  double* bb;          // [maxN][6] B's effective node boxes in A's frame
  double* e2b;         // [maxN] their squared extents
  uint32_t* cm;        // [maxN] B node -> mask of its effective children (0 for leaves)
  uint32_t* allowed;   // [maxN] A leaf -> B leaves whose boxes overlap; later the walk rows
  uint32_t* H;         // [maxN] A leaf -> B leaves holding an intersecting triangle pair
  uint32_t* lbb;       // [maxN] B node -> effective leaves below it
  uint32_t* pend;      // [maxN] pair-DAG walk: visited B nodes per A node
  uint16_t* l1;        // [max(maxT^2, maxN^2)] triangle pairs past filter 1 / walk frontier
  uint16_t* l2;        // [max(maxT^2, maxN^2)] triangle pairs past filter 2 / walk frontier
  int8_t* tleafb;      // [maxT]
  int8_t* leafb;       // [maxN] B's leaf node ids, ascending
};

__host__ __device__ constexpr int scratch_list_len(int maxT, int maxN) {
  return maxT * maxT > maxN * maxN ? maxT * maxT : maxN * maxN;
}

__host__ __device__ constexpr int warp_scratch_bytes(int maxT, int maxN) {
  return ((((12 + maxT * 14 + maxN * 7) * 8 + 5 * maxN * 4 + 2 * scratch_list_len(maxT, maxN) * 2 +
            maxT + maxN) + 15) & ~15) +
         2 * stage_bytes(maxT, maxN);  // + double-buffered staging
}

// The two staging buffers of a warp's scratch (16-byte aligned, after the scratch arrays).
__device__ __forceinline__ unsigned char* stage_buf(unsigned char* ws_base, int maxT, int maxN, int k) {
  return ws_base + warp_scratch_bytes(maxT, maxN) - (2 - k) * stage_bytes(maxT, maxN);
}

__device__ __forceinline__ WarpScratchView carve_scratch(unsigned char* base, int maxT, int maxN) {
  WarpScratchView v;
  double* d = reinterpret_cast<double*>(base);
  v.M = d;
  v.qb = d + 12;
  v.pb = v.qb + 9 * maxT;
  v.bb = v.pb + 5 * maxT;
  v.e2b = v.bb + 6 * maxN;
  uint32_t* u = reinterpret_cast<uint32_t*>(v.e2b + maxN);
  v.cm = u;
  v.allowed = u + maxN;
  v.H = u + 2 * maxN;
  v.lbb = u + 3 * maxN;
  v.pend = u + 4 * maxN;
  v.l1 = reinterpret_cast<uint16_t*>(u + 5 * maxN);
  v.l2 = v.l1 + scratch_list_len(maxT, maxN);
  v.tleafb = reinterpret_cast<int8_t*>(v.l2 + scratch_list_len(maxT, maxN));
  v.leafb = v.tleafb + maxT;
  return v;
}

struct alignas(16) WarpScratch {  // fixed-size variant (world API check_batch)
  unsigned char bytes[warp_scratch_bytes(kMaxEffTris, kMaxNodes)];
  __device__ __forceinline__ WarpScratchView view() {
    return carve_scratch(bytes, kMaxEffTris, kMaxNodes);
  }
};

// Candidate geometry (uniform per launch), staged in shared memory once per block, with
// the planes of its triangles (pure functions of the A triangles in A's own frame).
template <int NT, int NN>
struct GeomCacheT {
  double ta[NT][9];
  double pa[NT][5];  // TriPlane: n xyz, dc, tol
  double bmin[NN][3], bmax[NN][3];
  double ext2[NN];
  int8_t c0[NN], c1[NN];
  int8_t tleaf[NT];
  uint32_t leafmask;
  int8_t leaves[NN];  // leaf node ids, ascending
  uint32_t lbelow[NN];  // effective leaves under each node
  int n_tris, n_nodes, n_leaves;
};

// world API check_batch: any registrable geometry; placement engine: <= 16 / 16 (host-checked)
using GeomCache = GeomCacheT<kMaxEffTris, kMaxNodes>;
constexpr int kPlaceCacheTris = 16, kPlaceCacheNodes = 16;
using PlaceGeomCache = GeomCacheT<kPlaceCacheTris, kPlaceCacheNodes>;

template <class GC>
__device__ __forceinline__ void load_geom_cache(const WorldView& w, const SbGeom& gA, GC& gc) {
  const SbTri* t = w.tris + gA.tri_offset;
  const SbNode* nd = w.nodes + gA.node_offset;
  for (int k = threadIdx.x; k < gA.n_tris; k += blockDim.x) {
    double v[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) gc.ta[k][c] = v[c] = t[k].v[c];
    const TriPlane P = tri_plane(v);
    gc.pa[k][0] = P.n[0];
    gc.pa[k][1] = P.n[1];
    gc.pa[k][2] = P.n[2];
    gc.pa[k][3] = P.dc;
    gc.pa[k][4] = P.tol;
    gc.tleaf[k] = (int8_t)t[k].leaf;
  }
  for (int k = threadIdx.x; k < gA.n_nodes; k += blockDim.x) {
    for (int c = 0; c < 3; ++c) {
      gc.bmin[k][c] = nd[k].bmin[c];
      gc.bmax[k][c] = nd[k].bmax[c];
    }
    gc.ext2[k] = nd[k].ext2;
    gc.c0[k] = (int8_t)nd[k].child0;
    gc.c1[k] = (int8_t)nd[k].child1;
    gc.lbelow[k] = nd[k].leaves_below;
  }
  if (threadIdx.x == 0) {
    uint32_t lm = 0;
    for (int k = 0; k < gA.n_nodes; ++k)
      if (nd[k].child0 < 0) lm |= 1u << k;
    gc.leafmask = lm;
    int nl = 0;
    for (int k = 0; k < gA.n_nodes; ++k)
      if ((lm >> k) & 1u) gc.leaves[nl++] = (int8_t)k;
    gc.n_leaves = nl;
    gc.n_tris = gA.n_tris;
    gc.n_nodes = gA.n_nodes;
  }
}

// Appends the lanes with `pass` to list[n..] in lane order; returns the new length.
__device__ __forceinline__ int warp_append(bool pass, uint16_t value, uint16_t* list, int n) {
  const int lane = threadIdx.x & 31;
  const uint32_t m = __ballot_sync(kFull, pass);
  if (pass) list[n + __popc(m & ((1u << lane) - 1u))] = value;
  return n + __popc(m);
}

// Warp-cooperative MeshBvh::collide for one (candidate, object) pair. All 32 lanes call
// it with identical arguments. `Pn` (lanes < 12) holds the placed object's pose entries,
// loaded by the caller (software-pipelined one pair ahead).
//  1. M = other_in_cand (lanes < 12), B's effective triangles into A's frame and their
//     planes (one lane per triangle; A's planes are cached per launch);
//  2. every triangle pair of Eff(A) x Eff(B) runs through tri_tri_intersect as three
//     compacted filter passes -- B's plane vs A's vertices, A's plane vs B's vertices, the
//     interval / coplanar rest -- so the long FP64 tail runs only for the few pairs that
//     survive both plane tests. No intersecting pair => the reference cannot report a hit;
//  3. otherwise the node-pair tests and the pair-DAG walk decide which leaf pairs the
//     reference traversal reaches; hit = some reached leaf pair holds an intersecting pair.
// `stage` = the pair's staged pose + geometry record (warp_stage, copies complete and
// visible to the warp), nB / nTB = that geometry's node / triangle counts.
// `margin` = the world's margin (collision.hpp:78): box tests use Aabb3::overlaps(., margin)
// and, when margin > 0, a triangle pair counts when tri_tri_distance < margin
// (collision.cpp:312-313) instead of the staged intersection filters.
template <class GC>
__device__ __forceinline__ bool warp_collide(const GC& gc, const unsigned char* stage,
                                             int nB, int nTB, const WarpScratchView& ws,
                                             CheckCounters& cnt, double mg = 0.0) {
  const int lane = threadIdx.x & 31;
  SB_NP_MARK(np0);
  const double* P = reinterpret_cast<const double*>(stage);
  const double* I = reinterpret_cast<const double*>(stage + 96);
  const double* recbox = reinterpret_cast<const double*>(stage + 192);
  const uint32_t* recinfo = reinterpret_cast<const uint32_t*>(stage + 192 + 48 * nB);
  const double* rectri = reinterpret_cast<const double*>(stage + 192 + 56 * nB);
  const int8_t* recleaf = reinterpret_cast<const int8_t*>(stage + 192 + 56 * nB + 72 * nTB);
  if (lane < 12) {  // other_in_cand = inv(cand) * pose(ob), one entry per lane (shim order)
    const int i = lane >> 2, j = lane & 3;
    double s = I[4 * i + 0] * P[j];
    s = s + I[4 * i + 1] * P[4 + j];
    s = s + I[4 * i + 2] * P[8 + j];
    s = s + I[4 * i + 3] * (j == 3 ? 1.0 : 0.0);
    ws.M[lane] = s;
  }
  if (lane < gc.n_nodes) {
    ws.allowed[lane] = 0u;  // leaf-pair candidates (step 2)
    ws.H[lane] = 0u;        // intersecting leaf pairs (step 4)
  }
  __syncwarp();
  M34 M;
#pragma unroll
  for (int k = 0; k < 12; ++k) M.m[k] = ws.M[k];
  SB_NP_MARK(np1);
  SB_NP_ADD(0, np0, np1);

  const int nTA = gc.n_tris, nA = gc.n_nodes;

  // 1: lane b moves B's node b into A's frame (transform_aabb, collision.cpp:297-300; it
  // does not depend on the A node it meets)
  bool lb = false;
  if (lane < nB) {
    const double* nbox = recbox + 6 * lane;
    const uint32_t info = recinfo[2 * lane];
    double bmn[3], bmx[3];
    xform_aabb(M, nbox, nbox + 3, bmn, bmx);
    const double e0 = bmx[0] - bmn[0], e1 = bmx[1] - bmn[1], e2 = bmx[2] - bmn[2];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      ws.bb[6 * lane + c] = bmn[c];
      ws.bb[6 * lane + 3 + c] = bmx[c];
    }
    ws.e2b[lane] = (e0 * e0 + e1 * e1) + e2 * e2;
    lb = (info & 0xffu) == 0xffu;
    ws.cm[lane] = lb ? 0u : ((1u << (info & 0xffu)) | (1u << ((info >> 8) & 0xffu)));
    ws.lbb[lane] = recinfo[2 * lane + 1];
  }
  const uint32_t leafB = __ballot_sync(kFull, lb);
  if (lb) ws.leafb[__popc(leafB & ((1u << lane) - 1u))] = (int8_t)lane;
  const int nLB = __popc(leafB), nLA = gc.n_leaves;
  __syncwarp();

  // 2: leaf-box filter. The traversal tests triangles of a leaf pair only after that
  // pair's own box test passed, so a triangle pair whose leaf boxes are disjoint can never
  // be reported: collect the leaf pairs whose boxes overlap (ws.allowed[a] bit b).
  uint32_t anyc = 0u;
  {
    const int nlp = nLA * nLB;
    for (int k0 = 0; k0 < nlp; k0 += 32) {
      const int k = k0 + lane;
      bool ov = false;
      if (k < nlp) {
        const int a = gc.leaves[k / nLB], b = ws.leafb[k - (k / nLB) * nLB];
        const double* bb = ws.bb + 6 * b;
        ov = gc.bmin[a][0] <= bb[3] + mg && bb[0] <= gc.bmax[a][0] + mg &&
             gc.bmin[a][1] <= bb[4] + mg && bb[1] <= gc.bmax[a][1] + mg &&
             gc.bmin[a][2] <= bb[5] + mg && bb[2] <= gc.bmax[a][2] + mg;
      }
      if (__any_sync(kFull, ov)) {
        const uint32_t m = __ballot_sync(kFull, ov);
        anyc |= m;
        if (ov) atomicOr(ws.allowed + gc.leaves[k / nLB], 1u << ws.leafb[k - (k / nLB) * nLB]);
      }
    }
  }
  SB_NP_MARK(np1a);
  SB_NP_ADD(1, np1, np1a);
  if (!anyc) return false;
  __syncwarp();

  // 3: B's effective triangles into A's frame (transform_point, collision.cpp:308-310) and
  // their planes; A's planes are cached per launch.
  for (int v = lane; v < nTB * 3; v += 32) {
    const double* p = rectri + 3 * v;
    double* q = ws.qb + 3 * v;
    xform(M, p[0], p[1], p[2], q[0], q[1], q[2]);
  }
  for (int k = lane; k < nTB; k += 32) ws.tleafb[k] = recleaf[k];
  __syncwarp();
  for (int k = lane; k < nTB; k += 32) {
    const TriPlane P = tri_plane(ws.qb + 9 * k);
    double* pb = ws.pb + 5 * k;
    pb[0] = P.n[0];
    pb[1] = P.n[1];
    pb[2] = P.n[2];
    pb[3] = P.dc;
    pb[4] = P.tol;
  }
  const int ntp = nTA * nTB;
  __syncwarp();

  bool any = false;
  if (mg > 0.0) {  // 4': tri_tri_distance < margin over the candidate leaf pairs' triangles
    for (int k0 = 0; k0 < ntp; k0 += 32) {
      const int k = k0 + lane;
      bool hit = false;
      if (k < ntp) {
        const int ia = k / nTB, ib = k - ia * nTB;
        if ((ws.allowed[gc.tleaf[ia]] >> ws.tleafb[ib]) & 1u) {
          ++cnt.pairs;
          hit = tri_tri_distance(gc.ta[ia], ws.qb + 9 * ib) < mg;
        }
      }
      if (hit) atomicOr(ws.H + gc.tleaf[k / nTB], 1u << ws.tleafb[k - (k / nTB) * nTB]);
      any = __any_sync(kFull, hit) || any;
    }
  } else {
  // 4: staged tri_tri_intersect over the triangle pairs k = ia * nTB + ib of candidate
  // leaf pairs: filter 1 (B's plane vs A's vertices), filter 2 (A's plane vs B's
  // vertices), then the interval / coplanar rest.
  int n1 = 0;
  for (int k0 = 0; k0 < ntp; k0 += 32) {
    const int k = k0 + lane;
    bool pass = false;
    if (k < ntp) {
      const int ia = k / nTB, ib = k - ia * nTB;
      if ((ws.allowed[gc.tleaf[ia]] >> ws.tleafb[ib]) & 1u) {
        const double* pb = ws.pb + 5 * ib;
        double d0, d1, d2;
        plane_dists(pb, pb[3], pb[4], gc.ta[ia], d0, d1, d2);
        pass = straddles(d0, d1, d2);
        ++cnt.pairs;
      }
    }
    n1 = warp_append(pass, (uint16_t)k, ws.l1, n1);
  }
  __syncwarp();
  SB_NP_MARK(np1b_);
  SB_NP_ADD(6, np1a, np1b_);
  int n2 = 0;
  for (int j0 = 0; j0 < n1; j0 += 32) {
    const int j = j0 + lane;
    bool pass = false;
    int k = 0;
    if (j < n1) {
      k = ws.l1[j];
      const int ia = k / nTB, ib = k - ia * nTB;
      double d0, d1, d2;
      plane_dists(gc.pa[ia], gc.pa[ia][3], gc.pa[ia][4], ws.qb + 9 * ib, d0, d1, d2);
      pass = straddles(d0, d1, d2);
    }
    n2 = warp_append(pass, (uint16_t)k, ws.l2, n2);
  }
  __syncwarp();
  for (int j0 = 0; j0 < n2; j0 += 32) {
    const int j = j0 + lane;
    bool hit = false;
    int k = 0;
    if (j < n2) {
      k = ws.l2[j];
      const int ia = k / nTB, ib = k - ia * nTB;
      const double* pb = ws.pb + 5 * ib;
      const double* q = ws.qb + 9 * ib;
      double dp0, dp1, dp2, dq0, dq1, dq2;
      plane_dists(pb, pb[3], pb[4], gc.ta[ia], dp0, dp1, dp2);
      plane_dists(gc.pa[ia], gc.pa[ia][3], gc.pa[ia][4], q, dq0, dq1, dq2);
      hit = tri_tri_finish(gc.ta[ia], q, gc.pa[ia], pb, dp0, dp1, dp2, dq0, dq1, dq2);
    }
    if (hit) atomicOr(ws.H + gc.tleaf[k / nTB], 1u << ws.tleafb[k - (k / nTB) * nTB]);
    any = __any_sync(kFull, hit) || any;
  }
  }  // margin == 0
  SB_NP_MARK(np2);
  SB_NP_ADD(7, np1a, np2);  // filter 1 + filter 2 + rest (filter 1 alone in slot 6)
  if (!any) return false;
  __syncwarp();

  // 5: walk the pair DAG from (0,0) -- the reference's stack traversal with children read
  // as {left, left+1} (collision.cpp:285-329) -- level by level (one lane per frontier
  // pair; each node pair enters the frontier once), pruned to the node pairs whose
  // subtrees hold an intersecting leaf pair: rows[a] = { b : leaves_below(a) x
  // leaves_below(b) meets H }. Every path to such a leaf pair runs through these pairs
  // only, and an existential does not depend on the visiting order, so the verdict --
  // some intersecting leaf pair is reached with every box test on the way passing -- is
  // the reference's. Box tests and the descend rule are evaluated at visited pairs only.
  if (lane < nA) {
    uint32_t la = gc.lbelow[lane], RA = 0u;
    while (la) {
      RA |= ws.H[__ffs(la) - 1];
      la &= la - 1u;
    }
    uint32_t row = 0u;
    if (RA)
      for (int b = 0; b < nB; ++b)
        if (ws.lbb[b] & RA) row |= 1u << b;
    ws.allowed[lane] = row;
    ws.pend[lane] = lane == 0 ? 1u : 0u;  // visited
  }
  __syncwarp();
  SB_NP_MARK(np3);
  SB_NP_ADD(2, np2, np3);
  // Certificate: every path from (0,0) to an intersecting leaf pair runs through relevant
  // pairs only, and from any relevant pair the descend rule always continues towards one
  // (leaves_below of a node is the union of its children's). So if EVERY relevant pair
  // passes its box test, every intersecting leaf pair is reached: hit. Node boxes contain
  // their descendants', so this is the common case; a failing test (boxes that only touch
  // after rounding) falls back to the exact walk below.
  {
    bool all = true;
    const int np = nA * nB;
    for (int k0 = 0; k0 < np; k0 += 32) {
      const int k = k0 + lane;
      if (k < np) {
        const int a = k / nB, b = k - a * nB;
        if ((ws.allowed[a] >> b) & 1u) {
          const double* bb = ws.bb + 6 * b;
          ++cnt.nodes;
          all = all && gc.bmin[a][0] <= bb[3] + mg && bb[0] <= gc.bmax[a][0] + mg &&
                gc.bmin[a][1] <= bb[4] + mg && bb[1] <= gc.bmax[a][1] + mg &&
                gc.bmin[a][2] <= bb[5] + mg && bb[2] <= gc.bmax[a][2] + mg;
        }
      }
    }
    if (__all_sync(kFull, all)) {
      SB_NP_MARK(np4c);
      SB_NP_ADD(3, np3, np4c);
      SB_NP_ADD(5, 0, 1);
      return true;
    }
  }
  bool res = false;
  if (ws.allowed[0] & 1u) {
    uint16_t* F = ws.l1;
    uint16_t* G = ws.l2;
    if (lane == 0) F[0] = 0;
    int nf = 1;
    __syncwarp();
    while (nf > 0) {
      int ng = 0;
      bool hit = false;
      for (int i0 = 0; i0 < nf; i0 += 32) {
        const int i = i0 + lane;
        int ch0 = -1, ch1 = -1;  // children (a << 5 | b) entering the next level
        if (i < nf) {
          const int e = F[i];
          const int a = e >> 5, b = e & 31;
          ++cnt.nodes;
          const double* bb = ws.bb + 6 * b;
          if (gc.bmin[a][0] <= bb[3] + mg && bb[0] <= gc.bmax[a][0] + mg &&
              gc.bmin[a][1] <= bb[4] + mg && bb[1] <= gc.bmax[a][1] + mg &&
              gc.bmin[a][2] <= bb[5] + mg && bb[2] <= gc.bmax[a][2] + mg) {
            const bool la = (gc.leafmask >> a) & 1u, lb = (leafB >> b) & 1u;
            if (la && lb) {
              hit = (ws.H[a] >> b) & 1u;
            } else if (lb || (!la && gc.ext2[a] >= ws.e2b[b])) {  // descend A (collision.cpp:320)
              ch0 = (gc.c0[a] << 5) | b;
              ch1 = (gc.c1[a] << 5) | b;
            } else {
              const uint32_t cm = ws.cm[b];
              ch0 = (a << 5) | (__ffs(cm) - 1);
              ch1 = (a << 5) | (__ffs(cm & (cm - 1u)) - 1);
            }
            auto admit = [&](int c) {
              if (c < 0) return -1;
              const uint32_t bit = 1u << (c & 31);
              if (!(ws.allowed[c >> 5] & bit)) return -1;
              return (atomicOr(ws.pend + (c >> 5), bit) & bit) ? -1 : c;
            };
            ch0 = admit(ch0);
            ch1 = admit(ch1);
          }
        }
        if (__any_sync(kFull, hit)) {
          res = true;
          break;
        }
        ng = warp_append(ch0 >= 0, (uint16_t)ch0, G, ng);
        ng = warp_append(ch1 >= 0, (uint16_t)ch1, G, ng);
      }
      if (res) break;
      __syncwarp();
      uint16_t* t = F;
      F = G;
      G = t;
      nf = ng;
    }
  }
  SB_NP_MARK(np4);
  SB_NP_ADD(3, np3, np4);
  SB_NP_ADD(5, 0, 1);
  return res;
}

// Pooled check of the warp's 32 candidates (inactive lanes pass active = false but must
// still call). Returns the first colliding object id for this lane's candidate, or -1.
__device__ __forceinline__ int warp_check(const WorldView& w, const SbGeom& gA,
                                          const GeomCache& gc, bool active, const M34& pose,
                                          uint64_t inst, WarpScratch& wsf, double (*invs)[12],
                                          CheckCounters& cnt) {
  const int lane = threadIdx.x & 31;
  const WarpScratchView ws = wsf.view();
  double cmn[3] = {0, 0, 0}, cmx[3] = {0, 0, 0};
  if (active) {
    xform_aabb(pose, gA.box_c, gA.box_h, cmn, cmx);
    M34 inv;
    inverse_rigid(pose, inv);
#pragma unroll
    for (int k = 0; k < 12; ++k) invs[lane][k] = inv.m[k];
  }
  __syncwarp();
  int contact = -1;
  bool done = !active;
  for (int ob0 = 0; ob0 < w.n_objects; ob0 += 32) {
    uint32_t ovm = 0;
    if (!done) {
      uint32_t bits = w.enabled[sb_word_off(w, ob0 >> 5, inst)];
      while (bits) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1u;
        ++cnt.broad;
        const double2* bp =
            reinterpret_cast<const double2*>(w.box + sb_box_off(w, ob0 + b, inst));
        double2 b0 = bp[0], b1 = bp[1], b2 = bp[2];
        double omn[3] = {b0.x, b0.y, b1.x}, omx[3] = {b1.y, b2.x, b2.y};
        if (overlaps_m(cmn, cmx, omn, omx, w.margin)) ovm |= 1u << b;
      }
    }
    for (;;) {
      uint32_t pend = __ballot_sync(kFull, !done && ovm != 0u);
      if (!pend) break;
      while (pend) {
        const int L = __ffs(pend) - 1;
        pend &= pend - 1u;
        const uint32_t ovL = __shfl_sync(kFull, ovm, L);
        const uint64_t instL = __shfl_sync(kFull, inst, L);
        const int ob = ob0 + __ffs(ovL) - 1;
        const int4 gr = obj_grec(w, ob);
        unsigned char* st = stage_buf(wsf.bytes, kMaxEffTris, kMaxNodes, 0);
        warp_stage(w, gr, ob, instL, nullptr, st);
        if (lane < 12) reinterpret_cast<double*>(st + 96)[lane] = invs[L][lane];
        cp_async_wait<0>();
        __syncwarp();
        const bool hit = warp_collide(gc, st, gr.z, gr.w, ws, cnt, w.margin);
        if (lane == L) {
          ++cnt.narrow;
          ovm &= ovm - 1u;
          if (hit) {
            done = true;
            contact = ob;
          }
        }
        __syncwarp();
      }
    }
  }
  return contact;
}

}  // namespace sbd
