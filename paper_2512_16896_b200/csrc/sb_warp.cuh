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
// [0] pose load + M, [1] triangle transform + all triangle pairs, [2] node transform +
// node-pair tests (hits only), [3] DAG walk, [4] reached-hit check, [5] pairs.
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

struct WarpScratch {
  double M[12];                // other_in_self of the pair under test
  double qb[kMaxEffTris][9];   // B's effective triangles moved into A's frame
  double bb[kMaxNodes][6];     // B's effective node boxes in A's frame
  double e2b[kMaxNodes];       // their squared extents
  uint32_t cm[kMaxNodes];      // B node -> mask of its effective children (0 for leaves)
  uint32_t allowed[kMaxNodes]; // allowed[a] bit b: leaf pair reached by the traversal
  int8_t tleafb[kMaxEffTris];
  uint32_t hitw[kMaxEffTris * kMaxEffTris / 32];  // intersecting triangle pairs (bitset)
};

// Candidate geometry (uniform per launch), staged in shared memory once per block.
struct GeomCache {
  double ta[kMaxEffTris][9];
  double bmin[kMaxNodes][3], bmax[kMaxNodes][3];
  double ext2[kMaxNodes];
  int8_t c0[kMaxNodes], c1[kMaxNodes];
  int8_t tleaf[kMaxEffTris];
  uint32_t leafmask;
  int n_tris, n_nodes;
};

__device__ __forceinline__ void load_geom_cache(const WorldView& w, const SbGeom& gA,
                                                GeomCache& gc) {
  const SbTri* t = w.tris + gA.tri_offset;
  const SbNode* nd = w.nodes + gA.node_offset;
  for (int k = threadIdx.x; k < gA.n_tris * 9; k += blockDim.x) gc.ta[k / 9][k % 9] = t[k / 9].v[k % 9];
  for (int k = threadIdx.x; k < gA.n_tris; k += blockDim.x) gc.tleaf[k] = (int8_t)t[k].leaf;
  for (int k = threadIdx.x; k < gA.n_nodes; k += blockDim.x) {
    for (int c = 0; c < 3; ++c) {
      gc.bmin[k][c] = nd[k].bmin[c];
      gc.bmax[k][c] = nd[k].bmax[c];
    }
    gc.ext2[k] = nd[k].ext2;
    gc.c0[k] = (int8_t)nd[k].child0;
    gc.c1[k] = (int8_t)nd[k].child1;
  }
  if (threadIdx.x == 0) {
    uint32_t lm = 0;
    for (int k = 0; k < gA.n_nodes; ++k)
      if (nd[k].child0 < 0) lm |= 1u << k;
    gc.leafmask = lm;
    gc.n_tris = gA.n_tris;
    gc.n_nodes = gA.n_nodes;
  }
}

// Warp-cooperative MeshBvh::collide for one (candidate, object) pair. All 32 lanes call
// it with identical arguments.
__device__ __forceinline__ bool warp_collide(const WorldView& w, const GeomCache& gc,
                                             int32_t ob, uint64_t inst, const double* I,
                                             WarpScratch& ws, CheckCounters& cnt) {
  const int lane = threadIdx.x & 31;
  SB_NP_MARK(np0);
  const SbGeom gB = w.geoms[w.obj_geom[ob]];
  const double* P = w.pose + sb_pose_off(w, ob, inst);
  if (lane < 12) {  // other_in_cand = inv(cand) * pose(ob), one entry per lane (shim order)
    const int i = lane >> 2, j = lane & 3;

    double s = I[4 * i + 0] * P[j];
    s = s + I[4 * i + 1] * P[4 + j];
    s = s + I[4 * i + 2] * P[8 + j];
    s = s + I[4 * i + 3] * (j == 3 ? 1.0 : 0.0);
    ws.M[lane] = s;
  }
  __syncwarp();
  M34 M;
#pragma unroll
  for (int k = 0; k < 12; ++k) M.m[k] = ws.M[k];
  SB_NP_MARK(np1);
  SB_NP_ADD(0, np0, np1);

  // 1: B's effective triangles into A's frame (transform_point, collision.cpp:308-310).
  // Then, when the node-pair grid is large (deep effective DAGs, e.g. sphere sets), test
  // every effective triangle pair first: no intersecting pair in Eff(A) x Eff(B) means the
  // reference cannot report a hit (it only tests pairs of reachable leaves), so node tests
  // and the DAG walk run only when some pair intersects. Small grids (box-box: 4 x 4) cull
  // first and test only the reached leaf pairs.
  const SbTri* tB = w.tris + gB.tri_offset;
  const int nTB = gB.n_tris, nTA = gc.n_tris;
  const int nA = gc.n_nodes, nB = gB.n_nodes;
  const bool tri_first = nA * nB > 16;
  for (int v = lane; v < nTB * 3; v += 32) {
    const double* p = tB[v / 3].v + 3 * (v % 3);
    double* q = ws.qb[v / 3] + 3 * (v % 3);
    xform(M, p[0], p[1], p[2], q[0], q[1], q[2]);
  }
  for (int k = lane; k < nTB; k += 32) ws.tleafb[k] = (int8_t)tB[k].leaf;
  __syncwarp();
  const int ntp = nTA * nTB;
  if (tri_first) {
    bool any_hit = false;
    for (int k0 = 0; k0 < ntp; k0 += 32) {
      const int idx = k0 + lane;
      bool hit = false;
      if (idx < ntp) {
        const int ia = idx / nTB, ib = idx - ia * nTB;
        hit = tri_tri_intersect(gc.ta[ia], ws.qb[ib]);
      }
      const uint32_t hm = __ballot_sync(kFull, hit);
      if (lane == 0) ws.hitw[k0 >> 5] = hm;
      any_hit = any_hit || hm != 0u;
    }
    if (lane == 0) cnt.pairs += ntp;
    if (!any_hit) {
      SB_NP_MARK(npx);
      SB_NP_ADD(1, np1, npx);
      return false;
    }
    __syncwarp();
  }
  SB_NP_MARK(np2);
  SB_NP_ADD(1, np1, np2);

  // 2a: lane b moves B's node b into A's frame (independent of the A node it meets)
  const SbNode* nodesB = w.nodes + gB.node_offset;
  bool lb = false;
  if (lane < nB) {
    const SbNode& nb = nodesB[lane];
    double bmn[3], bmx[3];
    xform_aabb(M, nb.c, nb.h, bmn, bmx);
    const double e0 = bmx[0] - bmn[0], e1 = bmx[1] - bmn[1], e2 = bmx[2] - bmn[2];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      ws.bb[lane][c] = bmn[c];
      ws.bb[lane][3 + c] = bmx[c];
    }
    ws.e2b[lane] = (e0 * e0 + e1 * e1) + e2 * e2;
    lb = nb.child0 < 0;
    ws.cm[lane] = lb ? 0u : ((1u << nb.child0) | (1u << nb.child1));
  }
  const uint32_t leafB = __ballot_sync(kFull, lb);
  __syncwarp();

  // 2: pass(a,b) = na.box.overlaps(nb_in_a) and the descend rule
  // desc(a,b) = leaf(nb) || (!leaf(na) && ext2(na) >= ext2(nb_in_a)) for all (a, b),
  // 32 pairs per ballot; lane a collects row a (pair k = a * nB + b).
  uint32_t rpass = 0u, rdesc = 0u;
  const int np = nA * nB;
  for (int k0 = 0; k0 < np; k0 += 32) {
    const int k = k0 + lane;
    bool pb = false, db = false;
    if (k < np) {
      const int a = k / nB, bi = k - a * nB;
      const double* bb = ws.bb[bi];
      pb = gc.bmin[a][0] <= bb[3] && bb[0] <= gc.bmax[a][0] && gc.bmin[a][1] <= bb[4] &&
           bb[1] <= gc.bmax[a][1] && gc.bmin[a][2] <= bb[5] && bb[2] <= gc.bmax[a][2];
      db = ((leafB >> bi) & 1u) || (!((gc.leafmask >> a) & 1u) && gc.ext2[a] >= ws.e2b[bi]);
    }
    const uint32_t P = __ballot_sync(kFull, pb), D = __ballot_sync(kFull, db);
    if (lane < nA) {
      const int lo = lane * nB;
      const int s0 = lo > k0 ? lo : k0;
      const int e0 = (lo + nB) < (k0 + 32) ? (lo + nB) : (k0 + 32);
      if (s0 < e0) {
        const int len = e0 - s0;
        const uint32_t mk = len >= 32 ? 0xffffffffu : ((1u << len) - 1u);
        rpass |= ((P >> (s0 - k0)) & mk) << (s0 - lo);
        rdesc |= ((D >> (s0 - k0)) & mk) << (s0 - lo);
      }
    }
  }
  SB_NP_MARK(np3);
  SB_NP_ADD(2, np2, np3);

  // 3: walk the pair DAG from (0,0) in lexicographic order (a topological order: every
  // child id exceeds its parent's). Lane a owns the pending row of A node a; descending A
  // forwards the row's bits to the lanes of A's effective children.
  {
    uint32_t pend = lane == 0 ? 1u : 0u, allowed = 0u;
    const bool la = lane < nA && ((gc.leafmask >> lane) & 1u);
    const int c0 = lane < nA ? gc.c0[lane] : -1, c1 = lane < nA ? gc.c1[lane] : -1;
    unsigned visited = 0;
    for (int a = 0; a < nA; ++a) {
      uint32_t down = 0u;
      if (lane == a) {
        while (pend) {
          const int bi = __ffs(pend) - 1;
          pend &= pend - 1u;
          ++visited;
          if (!((rpass >> bi) & 1u)) continue;
          if (la && ((leafB >> bi) & 1u)) allowed |= 1u << bi;
          else if ((rdesc >> bi) & 1u) down |= 1u << bi;
          else pend |= ws.cm[bi];
        }
      }
      down = __shfl_sync(kFull, down, a);
      const int d0 = __shfl_sync(kFull, c0, a), d1 = __shfl_sync(kFull, c1, a);
      if (down && (lane == d0 || lane == d1)) pend |= down;
    }
    if (lane < nA) ws.allowed[lane] = allowed;
    cnt.nodes += visited;
  }
  __syncwarp();
  SB_NP_MARK(np4);
  SB_NP_ADD(3, np3, np4);

  // 4: tri-first: does some intersecting pair lie in a reached leaf pair? Cull-first:
  // test the triangle pairs of the reached leaf pairs.
  bool ok = false;
  unsigned tests = 0;
  for (int k0 = 0; k0 < ntp; k0 += 32) {
    const int idx = k0 + lane;
    if (idx >= ntp) continue;
    const int ia = idx / nTB, ib = idx - ia * nTB;
    const bool reached = (ws.allowed[gc.tleaf[ia]] >> ws.tleafb[ib]) & 1u;
    if (tri_first) {
      ok = ok || (reached && ((ws.hitw[k0 >> 5] >> lane) & 1u));
    } else if (reached) {
      ++tests;
      ok = ok || tri_tri_intersect(gc.ta[ia], ws.qb[ib]);
    }
  }
  cnt.pairs += tests;
  const bool res = __any_sync(kFull, ok);
  SB_NP_MARK(np5);
  SB_NP_ADD(4, np4, np5);
  SB_NP_ADD(5, 0, 1);
  return res;
}

// Pooled check of the warp's 32 candidates (inactive lanes pass active = false but must
// still call). Returns the first colliding object id for this lane's candidate, or -1.
__device__ __forceinline__ int warp_check(const WorldView& w, const SbGeom& gA,
                                          const GeomCache& gc, bool active, const M34& pose,
                                          uint64_t inst, WarpScratch& ws, double (*invs)[12],
                                          CheckCounters& cnt) {
  const int lane = threadIdx.x & 31;
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
        if (overlaps(cmn, cmx, omn, omx)) ovm |= 1u << b;
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
        const bool hit = warp_collide(w, gc, ob, instL, invs[L], ws, cnt);
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
