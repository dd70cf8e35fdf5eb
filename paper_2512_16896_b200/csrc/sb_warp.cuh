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
constexpr int kMaxEffTris = SB_MAX_EFF_TRIS;  // host-checked at registration
constexpr int kMaxNodes = SB_MAX_NODES_PER_GEOM;

struct WarpScratch {
  double M[12];                // other_in_self of the pair under test
  double qb[kMaxEffTris][9];   // B's effective triangles moved into A's frame
  uint32_t pass[kMaxNodes];    // pass[a] bit b: A node a overlaps B node b (in A's frame)
  uint32_t desc[kMaxNodes];    // desc[a] bit b: descend A at pair (a, b)
  uint32_t allowed[kMaxNodes]; // allowed[a] bit b: leaf pair reached by the traversal
  uint32_t pend[kMaxNodes];
  int8_t c0b[kMaxNodes], c1b[kMaxNodes];
  int8_t tleafb[kMaxEffTris];
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

  // 1-2: node pair box tests and descend decisions
  const int nA = gc.n_nodes, nB = gB.n_nodes;
  const SbNode* nodesB = w.nodes + gB.node_offset;
  bool lb = false;
  double bmn[3] = {0, 0, 0}, bmx[3] = {0, 0, 0}, ext2b = 0.0;
  if (lane < nB) {
    const SbNode& nb = nodesB[lane];
    xform_aabb(M, nb.c, nb.h, bmn, bmx);
    const double e0 = bmx[0] - bmn[0], e1 = bmx[1] - bmn[1], e2 = bmx[2] - bmn[2];
    ext2b = (e0 * e0 + e1 * e1) + e2 * e2;
    lb = nb.child0 < 0;
    ws.c0b[lane] = (int8_t)nb.child0;
    ws.c1b[lane] = (int8_t)nb.child1;
  }
  const uint32_t leafB = __ballot_sync(kFull, lb);
  for (int a = 0; a < nA; ++a) {
    const bool la = (gc.leafmask >> a) & 1u;
    const bool p = lane < nB && gc.bmin[a][0] <= bmx[0] && bmn[0] <= gc.bmax[a][0] &&
                   gc.bmin[a][1] <= bmx[1] && bmn[1] <= gc.bmax[a][1] &&
                   gc.bmin[a][2] <= bmx[2] && bmn[2] <= gc.bmax[a][2];
    const bool d = lb || (!la && gc.ext2[a] >= ext2b);
    const uint32_t pm = __ballot_sync(kFull, p);
    const uint32_t dm = __ballot_sync(kFull, d);
    if (lane == 0) {
      ws.pass[a] = pm;
      ws.desc[a] = dm;
    }
  }
  // B's effective triangles into A's frame (transform_point per vertex, collision.cpp:308-310)
  const SbTri* tB = w.tris + gB.tri_offset;
  const int nTB = gB.n_tris, nTA = gc.n_tris;
  for (int v = lane; v < nTB * 3; v += 32) {
    const double* p = tB[v / 3].v + 3 * (v % 3);
    double* q = ws.qb[v / 3] + 3 * (v % 3);
    xform(M, p[0], p[1], p[2], q[0], q[1], q[2]);
  }
  for (int k = lane; k < nTB; k += 32) ws.tleafb[k] = (int8_t)tB[k].leaf;
  __syncwarp();

  // 3: walk the pair DAG (lexicographic order is topological: children ids > parent ids)
  if (lane == 0) {
    for (int a = 0; a < nA; ++a) {
      ws.pend[a] = 0u;
      ws.allowed[a] = 0u;
    }
    ws.pend[0] = 1u;
    uint32_t visited = 0;
    for (int a = 0; a < nA; ++a) {
      uint32_t pend = ws.pend[a];
      const uint32_t pass = ws.pass[a], desc = ws.desc[a];
      const bool la = (gc.leafmask >> a) & 1u;
      uint32_t allowed = 0u;
      while (pend) {
        const int b = __ffs(pend) - 1;
        pend &= pend - 1u;
        ++visited;
        if (!((pass >> b) & 1u)) continue;
        if (la && ((leafB >> b) & 1u)) {
          allowed |= 1u << b;
        } else if ((desc >> b) & 1u) {
          ws.pend[gc.c0[a]] |= 1u << b;
          ws.pend[gc.c1[a]] |= 1u << b;
        } else {
          pend |= (1u << ws.c0b[b]) | (1u << ws.c1b[b]);
        }
      }
      ws.allowed[a] = allowed;
    }
    cnt.nodes += visited;
  }
  __syncwarp();

  // 4: triangle pairs of the reached leaf pairs
  bool hit = false;
  unsigned tests = 0;
  for (int idx = lane; idx < nTA * nTB; idx += 32) {
    const int ia = idx / nTB, ib = idx - ia * nTB;
    if ((ws.allowed[gc.tleaf[ia]] >> ws.tleafb[ib]) & 1u) {
      ++tests;
      hit = hit || tri_tri_intersect(gc.ta[ia], ws.qb[ib]);
    }
  }
  cnt.pairs += tests;
  return __any_sync(kFull, hit);
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
