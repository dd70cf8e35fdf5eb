// Device-resident table layouts shared by the host preparation code and the kernels.
// Plain PODs, no CUDA types, so both g++ and nvcc compile them.
#pragma once

#include <stdint.h>

// One node of a geometry's effective BVH DAG (see sb_host.hpp).
struct SbNode {
  double bmin[3], bmax[3];  // node box, A-side overlap test (aabb.hpp:29-33)
  double c[3], h[3];        // 0.5*(min+max), 0.5*(max-min): B-side transform_aabb
  double ext2;              // box.extent().squaredNorm(): descent rule (collision.cpp:320)
  int32_t child0, child1;   // compact child ids, -1 for a leaf
  int32_t tri_start, tri_count;
  uint32_t leaves_below;    // bit k: effective leaf k lies under this node (or is it)
  int32_t pad;
};

struct SbTri {
  double v[9];   // p0.xyz p1.xyz p2.xyz in the mesh frame
  int32_t leaf;  // compact id of the leaf node holding it
  int32_t pad;
};

struct SbGeom {
  int32_t node_offset, n_nodes;
  int32_t tri_offset, n_tris;
  double box_c[3], box_h[3];   // local_box center / half extent (transform_aabb)
  double box_min[3], box_max[3];
};

// Region triangle for the exact-uniform polygon sampler (polygon.cpp:336-338).
struct SbRegionTri {
  double a[2], b[2], c[2];
};

#ifndef SB_MAX_ANCHORS
#define SB_MAX_ANCHORS 8          // include/scenebatch_b200.h
#endif
#ifndef SB_MAX_SUPPORT_VERTS
#define SB_MAX_SUPPORT_VERTS 16
#endif

// Placement descriptor consumed by the generation kernels.
struct SbPlacementDev {
  int32_t geom;            // candidate geometry
  int32_t object;          // world object id receiving accepted poses
  int32_t orientation;     // SB_ORIENT_*
  int32_t face_object;     // world object id of the face_to target, -1
  double z_off;            // rest_pose z offset (sampler.cpp:45-52)
  double support[12];      // support frame -> world, row-major 3x4
  double rect[4];          // support rect x0 y0 x1 y1
  // relation (relationships.hpp:18-38), single anchor
  int32_t anchor_object;   // world object id of the anchor, -1 = none
  int32_t distance_type, direction, frame;
  double direction_vector[2];
  double distance;
  double angle_threshold;  // <= 0: default
  uint64_t salt;           // placement index (Appendix C)
  double erode_r;          // apply_ratio_on_support radius of relation regions, 0 = none
  // support_world per instance (sampler.hpp:78-80): when non-null the frame of instance i
  // is support_inst[i] (row-major 3x4), else `support`; inv_support_inst[i] = its
  // inverse_rigid (anchor states in the support frame). support_object >= 0: the frames
  // are (pose of that world object) * support, refreshed per run (k_support_frames).
  const double* support_inst;
  const double* inv_support_inst;
  int32_t support_object;
  // every anchor of the relation (anchor_objects[0] == anchor_object): `middle` uses all
  // positions, the per-instance test all states (relationships.cpp:178-196)
  int32_t n_anchors;
  int32_t anchor_objects[SB_MAX_ANCHORS];
  // support polygon: bounds = bounds(support) (x0 y0 x1 y1 over its vertices); poly_n > 0:
  // the convex clip operand (counter-clockwise, vertex 0 first), else `rect`
  double bounds[4];
  int32_t poly_n;
  int32_t serial;          // region built by the serial per-instance path (big_region_lane)
  double poly_x[SB_MAX_SUPPORT_VERTS];
  double poly_y[SB_MAX_SUPPORT_VERTS];
};

// Device view of a collision world (plain pointers; built by the host World class).
// Per-instance state is INSTANCE-major: one instance's objects are contiguous, so a warp
// checking one candidate against its placed objects (lanes over objects) reads one
// contiguous burst (32 boxes = 1.5 KB), and accepting writes one record.
struct SbWorldView {
  uint64_t n;                // instances held on this device
  int32_t n_objects;
  int32_t n_words;           // enable-bit words in use = ceil(n_objects / 32)
  int32_t obj_stride;        // object capacity per instance (record stride)
  int32_t word_stride;       // enable-word capacity per instance
  double margin;             // CollisionWorld margin (collision.hpp:78)
  const int32_t* obj_geom;   // [n_objects]
  double* pose;              // [n][obj_stride][12]  row-major 3x4 [R | t]
  double* box;               // [n][obj_stride][6]   world AABB min xyz, max xyz
  uint32_t* enabled;         // [n][word_stride]     bit (object & 31) of word (object >> 5)
  const SbGeom* geoms;
  const SbNode* nodes;
  const SbTri* tris;
  // Compact B-side narrow-phase record per geometry (sb_brec_* below), staged into shared
  // memory with cp.async one pair ahead: grec[g] = {offset, length} in 16-byte units,
  // n_nodes, n_tris.
  const int32_t* grec;        // [n_geoms][4]
  const void* brec;           // 16-byte aligned records
};

// Per-instance XY occupancy grid of the engine's broad phase: cell (cx, cy) of instance i
// holds the enabled objects whose world AABB meets the cell (bit o of word o >> 5).
// Cell index = clamp(floor((x - x0) * inv_x), 0, g - 1) -- monotone in x, so a candidate box
// and an object box that overlap always share a cell; the exact AABB test then decides.
struct SbCellGrid {
  double x0, y0, inv_x, inv_y;
  int32_t g;        // cells per side (0 = no grid)
  int32_t words;    // words per cell (= enable words)
  uint32_t* cells;  // [n][g * g][words]
};

// Narrow-phase record of one geometry, 16-byte aligned, byte offsets:
//   [0, 48 nN)                 node boxes: c xyz, h xyz (double)
//   [48 nN, 56 nN)             node info: u32 child0 | child1 << 8 (0xff = none),
//                                         u32 leaves_below
//   [56 nN, 56 nN + 72 nT)     effective triangles: 9 doubles
//   [56 nN + 72 nT, + nT)      leaf id of each triangle (int8)
#ifdef __CUDACC__
__host__ __device__
#endif
inline constexpr int sb_brec_bytes(int n_nodes, int n_tris) {
  return (56 * n_nodes + 73 * n_tris + 15) & ~15;
}

#ifdef __CUDACC__
#define SB_HDI __host__ __device__ __forceinline__
#else
#define SB_HDI inline
#endif
SB_HDI uint64_t sb_pose_off(const SbWorldView& w, int32_t ob, uint64_t inst) {
  return (inst * (uint64_t)w.obj_stride + (uint64_t)ob) * 12u;
}
SB_HDI uint64_t sb_box_off(const SbWorldView& w, int32_t ob, uint64_t inst) {
  return (inst * (uint64_t)w.obj_stride + (uint64_t)ob) * 6u;
}
SB_HDI uint64_t sb_word_off(const SbWorldView& w, int32_t word, uint64_t inst) {
  return inst * (uint64_t)w.word_stride + (uint64_t)word;
}

#define SB_MAX_NODES_PER_GEOM 32   // effective DAG nodes (bitmask traversal width)
#define SB_MAX_EFF_TRIS 32         // reachable triangles per geometry (pooled narrow phase)
#define SB_REGION_MAX_VERTS 96     // per-instance constraint region ring capacity

// PCG32 jump table of the FIFO fast path (sbd::pcg_jump_draws): entry [k][d] = {mult, plus}
// of the LCG map "advance 6 * d * 256^k steps" (6 steps per polygon draw, rng.hpp:24-60;
// Brown's arbitrary-stride jump), table[(k * 256 + d) * 2 + {0, 1}].
#define SB_PCG_JUMP_LEVELS 4
SB_HDI void sb_pcg_jump_entry(uint64_t delta, uint64_t* mult, uint64_t* plus) {
  const uint64_t kMult = 6364136223846793005ULL, kInc = (0xda3e39cb94b95bdbULL << 1u) | 1u;
  uint64_t cur_mult = kMult, cur_plus = kInc, acc_mult = 1u, acc_plus = 0u;
  while (delta > 0) {
    if (delta & 1u) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1u) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1u;
  }
  *mult = acc_mult;
  *plus = acc_plus;
}
inline void sb_pcg_jump_table_host(uint64_t* table) {
  for (int k = 0; k < SB_PCG_JUMP_LEVELS; ++k)
    for (uint64_t d = 0; d < 256; ++d)
      sb_pcg_jump_entry(6u * (d << (8 * k)), &table[(k * 256 + d) * 2], &table[(k * 256 + d) * 2 + 1]);
}
