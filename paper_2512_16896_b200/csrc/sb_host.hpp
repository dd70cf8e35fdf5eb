// Host-side geometry preparation for the B200 hot path (C++, no CUDA).
//
// Everything here runs once per geometry / support (cold start), and produces the
// flat, device-ready tables the kernels read. Arithmetic is written operation by
// operation so that results are bit-identical to the reference built without FMA
// (the reference's Eigen expressions reduce left to right -- see oracle/shim/Eigen/Dense).
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "sb_layout.h"

namespace sbh {

using V3 = std::array<double, 3>;
using V2 = std::array<double, 2>;

struct Mesh {
  std::vector<V3> v;
  std::vector<std::array<uint32_t, 3>> t;
};

// trimesh.cpp:40-104 (make_box / make_cylinder / make_sphere)
Mesh make_box(double sx, double sy, double sz);
Mesh make_cylinder(double radius, double height, int segments);
Mesh make_sphere(double radius, int stacks, int slices);
// load_obj (config.hpp:88-90, declared by the reference, defined here): the Wavefront OBJ
// subset -- `v x y z [w]` and `f a b c ...` records (a = i, i/j, i//k or i/j/k, 1-based,
// negative = relative to the end), polygon faces fan-triangulated (a, b, c), (a, c, d), ...;
// every other record ignored. Errors (std::runtime_error) carry "path:line:".
Mesh load_obj(const std::string& path);
Mesh parse_obj(const std::string& text, const std::string& name);
// trimesh.cpp:120-135
uint64_t mesh_fingerprint(const Mesh& m);
// trimesh.cpp:16-29 (returns number removed)
std::size_t drop_degenerate(Mesh& m, double area_eps = 1e-12);
// TriMesh::aabb (trimesh.cpp:10-14); box[0..2] = min, box[3..5] = max
void mesh_aabb(const Mesh& m, double box[6]);

// Reference-identical MeshBvh (collision.cpp:217-281), then the "effective DAG": the
// nodes reachable from the root when children are read as {left, left+1}
// (collision.hpp:46, collision.cpp:320-324) -- the reference's actual traversal graph.
struct EffectiveBvh {
  std::vector<SbNode> nodes;     // compact, topologically ordered (parents first)
  std::vector<SbTri> tris;       // triangles of reachable leaves, grouped per leaf
  int full_nodes = 0;            // nodes in the reference BVH
  int full_depth = 0;            // MeshBvh::depth()
  int reachable_tris = 0;
};
EffectiveBvh build_effective_bvh(const Mesh& m);

// triangulate(Polygon2D) for a single simple ring (polygon.cpp:260-368, no holes).
std::vector<std::array<V2, 3>> triangulate_ring(const std::vector<V2>& ring);
// PolygonSampler ctor (polygon.cpp:370-388): triangles with positive area + cum table.
struct SamplerTable {
  std::vector<SbRegionTri> tris;
  std::vector<double> cum;
};
SamplerTable sampler_table(const std::vector<std::vector<V2>>& part_rings);

// erode() (polygon.cpp:101-113) of a convex counter-clockwise ring by r, as the oracle's
// Boost stand-in defines buffer(-r): edges move inward by r along their unit normals,
// vertex i = intersection of offset edges i-1 and i; empty when eroded away.
std::vector<V2> erode_convex(const std::vector<V2>& ring, double r);

// splitmix64 / make_stream seed derivation (rng.hpp:9-21,63-67)
uint64_t mix64(uint64_t x);

// extract_all_support_surfaces (surface.cpp:53-142): upward facets (normal within 5 deg of
// +z) clustered by shared edges (quantized 1e-9 positions), each cluster's xy projection
// merged with the union stand-in (union_of, polygon.cpp:121-125, as oracle/shim defines
// bg::union_), parts below 1e-4 m^2 dropped, the roof flag by a majority vote of 16 upward
// ray casts from sampler draws; stable-sorted by area, largest first.
struct Surface {
  std::vector<V2> polygon;  // exterior ring in the z = z_top plane
  double z_top = 0.0;
  double area = 0.0;
  bool roofed = false;
};
std::vector<Surface> extract_all_support_surfaces(const Mesh& m);

}  // namespace sbh
