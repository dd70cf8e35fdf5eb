// Internal to the host runtime (sb_*_rt.cpp, sb_runtime.cpp): shared helpers of the C ABI
// implementation -- CUDA error checks, device / pinned buffers, status mapping.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/scenebatch_b200.h"
#include "sb_graph.h"
#include "sb_host.hpp"
#include "sb_reach.h"
#include "sb_kernels.h"
#include "sb_place.h"
#include "sb_poly.h"
#include "sb_region.h"
#include "sb_layout.h"

namespace sbrt {


inline thread_local std::string g_error;

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error(std::string("CUDA: ") + what + ": " + cudaGetErrorString(e));
  }
}

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class T>
struct DevArray {
  T* p = nullptr;
  size_t count = 0;
  DevArray() = default;
  DevArray(const DevArray&) = delete;
  DevArray& operator=(const DevArray&) = delete;
  ~DevArray() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    count = 0;
  }
  void alloc(size_t n) {
    release();
    if (n == 0) return;
    cuda_check(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
    count = n;
  }
  void ensure(size_t n) {
    if (n > count) alloc(n);
  }
};

template <class T>
struct PinnedArray {
  T* p = nullptr;
  size_t count = 0;
  ~PinnedArray() {
    if (p) cudaFreeHost(p);
  }
  void ensure(size_t n) {
    if (n <= count) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cuda_check(cudaMallocHost(&p, n * sizeof(T)), "cudaMallocHost");
    count = n;
  }
};

inline void require_homogeneous(const double* p) {
  if (p[3] != 0.0 || p[7] != 0.0 || p[11] != 0.0 || p[15] != 1.0)
    throw std::invalid_argument("pose bottom row must be exactly (0,0,0,1)");
  for (int k = 0; k < 16; ++k)
    if (!std::isfinite(p[k])) throw std::invalid_argument("pose must be finite");
}

// inverse_rigid (transform.hpp:63-69) on the host, same operation order as the device.
inline void inverse_rigid34(const double* colmajor16, double out[12]) {
  double R[3][3], t[3];
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) R[i][j] = colmajor16[4 * j + i];
    t[i] = colmajor16[12 + i];
  }
  for (int i = 0; i < 3; ++i) {
    for (int k = 0; k < 3; ++k) out[4 * i + k] = R[k][i];
    double s = (-R[0][i]) * t[0];
    s = s + (-R[1][i]) * t[1];
    s = s + (-R[2][i]) * t[2];
    out[4 * i + 3] = s;
  }
}

inline void colmajor_to_34(const double* c, double out[12]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 4; ++j) out[4 * i + j] = c[4 * j + i];
}

inline int current_device_checked(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw CudaError("no CUDA device available (this build has no CPU fallback)");
  }
  if (device < 0 || device >= count) throw std::out_of_range("device index out of range");
  cudaDeviceProp prop;
  cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10)
    throw CudaError("device " + std::to_string(device) + " is sm_" + std::to_string(prop.major) +
                    std::to_string(prop.minor) + "; this build targets sm_100a only");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  return device;
}

// Anchor count of an sb_relation (RelationshipSpec::anchors = {anchor, extra_anchors...}).
inline int relation_anchor_count(const sb_relation& r) {
  if (r.anchor < 0) return 0;
  if (r.n_extra_anchors < 0 || r.n_extra_anchors > SB_MAX_ANCHORS - 1)
    throw std::invalid_argument("relationship: n_extra_anchors outside [0, 7]");
  return 1 + r.n_extra_anchors;
}

// RelationshipSpec::validate (relationships.cpp:59-76), then the relation fields of the
// device record (anchor objects are filled by the caller). Returns whether region_for()
// needs the serial big-ring region path for its SHAPE: a full annulus with a hole (theta =
// pi, min_r > 0, bridged hole) or an annular sector wide enough to outgrow the group path's
// ring (SB_REGION_MAX_VERTS).
inline bool relation_to_dev(const sb_relation& r, SbPlacementDev& d) {
  const int na = relation_anchor_count(r);
  if (r.distance < 0.0) throw std::invalid_argument("relationship: distance must be >= 0");
  if (r.angle_threshold > M_PI) throw std::invalid_argument("relationship: angle_threshold outside (0, pi]");
  if (r.distance_type < SB_DIST_NONE || r.distance_type > SB_DIST_MIDDLE)
    throw std::invalid_argument("relationship: distance_type");
  const bool dist = r.distance_type == SB_DIST_GREATER || r.distance_type == SB_DIST_LESS ||
                    r.distance_type == SB_DIST_EQUAL;
  if (r.distance_type == SB_DIST_MIDDLE) {
    if (na < 2) throw std::invalid_argument("relationship: middle requires at least 2 anchors");
  } else if (dist && na != 1) {
    throw std::invalid_argument("relationship: greater/less/equal require exactly 1 anchor");
  }
  if (r.direction != SB_DIR_NONE && na != 1) throw std::invalid_argument("relationship: direction requires exactly 1 anchor");
  if (r.direction < SB_DIR_NONE || r.direction > SB_DIR_VECTOR) throw std::invalid_argument("relationship: direction");
  if (r.direction == SB_DIR_VECTOR &&
      std::sqrt(r.direction_vector[0] * r.direction_vector[0] + r.direction_vector[1] * r.direction_vector[1]) < 1e-12)
    throw std::invalid_argument("relationship: zero-length direction vector");
  if (r.distance_type == SB_DIST_LESS && !(0.0 < r.distance))
    throw std::invalid_argument("annulus_sector: min_r >= max_r");
  d.distance_type = r.distance_type;
  d.direction = r.direction;
  d.frame = r.frame;
  d.direction_vector[0] = r.direction_vector[0];
  d.direction_vector[1] = r.direction_vector[1];
  d.distance = r.distance;
  d.angle_threshold = r.angle_threshold;
  d.n_anchors = na;
  if (na == 0 || r.distance_type == SB_DIST_MIDDLE) return false;
  const double theta = r.angle_threshold > 0 ? r.angle_threshold : (r.direction == SB_DIR_NONE ? M_PI : M_PI / 4);
  double min_r = 0.0;  // distance_band (relationships.cpp:101-122)
  if (r.distance_type == SB_DIST_GREATER) min_r = r.distance;
  if (r.distance_type == SB_DIST_EQUAL) min_r = std::max(0.0, r.distance - std::max(0.05 * r.distance, 0.01));
  const bool full = theta >= M_PI - 1e-12;
  if (full && min_r > 0.0) return true;  // annulus with a hole
  // ring size of annulus_sector + up to 8 clip vertices (+1 arc point of rounding slack)
  const double step = 5.0 * M_PI / 180.0;
  const int arc = full ? 73 : static_cast<int>(std::ceil(2.0 * theta / step)) + 2;
  const int ring = arc + (!full && min_r > 0.0 ? arc : 1) + 8;
  return ring > SB_REGION_MAX_VERTS;  // the serial big-ring path
}

// The support polygon of an sb_support into the device record: bounds(support) over its
// vertices, and the clip operand -- the rect (poly_n = 0) when the polygon is an
// axis-aligned rectangle (the shim clips those exactly as a rect), else the convex ring
// corrected to counter-clockwise with vertex 0 first (bg::correct). Returns the ring as
// given (the canonical sampler triangulates it as is).
inline std::vector<std::array<double, 2>> support_to_dev(const sb_support& sup, SbPlacementDev& d) {
  std::vector<std::array<double, 2>> ring;
  if (sup.n_polygon == 0) {
    const double* rc = sup.rect;
    ring = {{rc[0], rc[1]}, {rc[2], rc[1]}, {rc[2], rc[3]}, {rc[0], rc[3]}};
  } else {
    if (sup.n_polygon < 3 || sup.n_polygon > SB_MAX_SUPPORT_VERTS || !sup.polygon_xy)
      throw std::invalid_argument("support polygon needs 3..16 vertices");
    for (uint32_t k = 0; k < sup.n_polygon; ++k) {
      const double x = sup.polygon_xy[2 * k], y = sup.polygon_xy[2 * k + 1];
      if (!std::isfinite(x) || !std::isfinite(y)) throw std::invalid_argument("support polygon must be finite");
      ring.push_back({x, y});
    }
  }
  const size_t k = ring.size();
  double x0 = ring[0][0], x1 = ring[0][0], y0 = ring[0][1], y1 = ring[0][1];
  double bx0 = HUGE_VAL, by0 = HUGE_VAL, bx1 = -HUGE_VAL, by1 = -HUGE_VAL;  // Aabb2::expand
  for (const auto& v : ring) {
    x0 = std::fmin(x0, v[0]);
    x1 = std::fmax(x1, v[0]);
    y0 = std::fmin(y0, v[1]);
    y1 = std::fmax(y1, v[1]);
    bx0 = std::min(bx0, v[0]);
    by0 = std::min(by0, v[1]);
    bx1 = std::max(bx1, v[0]);
    by1 = std::max(by1, v[1]);
  }
  d.bounds[0] = bx0;
  d.bounds[1] = by0;
  d.bounds[2] = bx1;
  d.bounds[3] = by1;
  bool is_rect = k == 4;
  for (const auto& v : ring)
    if (!((v[0] == x0 || v[0] == x1) && (v[1] == y0 || v[1] == y1))) is_rect = false;
  d.poly_n = 0;
  if (is_rect) {
    d.rect[0] = x0;  // intersect_rect takes min / max again
    d.rect[1] = y0;
    d.rect[2] = x1;
    d.rect[3] = y1;
    return ring;
  }
  std::vector<std::array<double, 2>> c = ring;  // bg::correct: counter-clockwise, v0 first
  double a = 0.0;
  for (size_t i = 0; i < k; ++i) a += c[i][0] * c[(i + 1) % k][1] - c[(i + 1) % k][0] * c[i][1];
  if (0.5 * a < 0.0) std::reverse(c.begin() + 1, c.end());
  for (size_t i = 0; i < k; ++i) {
    const auto& o = c[(i + k - 1) % k];
    const auto& p = c[i];
    const auto& q = c[(i + 1) % k];
    if ((p[0] - o[0]) * (q[1] - o[1]) - (p[1] - o[1]) * (q[0] - o[0]) < 0.0)
      throw std::invalid_argument("support polygon must be convex (non-convex supports are out of scope)");
  }
  d.poly_n = static_cast<int32_t>(k);
  for (size_t i = 0; i < k; ++i) {
    d.poly_x[i] = c[i][0];
    d.poly_y[i] = c[i][1];
  }
  d.rect[0] = x0;
  d.rect[1] = y0;
  d.rect[2] = x1;
  d.rect[3] = y1;
  return ring;
}


template <class F>
sb_status guard(F&& f) {
  try {
    f();
    return SB_OK;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return SB_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_error = e.what();
    return SB_ERR_OUT_OF_RANGE;
  } catch (const std::logic_error& e) {
    g_error = e.what();
    return SB_ERR_LOGIC;
  } catch (const CudaError& e) {
    g_error = e.what();
    return SB_ERR_CUDA;
  } catch (const std::exception& e) {
    g_error = e.what();
    std::string w = e.what();
    return w.rfind("CUDA", 0) == 0 ? SB_ERR_CUDA : SB_ERR_RUNTIME;
  }
}

inline bool homogeneous16(const double* m) {  // is_homogeneous (transform.hpp:28-30)
  return m[3] == 0.0 && m[7] == 0.0 && m[11] == 0.0 && m[15] == 1.0;
}

}  // namespace sbrt

using namespace sbrt;
