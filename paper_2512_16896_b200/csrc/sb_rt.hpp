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

// RelationshipSpec::validate (relationships.cpp:59-76) for the single-anchor subset, then
// the relation fields of the device record. Returns whether region_for() needs the serial
// big-ring region path: a full annulus with a hole (theta = pi, min_r > 0, bridged hole) or
// an annular sector wide enough to outgrow the group path's ring (SB_REGION_MAX_VERTS).
inline bool relation_to_dev(const sb_relation& r, SbPlacementDev& d) {
  if (r.distance < 0.0) throw std::invalid_argument("relationship: distance must be >= 0");
  if (r.angle_threshold > M_PI) throw std::invalid_argument("relationship: angle_threshold outside (0, pi]");
  const bool dist = r.distance_type == SB_DIST_GREATER || r.distance_type == SB_DIST_LESS ||
                    r.distance_type == SB_DIST_EQUAL;
  if (r.distance_type < SB_DIST_NONE || r.distance_type > SB_DIST_EQUAL)
    throw std::invalid_argument("relationship: distance_type (middle is out of scope)");
  if (dist && r.anchor < 0) throw std::invalid_argument("relationship: greater/less/equal require exactly 1 anchor");
  if (r.direction != SB_DIR_NONE && r.anchor < 0) throw std::invalid_argument("relationship: direction requires exactly 1 anchor");
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
  if (r.anchor < 0) return false;
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
