// BatchedSceneGraph device kernels (sb_graph.cu); plain C++ signatures for the host runtime.
#pragma once

#include <cstdint>

#include "sb_kernels.h"

namespace sbk {

struct GraphJoint {
  int32_t kind;    // 0 revolute, 1 prismatic (JointSpec::Kind)
  double axis[3];  // unit axis (JointSpec ctor normalises)
};

void graph_colmajor_to_34(const double* in16, uint64_t n, double* out12, sb_stream_t s);
void graph_34_to_colmajor(const double* in12, uint64_t n, double* out16, sb_stream_t s);
void graph_joint_compose(const double* base, const double* values, uint64_t i0, uint64_t n,
                         const GraphJoint& j, double* edge, sb_stream_t s);
// chain: device array of `depth` edge batches, chain[0] = the node, chain[depth-1] = the
// child of the root
void graph_world_poses(const double* const* chain, int depth, uint64_t n, double* out16,
                       sb_stream_t s);
void graph_world_pose_one(const double* const* chain, int depth, uint64_t i, double* out16,
                          sb_stream_t s);
void graph_count_valid(const uint8_t* v, uint64_t n, unsigned long long* out, sb_stream_t s);
// pose + i * inst_stride + obj_stride = instance i's 3x4 record of one world object
void graph_gather_object_poses(const double* pose, uint64_t obj_stride, uint64_t inst_stride,
                               uint64_t n, double* out12, sb_stream_t s);

// dst[i] = 0 where src[i] == 0 (mark_invalid for the instances a run left invalid)
void graph_and_valid(uint8_t* dst, const uint8_t* src, uint64_t n, sb_stream_t s);

}  // namespace sbk
