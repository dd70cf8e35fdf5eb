// JointSpec::motion on the device, shared by the scene graph (sb_graph.cu) and the
// reachability map build (sb_reach.cu).
#pragma once

#include "sb_crmath.cuh"
#include "sb_glibcm.cuh"
#include "sb_dev.cuh"
#include "sb_graph.h"

namespace sbd {

// JointSpec::motion (scene_graph.cpp:19-27): prismatic = translation(axis * v); revolute =
// AngleAxisd(v, axis).toRotationMatrix() (Rodrigues, Eigen's operation order).
__device__ __forceinline__ void joint_motion(const sbk::GraphJoint& j, double v, M34& m) {
#pragma unroll
  for (int k = 0; k < 12; ++k) m.m[k] = 0.0;
  m.m[0] = m.m[5] = m.m[10] = 1.0;
  const double ax = j.axis[0], ay = j.axis[1], az = j.axis[2];
  if (j.kind == 1) {
    m.m[3] = ax * v;
    m.m[7] = ay * v;
    m.m[11] = az * v;
    return;
  }
  double s, c;
  sbg::sincos(v, &s, &c);
  const double sx = ax * s, sy = ay * s, sz = az * s;
  const double c1 = 1.0 - c;
  const double cx = ax * c1, cy = ay * c1, cz = az * c1;
  double t = cx * ay;
  m.m[1] = t - sz;
  m.m[4] = t + sz;
  t = cx * az;
  m.m[2] = t + sy;
  m.m[8] = t - sy;
  t = cy * az;
  m.m[6] = t - sx;
  m.m[9] = t + sx;
  m.m[0] = cx * ax + c;
  m.m[5] = cy * ay + c;
  m.m[10] = cz * az + c;
}

}  // namespace sbd
