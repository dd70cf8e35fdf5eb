// Per-instance constraint regions on the device (see sb_region.cu).
#pragma once

#include <cstdint>

#include "sb_kernels.h"
#include "sb_layout.h"

namespace sbk {

// cos / sin of annulus_sector's arc points (polygon.cpp:146-153) when they do not depend on
// the anchor (no local-frame direction): computed once per placement on the host with the
// reference's own libm (std::atan2 / std::cos / std::sin), read by every instance.
constexpr int kArcCap = 80;  // a full circle is 72 segments at the 5 degree step
struct SbArcTable {
  double c[2][kArcCap], s[2][kArcCap];  // arc 0 = outer arc / full circle, arc 1 = inner arc
  int32_t na[2];                         // segments of arc k (points = na + 1), 0 = none
};
// Fills `t` for placement `pl`; false when the arcs depend on the anchor yaw (local frame)
// or do not fit the table.
bool arc_table_host(const SbPlacementDev& pl, SbArcTable& t);

struct RelationRegionParams {
  SbWorldView w;
  SbPlacementDev pl;
  int32_t anchor_object;
  int32_t owns_instance0;  // 1: global instance 0 is local instance 0 (compute s0 in-kernel)
  double inv_support[12];  // inverse_rigid(support pose), row-major 3x4 (host-computed)
  const double* s0;        // instance 0's anchor states (x, y, yaw per anchor) when
                           // !owns_instance0 (device)
  int32_t from_s0;         // 1: build a single region from s0 (canonical, sharded runs)
  int32_t cap;
  int32_t hole;            // full annulus with a hole: bridged-hole path (sbp::hole_annulus_table)
  const SbArcTable* arcs;  // optional device copy of arc_table_host (shared arcs)
  const double* states;    // optional [n][3] anchor states (x, y, yaw) in the support frame
                           // given directly (standalone sampler); else read from world poses
  SbRegionTri* tris;       // [n][cap] (or [1][cap] when from_s0)
  double* cum;
  int32_t* ntri;           // [n]
  int32_t* flags;          // [0] |= anchors vary, [1] = max region error status
};

// Stage cycle profile of the region kernel (zeros unless built with -DSB_REGION_PROF).
void region_profile(unsigned long long out[8], bool reset);
void relation_regions(const RelationRegionParams& p, int num_sms, sb_stream_t s);

}  // namespace sbk
