// Device helpers of the ReachMap4D query (reachability.cpp:113-141), shared by the map
// kernels (sb_reach.cu) and the placement engine's fused reachability filter (sb_place.cu).
#pragma once

#include "sb_crmath.cuh"
#include "sb_reach.h"

namespace sbd {

// std::hypot, correctly rounded (glibc's is: 0 misroundings in 20k random checks): x^2 + y^2
// in double-double, then one Newton correction of the square root.
__device__ __forceinline__ double hypot_cr(double x, double y) {
  x = fabs(x);
  y = fabs(y);
  const double big = fmax(x, y), small = fmin(x, y);
  if (!isfinite(big) || big > 1e150 || (small != 0.0 && small < 1e-150)) return hypot(x, y);
  if (big == 0.0) return 0.0;
  const sbm::dd s = sbm::dd_add(sbm::two_prod(x, x), sbm::two_prod(y, y));
  const double r = sqrt(s.hi);
  const sbm::dd e = sbm::dd_add(s, sbm::dd_neg(sbm::two_prod(r, r)));
  return r + e.hi / (2.0 * r);
}

// ReachMap4D::bin (reachability.cpp:113-119)
__device__ __forceinline__ bool reach_bin(const sbk::ReachGrid& g, double x, double y, double z,
                                    uint64_t& ir, uint64_t& iz) {
  const double r = hypot_cr(x, y);
  if (r >= g.r_max || z < g.z_min || z >= g.z_max) return false;
  ir = (uint64_t)(r / g.res);
  iz = (uint64_t)((z - g.z_min) / g.res);
  return ir < g.nr && iz < g.nz;
}

__device__ __forceinline__ bool reach_bit(const unsigned long long* w, uint64_t idx) {
  return (__ldg(w + (idx >> 6)) >> (idx & 63)) & 1ull;
}

}  // namespace sbd
