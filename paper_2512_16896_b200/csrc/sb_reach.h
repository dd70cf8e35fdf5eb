// ReachMap4D on the device (sb_reach.cu): FK-sampled occupancy build, batched queries and
// the placement filter (reachability.cpp:38-190). Plain C++ signatures for the host runtime.
#pragma once

#include <cstdint>

#include "sb_kernels.h"

namespace sbk {

struct ReachGrid {
  double res, psi_res, r_max, z_min, z_max;
  uint64_t nr, nz, npsi;
};

// links: n_links x 18 doubles = origin (row-major 3x4), kind, axis[3], lo, hi; ee12: the
// end-effector offset (row-major 3x4). occ / counts must be zeroed by the caller.
void reach_build(const double* links, int n_links, const double* ee12, uint64_t samples,
                 uint64_t seed, const ReachGrid& g, unsigned long long* occ, unsigned* counts,
                 sb_stream_t s);
// occ_any[(ir * nz + iz)] = any psi bin of (ir, iz) occupied
void reach_any(const ReachGrid& g, const unsigned long long* occ, unsigned long long* occ_any,
               sb_stream_t s);
// base16 (column-major, n) and targets (n x 3); inclination NaN: none (any psi)
void reach_query_batch(const ReachGrid& g, const unsigned long long* occ,
                       const unsigned long long* occ_any, const double* base16,
                       const double* targets, uint64_t n, double inclination, uint8_t* out,
                       sb_stream_t s);
// frames: n_frames device pointers (or NULL) to N column-major poses each
void reach_placement_filter(const ReachGrid& g, const unsigned long long* occ_any,
                            const double* base16, const double* const* frames, int n_frames,
                            const uint32_t* active, uint64_t m, uint8_t* out, sb_stream_t s);
void reach_popcount(const unsigned long long* words, uint64_t n, unsigned long long* out,
                    sb_stream_t s);

}  // namespace sbk
