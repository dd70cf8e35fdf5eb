// Kernel launch wrappers for CollisionWorld maintenance, the world-API check_batch and
// narrow-phase cycle profile of check_batch (zeros unless built with -DSB_NARROW_PROF)
void narrow_profile_check(unsigned long long out[8], bool reset);

// engine bookkeeping (implemented in sb_kernels.cu). Plain C++ signatures so the host
// runtime (sb_runtime.cpp, g++) can call them without CUDA types in its interfaces.
// The placement engine proper lives in sb_place.h, the relation regions in sb_region.h.
#pragma once

#include <cstddef>
#include <cstdint>

#include "sb_layout.h"

typedef struct CUstream_st* sb_stream_t;

namespace sbk {

// world maintenance (collision.cpp:365-412)
void init_object(const SbWorldView& w, int32_t obj, sb_stream_t s);
void set_enabled_list(const SbWorldView& w, int32_t obj, const uint32_t* inst, uint64_t n,
                      int enabled, sb_stream_t s);
void set_enabled_all(const SbWorldView& w, int32_t obj, int enabled, sb_stream_t s);
// poses16 + stride * j is slot j's column-major pose (stride 0 broadcasts one pose)
void update_transforms(const SbWorldView& w, int32_t obj, const double* poses16,
                       const uint32_t* inst /*nullable: all*/, uint64_t n, uint64_t stride,
                       sb_stream_t s);
// check_batch (collision.cpp:418-461); counters[1,2,4,5] = narrow, pairs, broad, nodes
void check_batch(const SbWorldView& w, int32_t geom, const double* poses16,
                 const uint32_t* active, uint64_t m, uint8_t* free_out, int32_t* contact_out,
                 unsigned long long* counters, sb_stream_t s);

// narrow-phase cycle profile of check_batch (zeros unless built with -DSB_NARROW_PROF)
void narrow_profile_check(unsigned long long out[8], bool reset);

// engine bookkeeping
void engine_reset(const SbWorldView& w, int32_t first_obj, int32_t n_obj, uint8_t* valid,
                  int16_t* accepted, int32_t n_place, sb_stream_t s);
// end of a run: identity pose + local box for every (placement object, instance) left
// unaccepted (accepted: [n_place][n])
void unaccepted_fixup(const SbWorldView& w, int32_t first_obj, int32_t n_place,
                      const int16_t* accepted, sb_stream_t s);
// one placement's column-major result poses [n][16]: identity where accepted[i] < 0
void out16_fixup(uint64_t n, const int16_t* accepted, double* out16, sb_stream_t s);
// broad-phase occupancy grid: clear, then insert the enabled fixed objects (ids < first_obj)
void cells_reset(const SbWorldView& w, const SbCellGrid& g, int32_t first_obj, sb_stream_t s);
// AnchorState per instance (support frame): out[3i..3i+2] = x, y, yaw
void anchor_states(const SbWorldView& w, int32_t anchor_obj, const double inv_support[12],
                   const double* inv_inst, double* out, sb_stream_t s);
// per-instance support frames: S[i] = pose(obj, i) * frame (obj >= 0) or as given,
// inv[i] = inverse_rigid(S[i]); row-major 3x4, [n][12]
void support_frames(const SbWorldView& w, int32_t obj, const double frame[12], double* S,
                    double* inv, sb_stream_t s);
// test hook for the device libm (sb_crmath.cuh): fn 0 sin, 1 cos, 2 atan2 (pairs y, x)
void debug_math(int fn, const double* in, uint64_t n, double* out, sb_stream_t s);
// accepted poses of one object as column-major Mat4 (N x 16 doubles)
void download_poses(const SbWorldView& w, int32_t obj, double* out16, sb_stream_t s);

// standalone PositionSampler / sample_orientations (sampler.cpp:54-156). sup34: one
// row-major 3x4 support pose per active entry (host-gathered); inst_tab: per instance
// (first table row, rows) into tris/cum, or NULL: [n][cap] tables with inst_n rows each.
// sup34 == NULL: supports read in place from sup16 (N column-major Mat4) at active[j]
void sampler_fifo(const double* sup34, const double* sup16, const uint32_t* active, uint64_t m,
                  const uint64_t* seg_first, const uint64_t* seg_draw, int nseg, uint64_t state0,
                  const SbRegionTri* tris, const double* cum, int nt, double* pos, sb_stream_t s);
void sampler_fallback(const double* sup34, const double* sup16, const uint32_t* active,
                      uint64_t m, uint64_t run_seed,
                      uint64_t salt, uint64_t attempt, const uint32_t* inst_tab,
                      const int32_t* inst_n, int cap, const SbRegionTri* tris, const double* cum,
                      double* pos, uint8_t* placeable, sb_stream_t s);
void orientations(int kind, const uint32_t* active, uint64_t m, const double* pos,
                  const double* face_xy, uint64_t run_seed, uint64_t salt, uint64_t attempt,
                  double* yaws, sb_stream_t s);

}  // namespace sbk
