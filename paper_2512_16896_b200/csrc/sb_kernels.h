// Kernel launch wrappers (implemented in sb_kernels.cu). Plain C++ signatures so the
// host runtime (sb_runtime.cpp, g++) can call them without CUDA headers in its types.
#pragma once

#include <cstddef>
#include <cstdint>

#include "sb_layout.h"

typedef struct CUstream_st* sb_stream_t;

namespace sbk {

// Per-round parameters of the fused sample -> compose -> check -> accept kernel.
struct RoundParams {
  SbWorldView w;
  SbPlacementDev pl;
  int32_t attempt;
  int32_t fast;                   // 1 = canonical region, FIFO stream (sampler.cpp:78-99)
  uint64_t run_seed;
  uint64_t global_begin;          // first global instance id of this shard
  uint64_t fast_state0;           // Pcg state after make_stream(run_seed,{salt,"cach"})
  uint64_t draw_base;             // global draw index of this rank's first active slot
  const SbRegionTri* canon_tris;  // canonical sampler table (fast path)
  const double* canon_cum;
  int32_t canon_n;
  int32_t inst_cap;               // per-instance table capacity (fallback path)
  const SbRegionTri* inst_tris;   // [n][inst_cap]
  const double* inst_cum;         // [n][inst_cap]
  const int32_t* inst_n;          // [n]
  const uint32_t* act;            // active local instance ids, ascending
  uint64_t m;                     // number of active slots
  uint8_t* fail;                  // [m] 1 = still failing after this attempt
  int16_t* accepted;              // [n] accepted attempt of this placement
  unsigned long long* counters;   // [8]: checked, narrow, pairs, sampled, broad, nodes, accepted
};

// Per-instance constraint region build (relationships.cpp:161-218 + polygon.cpp:136-176,
// 344-388) for one placement.
struct RegionParams {
  SbPlacementDev pl;
  const double* anchors;          // [count][3] position x, y, yaw (support frame)
  uint64_t count;
  int32_t cap;
  SbRegionTri* tris;              // [count][cap]
  double* cum;                    // [count][cap]
  int32_t* ntri;                  // [count]
  int32_t* status;                // worst RegionStatus seen (atomicMax)
};

// world maintenance
void init_object(const SbWorldView& w, int32_t obj, sb_stream_t s);
void set_enabled_list(const SbWorldView& w, int32_t obj, const uint32_t* inst, uint64_t n,
                      int enabled, sb_stream_t s);
void set_enabled_all(const SbWorldView& w, int32_t obj, int enabled, sb_stream_t s);
// poses16 + stride * j is slot j's column-major pose (stride 0 broadcasts one pose)
void update_transforms(const SbWorldView& w, int32_t obj, const double* poses16,
                       const uint32_t* inst /*nullable: all*/, uint64_t n, uint64_t stride,
                       sb_stream_t s);
// check_batch (collision.cpp:418-461)
void check_batch(const SbWorldView& w, int32_t geom, const double* poses16,
                 const uint32_t* active, uint64_t m, uint8_t* free_out, int32_t* contact_out,
                 unsigned long long* counters, sb_stream_t s);

// generation engine
void engine_reset(const SbWorldView& w, int32_t first_obj, int32_t n_obj, uint8_t* valid,
                  int16_t* accepted, int32_t n_place, sb_stream_t s);
// stable compaction: out = [i for i in range(n) if flags[i]] (ids) or in[j] for flagged j
size_t select_temp_bytes(uint64_t n);
void select_valid(const uint8_t* valid, uint64_t n, uint32_t* out, uint64_t* d_count, void* temp,
                  size_t temp_bytes, sb_stream_t s);
void select_flagged(const uint32_t* in, const uint8_t* flags, uint64_t m, uint32_t* out,
                    uint64_t* d_count, void* temp, size_t temp_bytes, sb_stream_t s);
void round_kernel(const RoundParams& p, sb_stream_t s);
void invalidate(const uint32_t* act, uint64_t m, uint8_t* valid, sb_stream_t s);
void anchor_states(const SbWorldView& w, int32_t anchor_obj, const double inv_support[12],
                   double* out, sb_stream_t s);
void vary_flag(const double* states, uint64_t n, double x0, double y0, double yaw0,
               int32_t* flag, sb_stream_t s);
void build_regions(const RegionParams& p, sb_stream_t s);
void download_poses(const SbWorldView& w, int32_t obj, double* out16, sb_stream_t s);

}  // namespace sbk
