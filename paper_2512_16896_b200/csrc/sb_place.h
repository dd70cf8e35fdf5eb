// Tiled placement engine: one placement's whole attempt loop on the device.
//
// The instances of a shard are cut into `ntiles` contiguous ranges ("tiles") of at most
// `tile_inst` (<= kPlaceBlock) instances. A tile is owned by one CTA for a round, and
// everything one attempt round does to it stays in that CTA's shared memory:
//   A1  thread per slot: sample (FIFO jump-ahead or counter stream), yaw, pose compose,
//       candidate AABB + inverse pose (sampler.cpp:70-156, transform.hpp:40-69)
//   A2  thread per (slot, object): AABB broad phase (collision.cpp:439-443); overlapping
//       pairs go to a shared-memory queue
//   B   warp per queued pair: exact MeshBvh::collide (sb_warp.cuh) -> atomicMin on the
//       slot's contact object (the reference's first hit in ascending object order)
//   C   thread per instance: first-valid accept (update_transform + set_enabled) or keep
//       the instance for the next attempt; survivors are compacted in place
// so a round has no grid-wide phase barrier. Tiles keep their own survivors, which makes
// the global active order (tile order, then ascending instance inside a tile) the
// reference's ascending `active` order at every attempt.
//
// FIFO fast path (canonical region, sampler.cpp:78-99): instance i at attempt a takes draw
// j = sum_{a'<a} |active_a'| + rank_a(i), so tiles advance in lockstep: per round every CTA
// scans the per-tile survivor counts once (its tiles' draw offsets + the round total) and
// the round ends with ONE grid barrier. Per-instance regions (counter streams
// make_stream(run_seed, {salt, "fall"|"yaw!", inst, attempt}), sampler.cpp:101-156): tiles
// are independent, so a CTA runs a tile to completion with no grid barrier at all, and
// evaluates W consecutive attempts of each survivor at once ("speculative slots"; W grows
// as the tile empties) -- attempt a of instance i depends only on its stream and on
// instance i's world, which is unchanged until i accepts, so accepting the lowest free
// slot is exactly the sequential first-valid result.
// Single GPU: one cooperative launch per placement. Sharded (multi-GPU): the fast path runs
// one launch per round with the per-rank counts exchanged on the host in between.
#pragma once

#include <cstddef>
#include <cstdint>

#include "sb_kernels.h"
#include "sb_layout.h"
#include "sb_reach.h"

namespace sbk {

struct PlaceParams {
  SbWorldView w;
  SbPlacementDev pl;
  int32_t attempts;             // K
  int32_t fast;                 // canonical region (FIFO stream) vs per-instance regions
  uint64_t run_seed;
  const uint64_t* seed_dev;     // optional: run_seed read on the device (graph replays)
  uint64_t global_begin;
  uint64_t fast_state0;
  const uint64_t* jump;         // pcg_jump_table_host: FIFO draw -> PCG state (draws < 2^32)
  const SbRegionTri* canon_tris;
  const double* canon_cum;
  int32_t canon_n;
  int32_t inst_cap;
  const SbRegionTri* inst_tris;
  const double* inst_cum;
  const int32_t* inst_n;
  uint8_t* valid;               // [n]
  int16_t* accepted;            // [n] of this placement
  double* out16;                // optional [n][16]: accepted poses, column-major (result download)
  uint32_t* tile_list;          // [ntiles * tile_inst] survivors of each tile
  uint32_t* tile_cnt;           // [2][cnt_stride] survivors per tile, ping-pong by round
  uint32_t cnt_stride;
  uint32_t ntiles;
  int32_t tile_inst;            // instances per tile (<= kPlaceBlock)
  uint32_t ntiles_pi;           // per-instance path: smaller tiles taken dynamically
  int32_t tile_inst_pi;
  int32_t spec_target;          // per-instance path: target slots per tile round
  const uint32_t* tile_perm;     // per-instance path: claim order -> tile (null = identity)
  uint32_t* tile_ns;             // ... and each tile's processing time (ns), or null
  int32_t solo_max;             // fast path: at most this many survivors -> CTA 0 alone
  int32_t solo_spec;            // fast path solo tail: target speculative slots per round
  int32_t ws_bytes;             // narrow-phase scratch per warp (sb_warp.cuh)
  int32_t max_tris, max_nodes;  // scratch geometry bounds over the world's geometries
  double* cpose;                // [grid][kPlaceBlock][12] candidate pose per CTA slot
  double* cinv;                 // [grid][kPlaceBlock][12] its inverse (narrow phase, cp.async)
  SbCellGrid grid;              // broad-phase occupancy grid
  uint32_t* ctrl;               // [8] per placement: see Ctrl in sb_place.cu
  unsigned long long* counters; // [8]
  uint64_t draw_base;           // sharded fast path: draws before this rank this round
  // Sharded fast path with a device-side count exchange (sb_shard.allgather_dev): round a
  // reads the gathered counts xrecv[a][world] and the draws before it xdraws[a] on the
  // device (no host round trip), adds its survivors into xcount[a + 1] and writes
  // xdraws[a + 1]; a round whose gathered total is 0 returns at once.
  const unsigned long long* xrecv;
  unsigned long long* xdraws;
  unsigned long long* xcount;
  int32_t xrank, xworld;
  unsigned* dbg;                // optional [attempts][3] per-round CTA maxima (ns), fast path
  unsigned* dbg_inst;           // optional [5] per-instance tiles: max ns, sum us, max/sum rounds, n
  uint64_t* prof;               // optional timers (ns) [init, rounds, -, -, -, rounds]
  // Relation placements on one GPU: the path is chosen on the device. When non-null,
  // *vary_flag != 0 selects the per-instance tables, else the FIFO fast path samples the
  // canonical region_for(0) = local instance 0's table (relationships.cpp:188-190).
  const int32_t* vary_flag;
  // Sharded relation placements with the device exchange: both paths are enqueued and the
  // OR-gathered flag picks one on the device -- k_place_instances runs iff *shard_vary != 0,
  // k_fast_init (and so the FIFO rounds) iff *shard_vary == 0; the FIFO rounds then read
  // the canonical table size from canon_n_dev.
  const int32_t* shard_vary;
  const int32_t* canon_n_dev;
  // Optional fused reachability filter: a candidate whose frame origin,
  // in its instance's robot base frame, misses the map's (r, z) occupancy is a failed
  // attempt that is not collision-checked (Appendix C item 8).
  const unsigned long long* reach_any;  // occ_any bitset of the map, NULL = no filter
  ReachGrid reach_grid;
  const double* reach_base;             // [n][12] robot base per local instance (row-major)
  // Wide round 0 (FIFO placements, place_wide_round0): k_place then starts at round
  // start_round = 1 from the survivors k_wide_accept left in tile_cnt buffer 1.
  int32_t start_round;
  const unsigned long long* start_draws;  // draws of the rounds before start_round
  // Persistent fast rounds without a grid barrier (decoupled look-back), or null: entry
  // lb_board[a * lb_stride + t] = lb_epoch << 32 | tile t's active count of round a, published
  // by the CTA owning t when it finishes round a - 1 (lb_epoch is unique per launch).
  unsigned long long* lb_board;
  uint32_t lb_stride;
  uint32_t lb_epoch;
  uint32_t lb_sleep;  // ns a waiting CTA sleeps between polls (0: spin)
  double* w_pose;                // [ntiles * kPlaceBlock][kWideRec] compact candidate record
                                 // per round-0 slot: tx, ty, tz, cos, sin, 0
  int32_t* w_contact;            // [..] lowest colliding object, INT32_MAX = free
  uint32_t* w_ovm;               // [..][8]  broad-phase overlap bits
  uint8_t* w_flag;               // [..]     slot state
  uint32_t* w_pairs;             // [<= n * n_objects] (slot << 8 | object)
  uint32_t* w_pairs2;            // [same] the pairs past the leaf-box filter
  uint32_t* w_pinst2;            // [same] their instance ids (no tile-list lookup to stage)
  int32_t wide_round;            // attempt a of this wide round (0; dense later rounds too)
  unsigned long long* w_surv;    // [kWideSurvRounds] survivors after each wide round, or null
  uint32_t* w_toff;              // [ntiles] first FIFO draw of each tile
  unsigned long long* w_ctl;     // [7] pairs appended, -, filtered pairs appended / claimed,
                                 // round-0 draws, round-1 active instances, tiles in use
  // Tiles holding survivors (k_wide_spread's w_ctl[6]); null = ntiles. The persistent
  // kernel's rounds >= 1 then scan / own only those (and keep them resident).
  const unsigned long long* ntiles_dev;
  uint32_t* w_list2;             // [ntiles * tile_inst] round 1's active list, re-dealt
  uint32_t* w_cnt2;              // [2][cnt_stride] its tile counts (buffer 1 = round 1)
};

#ifndef SB_PLACE_BLOCK
#define SB_PLACE_BLOCK 256
#endif
constexpr int kPlaceBlock = SB_PLACE_BLOCK;  // threads per placement CTA = max tile slots
constexpr int kPlaceMaxOwnedTiles = 64;  // tiles per CTA on the fast path
constexpr int kWideRec = 6;  // doubles per round-0 candidate record (w_pose)
#ifndef SB_WIDE_ROUNDS_MAX
#define SB_WIDE_ROUNDS_MAX 4
#endif
constexpr int kWideSurvRounds = SB_WIDE_ROUNDS_MAX;  // wide rounds per placement at most

// Dynamic shared memory of one placement CTA for a world with `n_words` enable words.
size_t place_smem_bytes(int n_words, int ws_bytes, int n_objects);
// Narrow-phase scratch bytes per warp for the given geometry bounds.
int place_ws_bytes(int max_tris, int max_nodes);
// Co-resident CTAs of the persistent placement kernel (0 if it cannot be launched).
// one: the 1-CTA-per-SM variant (no register spills) used by SB_PLACE1.
int place_grid(int num_sms, size_t smem, bool one = false);
// Single GPU: whole placement in one cooperative launch.
bool place_persistent(const PlaceParams& p, unsigned grid, size_t smem, sb_stream_t s, bool one = false);
// Cycle breakdown of the narrow phase (zeros unless built with -DSB_NARROW_PROF).
void narrow_profile(unsigned long long out[8], bool reset);
// Sharded runs. Per-instance path: one launch, no exchange (place_instances). Fast path:
// place_fast_init, then per round place_fast_round (ctrl[kTotal + (a+1)&1] receives the
// survivors; the host zeroes it before the launch), then place_fast_finish.
void place_instances(const PlaceParams& p, unsigned grid, size_t smem, sb_stream_t s);
void place_fast_init(const PlaceParams& p, unsigned grid, size_t smem, sb_stream_t s);
void place_fast_round(const PlaceParams& p, int32_t attempt, unsigned grid, size_t smem,
                      sb_stream_t s);
void place_fast_finish(const PlaceParams& p, int32_t attempt, unsigned grid, sb_stream_t s);
// Single GPU, FIFO placement: round 0 as k_fast_init + k_wide_scan + k_wide_sample +
// k_wide_narrow + k_wide_accept (no grid barrier); the caller then launches
// place_persistent with p.start_round = 1. Returns the number of launches.
int place_wide_round0(const PlaceParams& p, unsigned init_grid, size_t init_smem, int num_sms,
                      sb_stream_t s, unsigned spread_grid = 0);
// The same after k_fast_init (sharded runs exchange the round-0 counts in between: the
// sample kernel takes its draw base from p.xrecv / p.xdraws, the final scan writes the
// rank's round-1 count into p.xcount[1]); spread = false leaves the survivors compacted in
// their tiles (tile_cnt buffer 1) for k_fast_round. Returns the number of launches.
int place_wide_round0_rest(const PlaceParams& p, unsigned init_grid, int num_sms, sb_stream_t s,
                           unsigned spread_grid, bool spread);
// The same for wide round p.wide_round in two steps: (A) scan, sample, filter, narrow;
// (C) accept, scan, and (spread) the survivors re-dealt for the persistent kernel.
int place_wide_round0_a(const PlaceParams& p, int num_sms, sb_stream_t s);
int place_wide_round0_c(const PlaceParams& p, unsigned init_grid, sb_stream_t s,
                        unsigned spread_grid, bool spread);
// Narrow-kernel dynamic shared memory (per-warp scratch) for the given ws_bytes.
size_t wide_narrow_smem(int ws_bytes);
// ctrl word receiving the survivor total of round `attempt` (fast path, sharded)
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr int place_total_word(int32_t attempt) { return 5 + (attempt & 1); }

}  // namespace sbk
