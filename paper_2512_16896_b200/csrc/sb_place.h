// Phased placement engine: one placement's whole attempt loop on the device.
//
// A round (= one attempt over the still-failing instances) runs as four
// grid-wide phases:
//   A  warp per active slot: sample (FIFO jump-ahead or counter stream), yaw, pose compose,
//      candidate AABB + inverse pose, AABB broad phase with lanes over objects; overlapping
//      (slot, object) pairs are appended to a pair queue
//   B  warp per pair: exact MeshBvh::collide (sb_warp.cuh) -> atomicMin(contact[slot], obj)
//   C  thread per slot: first-valid accept (update_transform + set_enabled) or fail flag;
//      reference-equivalent narrow-phase count; per-chunk failure counts
//   D  stable compaction of the failing slots into the next round's active list
// Per-instance (counter-stream) regions: attempt a of instance i depends only on
// make_stream(run_seed, {salt, tag, i, a}) and on instance i's world, which is unchanged
// until i accepts. A round may therefore evaluate W consecutive attempts of every remaining
// instance at once ("virtual slots") and accept the lowest free one -- the sequential
// first-valid result; counters are reported as the sequential loop would have counted
// them. The FIFO fast path couples instances through the draw index, so W = 1 there.
// Every (candidate, object) pair of a round is evaluated in parallel; contact_object is the
// minimum colliding object id, i.e. the reference's first hit in ascending order
// (collision.cpp:439-448). Single GPU: one cooperative kernel loops over all rounds with
// grid.sync() between phases. Sharded: the host launches the phases per round and
// exchanges the per-rank counts between rounds.
#pragma once

#include <cstddef>
#include <cstdint>

#include "sb_kernels.h"
#include "sb_layout.h"

namespace sbk {

struct PlaceParams {
  SbWorldView w;
  SbPlacementDev pl;
  int32_t attempts;             // K
  int32_t fast;                 // canonical region (FIFO stream) vs per-instance regions
  uint64_t run_seed;
  uint64_t global_begin;
  uint64_t fast_state0;
  const SbRegionTri* canon_tris;
  const double* canon_cum;
  int32_t canon_n;
  int32_t inst_cap;
  const SbRegionTri* inst_tris;
  const double* inst_cum;
  const int32_t* inst_n;
  uint8_t* valid;               // [n]
  int16_t* accepted;            // [n] of this placement
  uint32_t* act0;               // active lists (ping-pong), slot -> local instance
  uint32_t* act1;
  double* cpose;                // [n][12] candidate pose per slot
  double* cinv;                 // [n][12] candidate inverse pose per slot
  uint8_t* cflag;               // [n] 1 = placeable (checked)
  int32_t* contact;             // [n] min colliding object, INT32_MAX = free
  uint32_t* ovmask;             // [words][n] overlap bits per slot
  uint8_t* failflag;            // [n]
  uint64_t* pairs;              // pair queue (slot << 32 | object)
  uint64_t pair_cap;
  uint32_t* chunk_cnt;          // [ceil(n / 256)]
  uint32_t* ctrl;               // [0] M, [1] pair count, [2] rounds, [3] error, [4] cur list
  unsigned long long* counters; // [8]
  uint64_t draw_base;           // sharded host loop: this rank's first draw index
  uint64_t slot_cap;            // capacity of the per-slot candidate arrays
  uint64_t spec_budget;         // target candidates per round for speculative attempts
  int32_t spec_width;           // host loop: attempts per instance this round (1 = none)
  uint64_t* prof;               // optional phase timers (ns) [init, A, B, C, D, rounds]
  // Relation placements on one GPU: the path is chosen on the device. When non-null,
  // *vary_flag != 0 selects the per-instance tables, else the FIFO fast path samples the
  // canonical region_for(0) = local instance 0's table (relationships.cpp:188-190).
  const int32_t* vary_flag;
};

constexpr int kPlaceBlock = 256;

// Single GPU: whole placement in one cooperative launch. Returns false if the device
// cannot co-schedule the grid (caller falls back to the host loop).
bool place_persistent(const PlaceParams& p, int num_sms, sb_stream_t s);
// Warps of the co-resident persistent grid (sizes the speculative-attempt budget).
int place_grid_warps(int num_sms);
// Cycle breakdown of the narrow phase (zeros unless built with -DSB_NARROW_PROF).
void narrow_profile(unsigned long long out[8], bool reset);
// Host loop building blocks (sharded runs): init active list, then per round
// phase_abcd(draw_base) with the count read back in between.
void place_init(const PlaceParams& p, sb_stream_t s);
void place_round(const PlaceParams& p, int32_t attempt, int cur, sb_stream_t s);
void place_finish(const PlaceParams& p, int cur, sb_stream_t s);

}  // namespace sbk
