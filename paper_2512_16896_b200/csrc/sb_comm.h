// Native shard communicator: launch wrappers of the count-board kernels.
// Plain C++ signatures so the host side (sb_comm_rt.cpp, g++) needs no CUDA types.
//
// Board layout (one per rank, in that rank's HBM, mapped by every peer through CUDA IPC):
//   board[slot][src_rank][kCommStride] u64 -- word 0 = epoch flag, words 1..n = values.
// A rank publishes the values of exchange `epoch` by storing them into EVERY rank's board
// (remote stores over NVLink / NVSwitch, or plain stores for itself), a system-scope fence,
// then the flag word. Readers wait on their own board only (local memory).
#pragma once

#include <cstdint>

typedef struct CUstream_st* sb_stream_t;

namespace sbk {

constexpr int kCommSlots = 64;      // exchanges in flight before a slot is reused
constexpr int kCommStride = 32;     // u64 words per (slot, source rank): flag + 31 values
constexpr int kCommMaxValues = kCommStride - 1;
constexpr int kCommMaxRanks = 64;

// Push this rank's n values (device memory) into slot `slot` of every rank's board.
// peers: device array of world_size board base pointers as mapped in this process.
void comm_push(uint64_t* const* peers, int world_size, int rank, int slot, uint64_t epoch,
               const uint64_t* d_send, uint32_t n, sb_stream_t s);
// Gather slot `slot` of this rank's own board into d_recv (rank-major, world_size * n).
// spin != 0: wait on the flags inside the kernel (when stream memory waits are
// unavailable); else the caller has already enqueued the stream waits.
void comm_collect(const uint64_t* board, int world_size, int slot, uint64_t epoch,
                  uint32_t n, uint64_t* d_recv, int spin, sb_stream_t s);

// Sharded relation placements, exchanged on the device (sb_runtime.cpp):
//   anchor_pack: send[0..3na) = bits of instance 0's anchor states s0 (x, y, yaw per anchor;
//     s0 != NULL iff this rank owns global instance 0), send[3na] = owner flag;
//   anchor_pick: s0 = the owner's entry of the gathered recv[world][3na + 1];
//   flag_pack / flag_or: the local "anchors vary" flag out, the OR over ranks back in.
void shard_anchor_pack(const double* s0, int na, uint64_t* send, sb_stream_t s);
void shard_anchor_pick(const uint64_t* recv, int world_size, int na, double* s0, sb_stream_t s);
void shard_flag_pack(const int32_t* flag, uint64_t* send1, sb_stream_t s);
void shard_flag_or(const uint64_t* recv, int world_size, int32_t* flag, sb_stream_t s);

}  // namespace sbk
