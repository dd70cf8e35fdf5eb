// Count-board kernels of the native shard communicator (see sb_comm.h). One tiny CTA per
// exchange: the payload is a few u64 per rank, so the cost is the NVLink / NVSwitch store
// latency, not bandwidth.
#include <stdexcept>
#include <string>

#include "sb_comm.h"

namespace {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t ld_volatile(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Items are (destination rank, value) pairs; after the CTA-wide system fence one thread per
// destination rank releases that rank's flag word.
__global__ void k_comm_push(uint64_t* const* peers, int world, int rank, int slot,
                            uint64_t epoch, const uint64_t* send, uint32_t n) {
  const uint32_t items = static_cast<uint32_t>(world) * n;
  for (uint32_t t = threadIdx.x; t < items; t += blockDim.x) {
    const uint32_t r = t / n, k = t - r * n;
    uint64_t* dst = peers[r] + (static_cast<uint64_t>(slot) * world + rank) * sbk::kCommStride;
    dst[1 + k] = send[k];
  }
  __threadfence_system();
  __syncthreads();
  for (int r = threadIdx.x; r < world; r += blockDim.x)
    st_release_sys(peers[r] + (static_cast<uint64_t>(slot) * world + rank) * sbk::kCommStride, epoch);
}

__global__ void k_comm_collect(const uint64_t* board, int world, int slot, uint64_t epoch,
                               uint32_t n, uint64_t* recv, int spin) {
  const uint64_t* base = board + static_cast<uint64_t>(slot) * world * sbk::kCommStride;
  if (spin) {
    for (int r = threadIdx.x; r < world; r += blockDim.x) {
      unsigned ns = 32;
      while (ld_acquire_sys(base + static_cast<uint64_t>(r) * sbk::kCommStride) < epoch) {
        __nanosleep(ns);
        if (ns < 1024) ns *= 2;
      }
    }
    __syncthreads();
  } else {
    // the stream waited on the flags; order the payload reads after them
    for (int r = threadIdx.x; r < world; r += blockDim.x)
      (void)ld_acquire_sys(base + static_cast<uint64_t>(r) * sbk::kCommStride);
    __syncthreads();
  }
  const uint32_t items = static_cast<uint32_t>(world) * n;
  for (uint32_t t = threadIdx.x; t < items; t += blockDim.x) {
    const uint32_t r = t / n, k = t - r * n;
    recv[t] = ld_volatile(base + static_cast<uint64_t>(r) * sbk::kCommStride + 1 + k);
  }
}

__global__ void k_anchor_pack(const double* s0, int na, uint64_t* send) {
  const int t = threadIdx.x, m = 3 * na;
  if (t < m) send[t] = s0 ? __double_as_longlong(s0[t]) : 0ull;
  if (t == m) send[m] = s0 ? 1ull : 0ull;
}

__global__ void k_anchor_pick(const uint64_t* recv, int world, int na, double* s0) {
  if (threadIdx.x != 0) return;
  const int m = 3 * na, stride = m + 1;
  for (int r = 0; r < world; ++r)
    if (recv[stride * r + m]) {
      for (int k = 0; k < m; ++k) s0[k] = __longlong_as_double(recv[stride * r + k]);
      return;
    }
}

__global__ void k_flag_pack(const int32_t* flag, uint64_t* send) {
  if (threadIdx.x == 0) send[0] = *flag != 0 ? 1ull : 0ull;
}

__global__ void k_flag_or(const uint64_t* recv, int world, int32_t* flag) {
  if (threadIdx.x != 0) return;
  int v = 0;
  for (int r = 0; r < world; ++r) v |= recv[r] != 0;
  *flag = v;
}

inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

namespace sbk {

void comm_push(uint64_t* const* peers, int world_size, int rank, int slot, uint64_t epoch,
               const uint64_t* d_send, uint32_t n, sb_stream_t s) {
  k_comm_push<<<1, 128, 0, reinterpret_cast<cudaStream_t>(s)>>>(peers, world_size, rank, slot,
                                                                epoch, d_send, n);
  check_launch("k_comm_push");
}

void comm_collect(const uint64_t* board, int world_size, int slot, uint64_t epoch, uint32_t n,
                  uint64_t* d_recv, int spin, sb_stream_t s) {
  k_comm_collect<<<1, 128, 0, reinterpret_cast<cudaStream_t>(s)>>>(board, world_size, slot,
                                                                   epoch, n, d_recv, spin);
  check_launch("k_comm_collect");
}

void shard_anchor_pack(const double* s0, int na, uint64_t* send, sb_stream_t s) {
  k_anchor_pack<<<1, 32, 0, reinterpret_cast<cudaStream_t>(s)>>>(s0, na, send);
  check_launch("k_anchor_pack");
}
void shard_anchor_pick(const uint64_t* recv, int world_size, int na, double* s0, sb_stream_t s) {
  k_anchor_pick<<<1, 32, 0, reinterpret_cast<cudaStream_t>(s)>>>(recv, world_size, na, s0);
  check_launch("k_anchor_pick");
}
void shard_flag_pack(const int32_t* flag, uint64_t* send1, sb_stream_t s) {
  k_flag_pack<<<1, 32, 0, reinterpret_cast<cudaStream_t>(s)>>>(flag, send1);
  check_launch("k_flag_pack");
}
void shard_flag_or(const uint64_t* recv, int world_size, int32_t* flag, sb_stream_t s) {
  k_flag_or<<<1, 32, 0, reinterpret_cast<cudaStream_t>(s)>>>(recv, world_size, flag);
  check_launch("k_flag_or");
}

}  // namespace sbk
