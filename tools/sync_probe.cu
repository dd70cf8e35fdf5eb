// Grid-barrier latency probe on the placement kernel's launch shape (296 x 256, cooperative):
// cooperative_groups grid.sync() vs a sense-reversing barrier (one relaxed atomic per CTA,
// acquire spin on a generation word), plus the kernel launch gap of an empty cooperative
// kernel. Run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 sync_probe.cu -o sp && ./sp
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, unsigned long long* out) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void k_custom(int iters, unsigned* bar, unsigned long long* out) {
  // bar[0] = arrivals, bar[1] = generation
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned gen = ld_acquire(bar + 1);
      __threadfence();
      const unsigned arrived = atomicAdd(bar, 1u);
      if (arrived == gridDim.x - 1) {
        bar[0] = 0;
        __threadfence();
        atomicAdd(bar + 1, 1u);
      } else {
        while (ld_acquire(bar + 1) == gen) {
        }
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = clock64() - t0;
}

__global__ void k_empty() {}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = 2 * sms, iters = 2000;
  unsigned long long* d;
  unsigned* bar;
  cudaMalloc(&d, 2 * sizeof(unsigned long long));
  cudaMalloc(&bar, 2 * sizeof(unsigned));
  cudaMemset(bar, 0, 8);
  int it = iters;
  void* a1[] = {&it, &d};
  cudaLaunchCooperativeKernel((void*)k_cg, grid, 256, a1, 0, 0);
  cudaLaunchCooperativeKernel((void*)k_cg, grid, 256, a1, 0, 0);
  void* a2[] = {&it, &bar, &d};
  cudaLaunchCooperativeKernel((void*)k_custom, grid, 256, a2, 0, 0);
  cudaLaunchCooperativeKernel((void*)k_custom, grid, 256, a2, 0, 0);
  cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("grid %d: cg grid.sync %.0f cycles, custom barrier %.0f cycles (%s)\n", grid,
         (double)h[0] / iters, (double)h[1] / iters, cudaGetErrorString(cudaGetLastError()));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int coop = 0; coop < 2; ++coop) {
    for (int w = 0; w < 10; ++w) {
      if (coop) cudaLaunchCooperativeKernel((void*)k_empty, grid, 256, nullptr, 0, 0);
      else k_empty<<<grid, 256>>>();
    }
    cudaEventRecord(e0);
    for (int w = 0; w < 1000; ++w) {
      if (coop) cudaLaunchCooperativeKernel((void*)k_empty, grid, 256, nullptr, 0, 0);
      else k_empty<<<grid, 256>>>();
    }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%s empty kernel: %.2f us per launch (back to back)\n", coop ? "cooperative" : "regular", ms);
  }
  return 0;
}
