// Probe: cooperative launch + thread-block clusters on sm_100a (cudaLaunchKernelEx with both
// attributes), DSMEM atomics into a peer CTA, grid.sync across the whole grid.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 cluster_probe.cu -o cp && ./cp
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_probe(unsigned* out, int rounds) {
  __shared__ unsigned box[4];
  cg::cluster_group cl = cg::this_cluster();
  cg::grid_group grid = cg::this_grid();
  if (threadIdx.x < 4) box[threadIdx.x] = 0;
  cl.sync();
  const unsigned peer = (cl.block_rank() + 1) % cl.num_blocks();
  unsigned* pbox = cl.map_shared_rank(box, peer);
  for (int r = 0; r < rounds; ++r) {
    atomicAdd(pbox + 0, 1u);  // every thread adds one into the next CTA's smem
    cl.sync();
    grid.sync();
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = box[0];
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* d;
  cudaMalloc(&d, 4096 * 4);
  for (int cs : {2, 4, 8}) {
    cudaFuncSetAttribute((const void*)k_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    int grid = 2 * sms;
    grid -= grid % cs;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = cs;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, (const void*)k_probe, &cfg);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_probe, d, 10);
    cudaError_t e2 = cudaDeviceSynchronize();
    unsigned h[8];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("cluster %d grid %d max active clusters %d: launch %s sync %s box[0]=%u (expect %u)\n", cs,
           grid, ncl, cudaGetErrorString(e), cudaGetErrorString(e2), h[0], 256u * 10u);
  }
  return 0;
}
