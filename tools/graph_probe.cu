// Probe: can a cooperative launch be stream-captured into a CUDA graph on sm_100a, and what
// is the per-kernel gap of a graph of N cooperative kernels vs plain stream launches?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 graph_probe.cu -o gp && ./gp
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_coop(int* x) {
  cg::this_grid().sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(x, 1);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* d;
  cudaMalloc(&d, 4);
  cudaMemset(d, 0, 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int grid = 2 * sms, N = 25;
  void* args[] = {&d};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < N; ++i) cudaLaunchCooperativeKernel((void*)k_coop, grid, 256, args, 0, s);
  cudaStreamSynchronize(s);
  cudaEventRecord(e0, s);
  for (int i = 0; i < N; ++i) cudaLaunchCooperativeKernel((void*)k_coop, grid, 256, args, 0, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms_stream = 0;
  cudaEventElapsedTime(&ms_stream, e0, e1);
  cudaGraph_t g;
  cudaError_t ec = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < N; ++i) cudaLaunchCooperativeKernel((void*)k_coop, grid, 256, args, 0, s);
  cudaError_t ee = cudaStreamEndCapture(s, &g);
  cudaGraphExec_t ge;
  cudaError_t ei = cudaGraphInstantiate(&ge, g, 0);
  printf("capture %s end %s instantiate %s\n", cudaGetErrorString(ec), cudaGetErrorString(ee),
         cudaGetErrorString(ei));
  if (ei == cudaSuccess) {
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(e0, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms_graph = 0;
    cudaEventElapsedTime(&ms_graph, e0, e1);
    int h = 0;
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("%d cooperative kernels: stream %.1f us, graph %.1f us (count %d, %s)\n", N,
           ms_stream * 1e3, ms_graph * 1e3, h, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
