// FP64 pipe peak microbenchmark (the roofline denominator MEASURED_PEAKS.json lacks).
// Each thread runs 8 independent DADD (or DMUL / DFMA) chains; grid = 148 SMs x 8 CTAs
// of 256 threads. Built with -fmad=false like the product so DADD/DMUL stay separate.
// Exported C function returns achieved GFLOP/s (DFMA counted as 2 flops).
#include <cuda_runtime.h>

#include <cstdio>

template <int MODE>
__global__ void k_fp64(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (MODE == 0) x[k] = x[k] + a;
      else if (MODE == 1) x[k] = x[k] * b;
      else x[k] = fma(x[k], b, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

extern "C" double sb_fp64_peak_gflops(int mode, int device) {
  if (cudaSetDevice(device) != cudaSuccess) return -1.0;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
  double* out;
  cudaMalloc(&out, sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    if (mode == 0) k_fp64<0><<<blocks, threads>>>(out, iters, 1e-9, 0.999999);
    else if (mode == 1) k_fp64<1><<<blocks, threads>>>(out, iters, 1e-9, 0.999999);
    else k_fp64<2><<<blocks, threads>>>(out, iters, 1e-9, 0.999999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  cudaFree(out);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  double ops = double(blocks) * threads * iters * 8.0 * (mode == 2 ? 2.0 : 1.0);
  return ops / (best * 1e-3) / 1e9;
}
