// Dependent-chain latency probe (cycles per op) for the ops on the narrow-phase critical
// path: DADD, DMUL, DFMA, DDIV, DSQRT, 64-bit IMUL, shared-memory load, shuffle, ballot.
// Built with -fmad=false like the product. Run: nvcc ... -o lat && ./lat
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 1024;

__global__ void k_lat(double seed, unsigned long long* out, double* sink) {
  __shared__ int chase[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) chase[i] = (i * 37 + 11) & 1023;
  __syncthreads();
  double x = seed + threadIdx.x, y = 1.0000001, z = 0.9999999;
  long long t0, t1;
  // DADD
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x + y;
  t1 = clock64();
  out[0] = t1 - t0;
  // DMUL
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x * z;
  t1 = clock64();
  out[1] = t1 - t0;
  // DFMA
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, z, y);
  t1 = clock64();
  out[2] = t1 - t0;
  // DDIV
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N / 8; ++i) x = y / x;
  t1 = clock64();
  out[3] = (t1 - t0) * 8;
  // DSQRT
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N / 8; ++i) x = sqrt(x + y);
  t1 = clock64();
  out[4] = (t1 - t0) * 8;
  // 64-bit integer multiply-add
  unsigned long long u = (unsigned long long)seed + threadIdx.x;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) u = u * 6364136223846793005ULL + 1442695040888963407ULL;
  t1 = clock64();
  out[5] = t1 - t0;
  // shared-memory pointer chase
  int p = threadIdx.x & 1023;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) p = chase[p];
  t1 = clock64();
  out[6] = t1 - t0;
  // shuffle chain
  int s = threadIdx.x;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) s = __shfl_sync(0xffffffffu, s, (s + 1) & 31);
  t1 = clock64();
  out[7] = t1 - t0;
  // FP32 add
  float f = (float)seed, g = 1.0001f;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) f = f + g;
  t1 = clock64();
  out[8] = t1 - t0;
  sink[threadIdx.x] = x + (double)u + p + s + f;
}

int main() {
  unsigned long long* d;
  double* sink;
  cudaMalloc(&d, 16 * sizeof(unsigned long long));
  cudaMalloc(&sink, 32 * sizeof(double));
  k_lat<<<1, 32>>>(1.5, d, sink);
  k_lat<<<1, 32>>>(1.5, d, sink);
  unsigned long long h[16];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  const char* names[] = {"dadd", "dmul", "dfma", "ddiv", "dsqrt", "imad64", "lds_chase", "shfl", "fadd"};
  for (int i = 0; i < 9; ++i) printf("%-10s %7.1f cycles/op\n", names[i], (double)h[i] / N);
  return 0;
}
