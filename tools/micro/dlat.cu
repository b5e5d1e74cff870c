// Latency microbenchmark (one warp): dependent DADD / DMUL / FADD / SHFL.f64 / LDS chains.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b) {
  __shared__ double sm[64];
  sm[threadIdx.x] = a; sm[threadIdx.x + 32] = b;
  __syncwarp();
  double x = a + threadIdx.x;
  float f = (float)x;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { x = x + b; x = x + b; x = x + b; x = x + b; }
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { x = x * b; x = x * b; x = x * b; x = x * b; }
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { x = __shfl_up_sync(~0u, x, 1) + 0.0; x = __shfl_up_sync(~0u, x, 1); x = __shfl_up_sync(~0u, x, 1); x = __shfl_up_sync(~0u, x, 1); }
  long long t3 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { f = f + (float)b; f = f + (float)b; f = f + (float)b; f = f + (float)b; }
  long long t4 = clock64();
  int idx = threadIdx.x;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { idx = (int)sm[idx & 31]; idx = (int)sm[idx & 31]; idx = (int)sm[idx & 31]; idx = (int)sm[idx & 31]; }
  long long t5 = clock64();
  out[threadIdx.x] = x + f + idx;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  for (int r = 0; r < 2; ++r) k<<<1, 32>>>(o, c, 1.0, 1.0000001);
  long long h[5]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char* n[5] = {"DADD", "DMUL", "SHFL.f64(2x32)", "FADD", "LDS+cvt"};
  for (int i = 0; i < 5; ++i) printf("%-16s %.1f cycles/op\n", n[i], h[i] / 1024.0);
  return 0;
}
