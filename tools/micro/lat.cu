// Microbenchmarks of the latencies that make up one wavefront step (B200).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k_lat(double* out, long long* cyc, int n) {
  __shared__ double sm[1024];
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x;
  for (int i = t; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(&bar)), "r"(1));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(&bar)));  // phase 0 done
  }
  __syncthreads();
  double a = out[0], b = out[1];
  for (int i = 0; i < n; ++i) { a = a + b; a = a + b; a = a + b; a = a + b; }  // warm-up
  __syncthreads();
  // 1. dependent DADD chain
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) { a = a + b; a = a + b; a = a + b; a = a + b; }
  long long c1 = clock64();
  // 2. dependent DMUL chain
  for (int i = 0; i < n; ++i) { b = b * 1.0000001; b = b * 1.0000001; b = b * 1.0000001; b = b * 1.0000001; }
  long long c2 = clock64();
  // 3. dependent LDS chain (pointer chasing through smem)
  int idx = t & 7;
  for (int i = 0; i < n; ++i) { idx = (int)sm[idx] & 7; idx = (int)sm[idx + 8] & 7; idx = (int)sm[idx + 16] & 7; idx = (int)sm[idx + 24] & 7; }
  long long c3 = clock64();
  // 4. mbarrier try_wait on a completed phase
  uint32_t ok = 0;
  for (int i = 0; i < n * 4; ++i) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(saddr(&bar)), "r"(0) : "memory");
  }
  long long c4 = clock64();
  // 5. __syncthreads
  for (int i = 0; i < n * 4; ++i) __syncthreads();
  long long c5 = clock64();
  // 6. fp32 chain
  float f = (float)a, g = (float)b;
  for (int i = 0; i < n; ++i) { f = f + g; f = f + g; f = f + g; f = f + g; }
  long long c6 = clock64();
  // 7. globaltimer reads
  unsigned long long gt = 0;
  for (int i = 0; i < n * 4; ++i) { unsigned long long x; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(x)); gt += x; }
  long long c7 = clock64();
  // 8. __syncwarp + lane-0 mbarrier arrive (release) on a fresh barrier ring
  for (int i = 0; i < n * 4; ++i) {
    __syncwarp();
    if ((t & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(&bar)) : "memory");
  }
  long long c8 = clock64();
  if (t == 0) {
    out[2] = a + b + idx + ok + f + (double)(gt & 1);
    cyc[0] = c1 - c0; cyc[1] = c2 - c1; cyc[2] = c3 - c2; cyc[3] = c4 - c3; cyc[4] = c5 - c4;
    cyc[5] = c6 - c5; cyc[6] = c7 - c6; cyc[7] = c8 - c7;
  }
}
int main() {
  double* out; long long* cyc;
  cudaMallocManaged(&out, 64); cudaMallocManaged(&cyc, 128);
  out[0] = 1.0; out[1] = 1e-12;
  const int n = 1000;
  for (int threads : {32, 256}) {
    k_lat<<<1, threads>>>(out, cyc, n);
    cudaDeviceSynchronize();
    const double ops = 4.0 * n;
    printf("threads %d: DADD %.1f  DMUL %.1f  LDS-chain %.1f  mbar-trywait %.1f  syncthreads %.1f  FADD %.1f  globaltimer %.1f  syncwarp+arrive %.1f cycles/op\n",
           threads, cyc[0] / ops, cyc[1] / ops, cyc[2] / ops, cyc[3] / ops, cyc[4] / ops, cyc[5] / ops, cyc[6] / ops, cyc[7] / ops);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
