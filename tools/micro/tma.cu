// Per-SM bulk-copy (TMA) and LDGSTS throughput / latency from an L2-resident source.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int DEPTH>
__global__ void k_tma(const char* src, long long* cyc, int n, int bytes) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[8];
  if (threadIdx.x == 0) {
    for (int i = 0; i < DEPTH; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long c0 = clock64();
  for (int i = 0; i < n + DEPTH; ++i) {
    const int slot = i % DEPTH;
    if (i >= DEPTH) {  // wait for copy i-DEPTH
      const uint32_t par = ((i - DEPTH) / DEPTH) & 1;
      uint32_t ok;
      do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(saddr(&bar[slot])), "r"(par) : "memory");
      } while (!ok);
    }
    if (i < n) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&bar[slot])), "r"(bytes));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(saddr(sm + slot * bytes)), "l"(src + (long long)(i % 64) * bytes), "r"(bytes), "r"(saddr(&bar[slot])) : "memory");
    }
  }
  cyc[blockIdx.x] = clock64() - c0;
}
__global__ void k_ldgsts(const char* src, long long* cyc, int n, int bytes) {
  extern __shared__ __align__(128) char sm[];
  long long c0 = clock64();
  const int per = bytes / 16 / blockDim.x;
  for (int i = 0; i < n; ++i) {
    const char* s = src + (long long)(i % 64) * bytes;
    char* d = sm + (i % 3) * bytes;
    for (int j = 0; j < per; ++j) {
      const int off = (j * blockDim.x + threadIdx.x) * 16;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr(d + off)), "l"(s + off) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 2;" ::: "memory");
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
}
int main() {
  const int bytes = 24576, n = 2000;
  char* src; long long* cyc;
  cudaMalloc(&src, 64 * bytes); cudaMemset(src, 1, 64 * bytes);
  cudaMallocManaged(&cyc, 1024 * 8);
  cudaFuncSetAttribute(k_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * bytes);
  cudaFuncSetAttribute(k_tma<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * bytes);
  cudaFuncSetAttribute(k_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * bytes);
  cudaFuncSetAttribute(k_ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * bytes);
  for (int rep = 0; rep < 2; ++rep) {
    k_tma<1><<<1, 32, 3 * bytes>>>(src, cyc, n, bytes); cudaDeviceSynchronize();
    printf("TMA depth1 (latency): %.0f cycles per 24KB copy\n", (double)cyc[0] / n);
    k_tma<3><<<1, 32, 3 * bytes>>>(src, cyc, n, bytes); cudaDeviceSynchronize();
    printf("TMA depth3: %.0f cycles/copy = %.1f B/clk\n", (double)cyc[0] / n, bytes * (double)n / cyc[0]);
    k_tma<4><<<1, 32, 4 * bytes>>>(src, cyc, n, bytes); cudaDeviceSynchronize();
    printf("TMA depth4: %.0f cycles/copy = %.1f B/clk\n", (double)cyc[0] / n, bytes * (double)n / cyc[0]);
    k_tma<3><<<148, 32, 3 * bytes>>>(src, cyc, n, bytes); cudaDeviceSynchronize();
    printf("TMA depth3 x148 CTAs: %.0f cycles/copy = %.1f B/clk/SM\n", (double)cyc[0] / n, bytes * (double)n / cyc[0]);
    k_ldgsts<<<1, 256, 3 * bytes>>>(src, cyc, n, bytes); cudaDeviceSynchronize();
    printf("LDGSTS 256 thr depth3: %.0f cycles/copy = %.1f B/clk\n", (double)cyc[0] / n, bytes * (double)n / cyc[0]);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
