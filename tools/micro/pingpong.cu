// Cross-SM one-way latency of a tagged 64-bit word through global memory
// (st.relaxed.gpu -> poll with ld.relaxed.gpu), as the mailboxes use it.
// Two CTAs ping-pong N times; prints ns per one-way trip (globaltimer).
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void pp(unsigned long long* box, int n, unsigned long long* out, int mode) {
  if (threadIdx.x) return;
  const int me = blockIdx.x;  // 0 pings, 1 pongs (other CTAs idle)
  if (me > 1) return;
  unsigned long long* mine = box + 32 * me;
  unsigned long long* other = box + 32 * (1 - me);
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  out[2 + me] = smid;
  unsigned long long t0 = gt();
  for (int i = 1; i <= n; ++i) {
    if (me == 0) {
      st_relaxed(other, i);
      if (mode) __threadfence();
      while (ld_relaxed(mine) != (unsigned long long)i) {}
    } else {
      while (ld_relaxed(mine) != (unsigned long long)i) {}
      st_relaxed(other, i);
      if (mode) __threadfence();
    }
  }
  if (me == 0) out[mode] = (gt() - t0);
}
int main() {
  unsigned long long *box, *out, h[4];
  cudaMalloc(&box, 4096);
  cudaMalloc(&out, 64);
  const int n = 20000;
  for (int grid : {2, 74, 148}) {
    for (int mode = 0; mode < 2; ++mode) {
      cudaMemset(box, 0, 4096);
      pp<<<grid, 32>>>(box, n, out, mode);
      cudaDeviceSynchronize();
      cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
      printf("grid %3d mode %s: %.0f ns one-way (SMs %llu, %llu)\n", grid, mode ? "fence  " : "relaxed",
             (double)h[mode] / (2.0 * n), h[2], h[3]);
    }
  }
  return 0;
}
