// Microbenchmark of K3's compute-warp stage loop in isolation (one warp, data
// in shared memory, no producer): per stage 8 chain steps, 32 LDS of inputs,
// 8 STS of results, an mbarrier try_wait (pre-completed) + arrive.
//   mode 0: serial   (wait, loads, chain, stores)         -- today's K3 shape
//   mode 1: pipelined (loads of stage m+1 issued before the chain of stage m)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int S = 8, L = 32, D = 6;
template <typename T>
struct In { T rr[S], un[S], ue[S], ut[S]; };
template <typename T>
__device__ __forceinline__ void load(In<T>& x, const T* s, int lane) {
#pragma unroll
  for (int k = 0; k < S; ++k) {
    x.un[k] = s[(k * 4 + 0) * L + lane];
    x.ue[k] = s[(k * 4 + 1) * L + lane];
    x.ut[k] = s[(k * 4 + 2) * L + lane];
    x.rr[k] = s[(k * 4 + 3) * L + lane];
  }
}
__device__ __forceinline__ void arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ bool try_wait(uint32_t b, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}\n"
               : "=r"(ok) : "r"(b), "r"(par) : "memory");
  return ok;
}
template <typename T, int MODE>
__global__ void stage(T* out, long long* cyc, int nst) {
  extern __shared__ __align__(16) unsigned char sm[];
  T* slots = reinterpret_cast<T*>(sm);
  const int lane = threadIdx.x;
  for (int i = lane; i < D * S * 5 * L; i += 32) slots[i] = (T)(1.0 / (i + 3));
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + D * S * 5 * L * sizeof(T));
  const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(bars);
  if (lane == 0)
    for (int q = 0; q < D; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0 + 8 * q));
  __syncwarp();
  T dprev = (T)lane * (T)1e-3, win[S];
#pragma unroll
  for (int s = 0; s < S; ++s) win[s] = 0;
  const int eedge = (8 - (lane & 7)) & 7;
  In<T> cur, nxt;
  load(cur, slots + lane, 0);
  long long t0 = clock64();
#pragma unroll 1
  for (int m = 0; m < nst; ++m) {
    const int q = m % D, q1 = (m + 1) % D;
    T* s = slots + q * S * 5 * L;
    if (MODE == 0) {
      load(cur, s + lane, 0);
    } else {
      load(nxt, slots + q1 * S * 5 * L + lane, 0);
    }
    if (lane == 0) arrive(b0 + 8 * q);
    const T dE = (T)0.5, eN = (T)0.25;
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const T dN1 = __shfl_down_sync(0xffffffffu, dprev, 1);
      const T dEv = k == eedge ? dE : dprev;
      const T dN = lane == 31 ? eN : dN1;
      const T d = ((cur.rr[k] - cur.un[k] * dN) - cur.ue[k] * dEv) - cur.ut[k] * win[k];
      win[k] = d;
      dprev = d;
    }
#pragma unroll
    for (int k = 0; k < S; ++k) s[(S * 4 + k) * L / 8 * 0 + (4 * S) * L + k * 0 + lane + k * 0] = win[k];
    if (MODE == 1) cur = nxt;
  }
  long long t1 = clock64();
  out[lane] = dprev;
  if (lane == 0) cyc[0] = t1 - t0;
}
template <typename T, int MODE>
void run(const char* name) {
  T* o; long long* c; cudaMalloc(&o, 512); cudaMalloc(&c, 64);
  const int nst = 4096;
  size_t sh = D * S * 5 * L * sizeof(T) + 8 * D;
  cudaFuncSetAttribute(stage<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh);
  long long h = 0;
  for (int r = 0; r < 2; ++r) stage<T, MODE><<<1, 32, sh>>>(o, c, nst);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%s: %.1f cycles/stage (%s)\n", name, (double)h / nst, cudaGetErrorString(e));
}
int main() {
  run<double, 0>("fp64 serial   ");
  run<double, 1>("fp64 pipelined");
  run<float, 0>("fp32 serial   ");
  run<float, 1>("fp32 pipelined");
  return 0;
}
