// Microbenchmark: K3's per-step dependency chain in one warp (fp64 and fp32):
//   dN = shfl_down(dprev); dN = lane==31 ? e : dN; dE = p ? e2 : dprev
//   d = ((R - UN*dN) - UE*dE) - UTdT ; dprev = d
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void chain(T* out, long long* cyc, int steps, T a, T b, T c) {
  const int lane = threadIdx.x;
  T dprev = (T)lane * (T)1e-3, e = (T)0.5, e2 = (T)0.25;
  T rr = a, un = b, ue = c, utdt = (T)1e-9;
  const bool p = (lane & 7) == 3;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < steps; i += 8) {
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      T dN1 = __shfl_down_sync(0xffffffffu, dprev, 1);
      T dEv = p ? e2 : dprev;
      T dN = lane == 31 ? e : dN1;
      T d = ((rr - un * dN) - ue * dEv) - utdt;
      dprev = d;
    }
  }
  long long t1 = clock64();
  out[lane] = dprev;
  if (lane == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  long long h;
  const int steps = 8 * 4096;
  chain<double><<<1, 32>>>(o, c, steps, 1.0, 0.25, 0.125);
  chain<double><<<1, 32>>>(o, c, steps, 1.0, 0.25, 0.125);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("fp64 chain: %.1f cycles/step\n", (double)h / steps);
  chain<float><<<1, 32>>>((float*)o, c, steps, 1.f, 0.25f, 0.125f);
  chain<float><<<1, 32>>>((float*)o, c, steps, 1.f, 0.25f, 0.125f);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("fp32 chain: %.1f cycles/step\n", (double)h / steps);
  return 0;
}
