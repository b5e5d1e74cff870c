// sip_kernels.cu -- sm_100a kernels of the SIP hot path.
//
//   K1 k_factor    Stone ILU factor          wavefront, fp64
//   K2 k_forward   residual + L1 norm + forward substitution   wavefront, bulk-copy ring
//                  (resforward3d, SPEC.md:155 + SPEC.md:173)
//   K3 k_backward  backward substitution + phi update          wavefront, bulk-copy ring
//                  (backward3d)
//   K4 k_face_copy face-halo copies / pack / unpack (exvec)
//   K5 k_convert   fp64 -> fp32 (Field3::cast, field.hpp:61-68)
//   K7 k_scatter / k_gather / k_ghost_in   Field3 <-> tile-slice layout
//
// Wavefront scheme: a CTA owns a 16x16-column tile and walks the
// tile's hyperplanes t = k + ti + tj.  Inside a tile the W/S neighbours of a
// cell were produced one step earlier by neighbouring threads (double-buffered
// shared memory, one __syncthreads per step); the B neighbour is the thread's
// own previous value (register).  Across tiles, values travel through L2 and
// each tile publishes a monotone progress counter (release/acquire), so there
// is no grid-wide barrier: upstream tiles run ahead and the hand-off latency
// becomes pipeline skew.  Tiles are claimed through an atomic ticket in
// topological order, so the kernel is deadlock-free for any residency.
//
// Bitwise parity: every cell performs the oracle's operations in the oracle's
// order (oracle/sip_oracle.c header); this file is compiled with
// --fmad=false and IEEE division, so no contraction changes the rounding.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "sip_internal.h"

namespace sipb {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}
// Watchdog: a spin that makes no progress for kWatchdogNs aborts the kernel
// (__trap -> the launch fails with an error instead of hanging the GPU).
constexpr unsigned long long kWatchdogNs = 4000000000ULL;
#define TRCLK() clock64()
// per-step cycle tracing of one tile (tools/trace_steps.py): debug builds only
#ifdef SIPB_STEP_TRACE
constexpr bool kStepTrace = true;
#else
constexpr bool kStepTrace = false;
#endif  // debug trace clock (SM cycles; use gtime() for cross-SM analysis)
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __noinline__ void watchdog_fire(int where) {
  printf("sip watchdog: block %d thread %d stalled at site %d\n", blockIdx.x, threadIdx.x, where);
  __trap();
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity, int where = 0) {
  const uint32_t a = saddr(b);
  uint32_t ok;
  unsigned long long t0 = 0;
  int n = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (!ok && ((++n & 255) == 0)) {
      if (t0 == 0) t0 = gtime();
      else if (gtime() - t0 > kWatchdogNs) watchdog_fire(where);
    }
  } while (!ok);
}
// Idle-loop watchdog of the service warps (reset whenever work was done).
struct Watchdog {
  unsigned long long t0 = 0;
  int n = 0;
  __device__ __forceinline__ void progress() { t0 = 0; n = 0; }
  __device__ __forceinline__ void idle(int where) {
    if ((++n & 255) == 0) {
      if (t0 == 0) t0 = gtime();
      else if (gtime() - t0 > kWatchdogNs) watchdog_fire(where);
    }
  }
};
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u32(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ float ld_relaxed(const float* p) {
  float v;
  asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}

// thread position p -> (ti, tj) of the anti-diagonal numbering
__device__ __forceinline__ void pos_to_tij(int p, int& ti, int& tj) {
  int d = 0;
  while (diag_off(d + 1) <= p) ++d;
  const int lo = d - (kTJ - 1) > 0 ? d - (kTJ - 1) : 0;
  ti = lo + (p - diag_off(d));
  tj = d - ti;
}

// Valid cell range [lo, hi) of slice t in a tile of nz planes, widened to 16 B.
template <typename T>
__device__ __forceinline__ void slice_range(int t, int nz, int& lo, int& hi) {
  constexpr int EPV = 16 / sizeof(T);
  const int dlo = t - nz + 1 > 0 ? t - nz + 1 : 0;
  const int dhi = t < kD - 1 ? t : kD - 1;  // inclusive
  lo = diag_off(dlo) & ~(EPV - 1);
  hi = (diag_off(dhi + 1) + EPV - 1) & ~(EPV - 1);
  if (hi > kTT) hi = kTT;
}

// Copy `na` arrays of one slice (pack stride na*TT) into smem (stride TT).
template <typename T>
__device__ __forceinline__ uint32_t issue_slice(T* dst, const T* src, int na, int t, int nz,
                                                uint64_t* bar, bool arm, uint32_t extra_tx) {
  int lo, hi;
  slice_range<T>(t, nz, lo, hi);
  const uint32_t bytes = static_cast<uint32_t>(na * (hi - lo) * sizeof(T));
  if (arm) mbar_expect_tx(bar, bytes + extra_tx);
  if (lo == 0 && hi == kTT) {
    bulk_g2s(dst, src, bytes, bar);
  } else {
    for (int a = 0; a < na; ++a)
      bulk_g2s(dst + a * kTT + lo, src + a * kTT + lo, static_cast<uint32_t>((hi - lo) * sizeof(T)),
               bar);
  }
  return bytes;
}
template <typename T>
__device__ __forceinline__ uint32_t slice_bytes(int t, int nz, int na) {
  int lo, hi;
  slice_range<T>(t, nz, lo, hi);
  return static_cast<uint32_t>(na * (hi - lo) * sizeof(T));
}

// Deterministic CTA sum (fixed xor-tree per warp, warps summed in order).
__device__ __forceinline__ double cta_sum(double v, double* s_red) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) s_red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int x = 0; x < (int)(blockDim.x >> 5); ++x) s += s_red[x];
  return s;  // valid on thread 0
}

constexpr int kProgOff = 32;  // state layout: [0] ticket, [1] done, progress at +32

// =============================================================================
// K1: Stone factorisation (fp64), SPEC.md:146 -- once per system revision.
// =============================================================================
__global__ void __launch_bounds__(kTT, 1) k_factor(const FactorParams P) {
  __shared__ double s_U[2][3][kTT];
  __shared__ int s_tile;
  const int p = threadIdx.x;
  int ti, tj;
  pos_to_tij(p, ti, tj);
  const int d = ti + tj;
  const int pW = ti > 0 ? tile_pos(ti - 1, tj) : p;
  const int pS = tj > 0 ? tile_pos(ti, tj - 1) : p;
  unsigned* const prog = P.state + kProgOff;
  const double alpha = P.alpha;

  for (;;) {
    __syncthreads();
    if (p == 0) s_tile = atomicAdd(P.state, 1u);
    __syncthreads();
    const int tk = s_tile;
    if (tk >= P.ntiles) break;
    const int tid = P.order[tk];
    const TileDesc td = P.tiles[tid];
    const BlockDesc bd = P.blocks[td.block];
    const int NS = td.ns, nz = td.nz;
    const bool col = ti < td.wI && tj < td.wJ;
    const bool inW = ti > 0, inS = tj > 0;
    const long long slotW = td.nW >= 0 ? P.tiles[td.nW].slot : 0;
    const long long slotS = td.nS >= 0 ? P.tiles[td.nS].slot : 0;
    const int posW = tile_pos(kTI - 1, tj), posS = tile_pos(ti, kTJ - 1);
    double unB = 0.0, ueB = 0.0, utB = 0.0;
    unsigned cW = 0, cS = 0;
    for (int t = 0; t < NS; ++t) {
      __syncthreads();
      if (p == 0 && t > 0) {
        __threadfence();
        st_release(&prog[tid], (unsigned)t);
      }
      const int k = t - d;
      if (col && k >= 0 && k < nz) {
        double unW = 0.0, ueW = 0.0, utW = 0.0, unS = 0.0, ueS = 0.0, utS = 0.0;
        if (inW) {
          const int b = ((t - 1) & 1);
          unW = s_U[b][0][pW]; ueW = s_U[b][1][pW]; utW = s_U[b][2][pW];
        } else if (td.nW >= 0) {
          const unsigned need = min(t + kTI, NS);
          Watchdog wd;
          while (cW < need) {
            cW = ld_acquire(&prog[td.nW]);
            wd.idle(1);
          }
          const long long base = (slotW + k + kTI - 1 + tj) * B_NA * kTT + posW;
          unW = ld_relaxed(P.bw + base + B_UN * kTT);
          ueW = ld_relaxed(P.bw + base + B_UE * kTT);
          utW = ld_relaxed(P.bw + base + B_UT * kTT);
        }
        if (inS) {
          const int b = ((t - 1) & 1);
          unS = s_U[b][0][pS]; ueS = s_U[b][1][pS]; utS = s_U[b][2][pS];
        } else if (td.nS >= 0) {
          const unsigned need = min(t + kTJ, NS);
          Watchdog wd;
          while (cS < need) {
            cS = ld_acquire(&prog[td.nS]);
            wd.idle(2);
          }
          const long long base = (slotS + k + ti + kTJ - 1) * B_NA * kTT + posS;
          unS = ld_relaxed(P.bw + base + B_UN * kTT);
          ueS = ld_relaxed(P.bw + base + B_UE * kTT);
          utS = ld_relaxed(P.bw + base + B_UT * kTT);
        }
        double* f = P.fw + (td.slot + t) * F_NA * kTT + p;
        const double ap = f[F_AP * kTT], aw = f[F_AW * kTT], ae = f[F_AE * kTT];
        const double as = f[F_AS * kTT], an = f[F_AN * kTT], ab = f[F_AB * kTT];
        const double at = f[F_AT * kTT];
        // SPEC.md:146 with m_nb = A_nb, operation order of oracle/sip_oracle.c
        const double lb = ab / (1.0 + alpha * (unB + ueB));
        const double lw = aw / (1.0 + alpha * (unW + utW));
        const double ls = as / (1.0 + alpha * (ueS + utS));
        const double p1 = alpha * (lb * unB + lw * unW);
        const double p2 = alpha * (lb * ueB + ls * ueS);
        const double p3 = alpha * (lw * utW + ls * utS);
        const double den = ap + p1 + p2 + p3 - lb * utB - lw * ueW - ls * unS;
        if (!(fabs(den) >= 1e-30)) {
          const long long c = (long long)(td.i0 + ti + 1) +
                              (long long)(bd.nx + 2) *
                                  ((long long)(td.j0 + tj + 1) + (long long)(bd.ny + 2) * (k + 1));
          atomicMin(P.bad, ((unsigned long long)bd.id << 40) | (unsigned long long)c);
        }
        const double lp = 1.0 / den;
        const double un = (an - p1) * lp, ue = (ae - p2) * lp, ut = (at - p3) * lp;
        f[F_LB * kTT] = lb;
        f[F_LW * kTT] = lw;
        f[F_LS * kTT] = ls;
        f[F_LP * kTT] = lp;
        double* u = P.bw + (td.slot + t) * B_NA * kTT + p;
        u[B_UN * kTT] = un;
        u[B_UE * kTT] = ue;
        u[B_UT * kTT] = ut;
        s_U[t & 1][0][p] = un;
        s_U[t & 1][1][p] = ue;
        s_U[t & 1][2][p] = ut;
        unB = un; ueB = ue; utB = ut;
      }
    }
    __syncthreads();
    if (p == 0) {
      __threadfence();
      st_release(&prog[tid], (unsigned)NS);
    }
  }
}

// =============================================================================
// K2 / K3 are warp-specialised: 8 compute warps (one thread per tile column)
// plus two service warps.
//   loader warp: retires finished steps and refills the slice ring with bulk
//                copies (cp.async.bulk -> shared, mbarrier complete_tx), and
//                keeps an L2 prefetch front (cp.async.bulk.prefetch.L2) kPF
//                slices ahead, so ring refills hit L2 even on the wavefront's
//                latency-bound critical path.  Shared-memory work only.
//   linker warp: forwards the tile's outgoing edge values (copied by the
//                compute warps into a shared out-record) to global memory,
//                publishes the tile's progress counter (fence.acq_rel.gpu +
//                relaxed store = release pattern), polls the upstream tiles'
//                counters and prefetches every cross-tile value a step needs
//                (neighbour phi / R / delta, ghost phi) into a shared
//                "edge record".
// The compute warps never wait on a global-memory latency: per step they wait
// on shared-memory mbarriers, compute, store, and meet at one named barrier.
// =============================================================================
constexpr int kCompute = kTT;       // compute threads (8 warps)
constexpr int kThreads = kTT + 64;  // + publisher, fetcher warps
constexpr int kComputeWarps = kTT / 32;
constexpr int kPublisherWarp = kComputeWarps, kFetcherWarp = kComputeWarps + 1;
constexpr int kPF = 0;              // L2 prefetch distance (slices; 0 = off: the TMA unit is the per-SM bottleneck)

__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(saddr(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void bar_compute() {  // named barrier of the compute warps
  asm volatile("bar.sync 1, %0;" ::"n"(kCompute) : "memory");
}
// Explicit 32-bit shared-window accesses: keep ring addresses in plain
// registers (no generic->shared rematerialisation in the step loops).
template <typename T>
__device__ __forceinline__ T lds(uint32_t a);
template <>
__device__ __forceinline__ double lds<double>(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
template <>
__device__ __forceinline__ float lds<float>(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v));
}
__device__ __forceinline__ void sts(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v));
}
__device__ __forceinline__ void mbar_arrive_a(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __noinline__ void mbar_wait_slow(uint32_t a, uint32_t parity, int where) {
  const unsigned long long t0 = gtime();
  uint32_t ok;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (!ok && gtime() - t0 > kWatchdogNs) watchdog_fire(where);
  } while (!ok);
}
// Fast path: one try_wait; the (rare) retry loop with its watchdog is out of line.
__device__ __forceinline__ void mbar_wait_a(uint32_t a, uint32_t parity, int where) {
  uint32_t ok;
  asm volatile(
      "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  if (!ok) mbar_wait_slow(a, parity, where);
}
// advance a ring address by one slot (wrap-around without division)
__device__ __forceinline__ uint32_t ring_next(uint32_t a, uint32_t base, uint32_t slot, uint32_t size) {
  a += slot;
  return a >= base + size ? a - size : a;
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// LSU-side L2 prefetch of one 128-byte line (does not use the TMA engine)
__device__ __forceinline__ void prefetch_line_l2(const void* p) {
#ifdef SIPB_EXP_NOPF
  return;
#endif
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}
constexpr int kPFL = 6;  // steps of LSU L2 prefetch beyond the slice ring
__device__ __forceinline__ void st_release_cta_s(int* p, int v) {
  asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(saddr(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed_cta_s(const int* p) {
  int v;
  asm volatile("ld.relaxed.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr(p)) : "memory");
  return v;
}
__device__ __forceinline__ void fence_cta() { asm volatile("fence.acq_rel.cta;" ::: "memory"); }
// Spin until *p >= need with cheap relaxed loads, then one CTA fence (the
// relaxed load that observed the released value + fence = acquire pattern).
__device__ __forceinline__ void wait_counter(const int* p, int need, int site) {
  if (ld_relaxed_cta_s(p) < need) {
    unsigned long long t0 = 0;
    int n = 0;
    while (ld_relaxed_cta_s(p) < need) {
      if ((++n & 255) == 0) {
        if (t0 == 0) t0 = gtime();
        else if (gtime() - t0 > kWatchdogNs) watchdog_fire(site);
      }
    }
  }
  fence_cta();
}
__device__ __forceinline__ int ld_acquire_cta_s(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(saddr(p)) : "memory");
  return v;
}

// ---- tagged edge words: value bits + 32-bit tag, single-copy atomic 64-bit stores
__device__ __forceinline__ uint32_t edge_tag(unsigned epoch, int k) {
  return ((epoch & 0xFFFFu) << 16) | (uint32_t)(k & 0xFFFF);
}
__device__ __forceinline__ void put_tagged(unsigned long long* dst, float v, uint32_t tag) {
  const unsigned long long w = ((unsigned long long)tag << 32) | __float_as_uint(v);
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(dst), "l"(w) : "memory");
}
__device__ __forceinline__ void put_tagged(unsigned long long* dst, double v, uint32_t tag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned long long w0 = ((unsigned long long)tag << 32) | (b >> 32);
  const unsigned long long w1 = ((unsigned long long)tag << 32) | (b & 0xFFFFFFFFull);
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(dst), "l"(w0), "l"(w1) : "memory");
}
__device__ __forceinline__ bool get_tagged(const unsigned long long* src, uint32_t tag, float& v) {
  unsigned long long w;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(src) : "memory");
  v = __uint_as_float((uint32_t)w);
  return (uint32_t)(w >> 32) == tag;
}
__device__ __forceinline__ bool get_tagged(const unsigned long long* src, uint32_t tag, double& v) {
  unsigned long long w0, w1;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(src) : "memory");
  v = __longlong_as_double((long long)((w0 << 32) | (w1 & 0xFFFFFFFFull)));
  return (uint32_t)(w0 >> 32) == tag && (uint32_t)(w1 >> 32) == tag;
}
template <typename T>
constexpr int kTagWords = sizeof(T) / 4;  // 64-bit words per tagged value

// Warp-collective poll of a neighbour's progress counter.  Every lane performs
// its own acquire (so its later loads are ordered) and the warp takes the
// minimum, so all lanes agree on a value each of them has acquired.  Lanes of
// a warp may execute independently (Volta+ scheduling): decisions taken from
// memory must be made uniform explicitly.
__device__ __forceinline__ unsigned poll_progress(const unsigned* p, unsigned cached, unsigned need) {
  if (cached >= need) return cached;
  return __reduce_min_sync(0xffffffffu, ld_acquire(p));
}
// Warp-collective test of a step-done barrier: complete only if every lane
// observed completion (each such lane holds its own acquire).
__device__ __forceinline__ bool warp_test(uint64_t* b, uint32_t parity) {
  return __all_sync(0xffffffffu, mbar_test(b, parity));
}

template <typename T, int SF>
struct FwdCfg {
  static constexpr int SP = SF + 2;  // phi slice s is read while preparing steps s-1, s, s+1
  static constexpr int ER = 16;      // edge records (deep ring; readiness rides on the slot barrier)
  static constexpr int OR = 8;       // outgoing edge records
  static constexpr int EB = 32;      // step barriers E[x] (> ER + SF, > OR + SF + 1)
  static constexpr int NE = 96;      // phiW, phiE, phiS, phiN, RW, RS (16 each)
  // the forward pack is not staged in shared memory: each compute thread
  // loads its own cell's 12 values with coalesced LDG one step ahead
  static constexpr size_t bytes = (size_t)(SP + 4) * kTT * sizeof(T) +
                                  (size_t)(ER * NE + OR * 32) * sizeof(T) +
                                  (SF + EB) * sizeof(uint64_t);
};

// Step pipeline of one compute thread (K2):
//   prep(x):  wait for slice x / edge record x, evaluate the residual of step x
//             and pre = r - LB*R_B (everything that does not depend on the
//             in-tile neighbours of step x-1), then signal "slice x consumed";
//   step(t):  after the named barrier, R = ((pre - LW*R_W) - LS*R_S) * LP,
//             store, signal "step t done", prep(t+1), barrier.
// The recurrence's critical path per step is thus two shared loads, four
// dependent flops and one barrier; the operation order per cell is exactly
// the oracle's (pre is the oracle's first subtraction).
template <typename T, int SF>
__global__ void __launch_bounds__(kThreads, 2) k_forward(const SweepParams<T> P) {
  using C = FwdCfg<T, SF>;
  constexpr int SP = C::SP, ER = C::ER, EB = C::EB, NE = C::NE, OR = C::OR;
  static_assert(EB > ER + SF && EB > OR + SF + 1, "barrier rings must cover the run-ahead");
  extern __shared__ __align__(128) unsigned char smem[];
  T* s_ph = reinterpret_cast<T*>(smem);
  T* s_R = s_ph + SP * kTT;
  T* s_edge = s_R + 2 * kTT;
  T* s_out = s_edge + ER * NE;  // [OR][32]: R of the E column (tj) and N row (16 + ti)
  T* s_gh = s_out + OR * 32;    // [2][kTT]: ghost phi below / above each column
  // b_fw[x % SF] completes when phi slice x+1 (and, for x = 0, phi slice 0)
  // has landed AND the fetcher has written edge record x
  uint64_t* b_fw = reinterpret_cast<uint64_t*>(s_gh + 2 * kTT);
  // E[x] (b_step[(eq + x) % EB], x = 0..NS): prep(x) is done -- slice x, phi
  // slice x-1 and edge record x are consumed -- and step x-1 is complete
  // (its R is in s_R / s_out).  One arrival per compute warp per step.
  uint64_t* b_step = b_fw + SF;
  __shared__ int s_tile, s_last, s_linked;
  __shared__ double s_red[kThreads / 32];

  const int p = threadIdx.x;
  const int warp = p >> 5, lane = p & 31;
  int ti = 0, tj = 0;
  if (warp < kComputeWarps) pos_to_tij(p, ti, tj);
  const int d = ti + tj;
  const int pW = ti > 0 ? tile_pos(ti - 1, tj) : 0;
  const int pE = ti < kTI - 1 ? tile_pos(ti + 1, tj) : 0;
  const int pS = tj > 0 ? tile_pos(ti, tj - 1) : 0;
  const int pN = tj < kTJ - 1 ? tile_pos(ti, tj + 1) : 0;
  unsigned* const prog = P.state + kProgOff;

  if (p == 0) {
    for (int b = 0; b < SF; ++b) mbar_init(&b_fw[b], 2);  // fetcher: phi slice (expect_tx) + record
    for (int b = 0; b < EB; ++b) mbar_init(&b_step[b], kCompute / 32);
    fence_mbar_init();
  }
  uint32_t sq = 0;  // CTA-uniform step sequence base (slot rings advance NS per tile)
  uint32_t eq = 0;  // E ring base (advances NS + 1 per tile)
  const unsigned epoch = *P.epoch;  // stable for this launch (bumped by the finaliser)

  for (;;) {
    __syncthreads();
    if (p == 0) {
      s_tile = atomicAdd(P.state, 1u);
      s_linked = 0;
    }
    __syncthreads();
    const int tk = s_tile;
    if (tk >= P.ntiles) break;
    const int tid = P.order[tk];
    const TileDesc td = P.tiles[tid];
    const BlockDesc bd = P.blocks[td.block];
    const int NS = td.ns, nz = td.nz;
    double nrm = 0.0;
    if (P.trace && p == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      P.trace[4 * tid + 0] = gtime();
      P.trace[4 * tid + 2] = smid;
      P.trace[4 * tid + 3] = blockIdx.x;
    }

    if (warp == kPublisherWarp) {
      // --------------------------------------------------------- publisher
      // outgoing edge: lane c < 16 -> E column cell (TI-1, c), lane >= 16 -> N row cell (c, TJ-1)
      // written as tagged words: the consumer validates each value by its tag,
      // so no fence or progress counter is needed
      const bool we = lane < 16;
      const int c = lane & 15;
      const bool outok = we ? (td.nE >= 0 && c < td.wJ) : (td.nN >= 0 && c < td.wI);
      const int outoff = we ? (kTI - 1) + c : c + (kTJ - 1);
      unsigned long long* outdst = (we ? P.tagA : P.tagB) + (td.edge + c) * kTagWords<T>;
      const T* fw_pf = P.fw + td.slot * F_NA * kTT;
      if (lane == 0)  // warm the first kPFL + 1 forward-pack slices (one bulk L2 prefetch each)
        for (int xs = 0; xs <= kPFL && xs < NS; ++xs)
          prefetch_l2(fw_pf + (long long)xs * F_NA * kTT, F_NA * kTT * sizeof(T));
      // phi slices: step s's transaction (phi slice s+1, + slice 0 for s = 0)
      // on b_fw[s % SF], armed once prep(s - SF) is done (phi slice s+1 reuses
      // the slot of slice s+1-SP, SP = SF + 2)
      const T* ph_src = P.phi + td.slot * kTT;
      auto fw = [&](int s) {  // lane 0
        const uint32_t q = sq + s;
        uint64_t* bar = &b_fw[q % SF];
        uint32_t tx = 64 * sizeof(T);  // static part of edge record s
        if (s + 1 < NS) tx += slice_bytes<T>(s + 1, nz, 1);
        if (s == 0) tx += slice_bytes<T>(0, nz, 1);
        mbar_expect_tx(bar, tx);
        bulk_g2s(s_edge + (q & (ER - 1)) * NE, P.rec_phi + (td.slot + s) * 64, 64 * sizeof(T), bar);
        if (s + 1 < NS)
          issue_slice<T>(s_ph + ((q + 1) % SP) * kTT, ph_src + (long long)(s + 1) * kTT, 1, s + 1,
                         nz, bar, false, 0);
        if (s == 0) issue_slice<T>(s_ph + (q % SP) * kTT, ph_src, 1, 0, nz, bar, false, 0);
      };
      int f = 0;  // next transaction to issue (lane 0)
      if (lane == 0)
        for (; f < NS && f < SF; ++f) fw(f);
      int t = 0;
      while (t < NS) {
        {
          const uint32_t q = eq + t + 1;  // E[t+1]: step t complete
          mbar_wait(&b_step[q % EB], (q / EB) & 1, 43);
        }
        int t_end = t + 1;
        while (t_end < NS) {
          const uint32_t q = eq + t_end + 1;
          if (!warp_test(&b_step[q % EB], (q / EB) & 1)) break;
          ++t_end;
        }
        if (lane == 0)  // E[t_end] seen: prep(0 .. t_end) done
          for (; f < NS && f < t_end + 1 + SF; ++f) fw(f);
        const int t_pub = t;
        (void)t_pub;
        for (; t < t_end; ++t) {
          const int k = t - outoff;
          if (outok && k >= 0 && k < nz)
            put_tagged(outdst + (long long)k * 16 * kTagWords<T>, s_out[(t % OR) * 32 + lane],
                       edge_tag(epoch, k));
          // keep the forward pack warm in L2 kPFL steps ahead of the compute LDGs
          const int xs = t + 1 + kPFL;
          if (xs < NS && lane == 0) prefetch_l2(fw_pf + (long long)xs * F_NA * kTT, F_NA * kTT * sizeof(T));
        }
        __syncwarp();
        if (lane == 0) {
          if (kStepTrace && P.trace && tid == P.trace_tile)  // step-trace slot 2: tile A published steps < t
            for (int u = t_pub; u < t; ++u) P.trace[8 * P.ntiles + 16 * u + 2] = gtime();
          st_release_cta_s(&s_linked, t);
        }
      }
    } else if (warp == kFetcherWarp) {
      // ----------------------------------------------------------- fetcher
      // lanes 0-15 poll R of the W neighbour's E column (index = tj), lanes
      // 16-31 R of the S neighbour's N row (index = ti); the static phi part
      // of each record comes with the step's bulk copy (k_edge_phi)
      const bool we = lane < 16;
      const int c = lane & 15;
      const bool colok = we ? (c < td.wJ) : (c < td.wI);
      const int nA = we ? td.nW : td.nS;  // upstream neighbour
      const bool live = nA >= 0 && colok;  // lanes with a value to poll (others: R = 0)
      const long long edgeA = nA >= 0 ? P.tiles[nA].edge : 0;
      const unsigned long long* eA = (we ? P.tagA : P.tagB) + (edgeA + c) * kTagWords<T>;
      // Step s's slot barrier b_fw[s % SF] completes when (1) phi slice s+1
      // (+ slice 0 for s = 0) and the static part of record s have landed
      // (armed and copied by the publisher) and (2) the R part of record s
      // is announced here, which also waits for the publisher (compute step
      // s writes out-record s % OR).  e: next record to fetch into deep-ring
      // slot e % ER (reusable once prep(e - ER + 1) is done).
      int e = 0, a = 0, freed = 0;
      Watchdog wd;
      constexpr int kB = 8;  // records polled per round trip
      while (a < NS) {
        while (freed < NS) {  // prep(freed) done? (compute cannot pass the records: bounded)
          const uint32_t q = eq + freed;
          if (!warp_test(&b_step[q % EB], (q / EB) & 1)) break;
          ++freed;
        }
        {
          const int a_end = __shfl_sync(0xffffffffu,
                                        min(min(e, freed + SF), ld_relaxed_cta_s(&s_linked) + OR), 0);
          if (a_end > a) {
            fence_cta();  // acquire the publisher's progress / order the record stores
            __syncwarp();
            if (lane == 0)
              for (int s2 = a; s2 < a_end; ++s2) {
                if (kStepTrace && P.trace && tid == P.trace_tile + 1) P.trace[8 * P.ntiles + 16 * s2 + 4] = gtime();
                mbar_arrive(&b_fw[(sq + s2) % SF]);
              }
            a = a_end;
          }
        }
        const int m = min(NS - 1, freed + ER - 2);
        if (e > m) {
          wd.idle(45);
          continue;
        }
        // issue the loads of up to kB records at once, then accept the valid prefix
        T rA[kB];
        bool ok[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) {
          const int s2 = e + j;
          const int kA = s2 - c;  // W side cell (0, c) / S side cell (c, 0)
          rA[j] = T(0);
          ok[j] = true;
          if (live && s2 <= m && kA >= 0 && kA < nz)
            ok[j] = get_tagged(eA + (long long)kA * 16 * kTagWords<T>, edge_tag(epoch, kA), rA[j]);
        }
        int n = 0;
#pragma unroll
        for (int j = 0; j < kB; ++j) {
          if (n == j && e + j <= m && __all_sync(0xffffffffu, ok[j])) {
            s_edge[((sq + e + j) % ER) * NE + (we ? 64 : 80) + c] = rA[j];
            n = j + 1;
          }
        }
        if (n == 0) {
          wd.idle(44);
          continue;
        }
        wd.progress();
        if (kStepTrace && P.trace && tid == P.trace_tile + 1 && lane == 0)  // slot 3: tile B fetched records
          for (int u = e; u < e + n; ++u) P.trace[8 * P.ntiles + 16 * u + 3] = gtime();
        e += n;
      }
    } else if (warp < kComputeWarps) {
      // --------------------------------------------------------- compute warps
      // Iteration t: the shared loads of critical(t) and of the residual of
      // step t+1 are issued first (branch-free, always-valid addresses), then
      // both FP chains, so the residual fills the latency of the recurrence;
      // then one step-done arrival, one wait for the data of step t+2 and one
      // named barrier.  All ring positions are 32-bit shared addresses.
      constexpr uint32_t SZ = sizeof(T);
      constexpr uint32_t SLICE = kTT * SZ;
      const bool col = ti < td.wI && tj < td.wJ;
      const bool inW = ti > 0, inE = ti + 1 < td.wI, inS = tj > 0, inN = tj + 1 < td.wJ;
      const uint32_t aPh = saddr(smem);
      const uint32_t aR = aPh + SP * SLICE;
      const uint32_t aEdge = aR + 2 * SLICE;
      const uint32_t aOut = aEdge + ER * NE * SZ;
      const uint32_t aGh = aOut + OR * 32 * SZ;
      const uint32_t aFw = saddr(b_fw), aStep = saddr(b_step);
      const uint32_t oP = p * SZ;
      {
        const int gi = td.i0 + ti, gj = td.j0 + tj;
        T gb = T(0), gt = T(0);
        if (col) {
          gb = P.ghost[ghost_face_offset(bd, G_B) + gi + (long long)bd.nx * gj];
          gt = P.ghost[ghost_face_offset(bd, G_T) + gi + (long long)bd.nx * gj];
        }
        sts(aGh + oP, gb);  // own slots: read back by this thread only
        sts(aGh + SLICE + oP, gt);
      }
      // neighbour operands: in-tile (offset into a phi slot / R buffer) or
      // from the edge record (phiW, phiE, phiS, phiN, RW, RS; 16 each)
      const uint32_t offW = (inW ? pW : tj) * SZ, offE = (inE ? pE : 16 + tj) * SZ;
      const uint32_t offS = (inS ? pS : 32 + ti) * SZ, offN = (inN ? pN : 48 + ti) * SZ;
      const uint32_t offRW = (inW ? pW : 64 + tj) * SZ, offRS = (inS ? pS : 80 + ti) * SZ;
      const uint32_t oOutE = (ti == kTI - 1) ? tj * SZ : 0xFFFFFFFFu;
      const uint32_t oOutN = (tj == kTJ - 1) ? (16 + ti) * SZ : 0xFFFFFFFFu;
      uint32_t ph0 = aPh + (sq % SP) * SLICE;  // slot of phi slice x while preparing step x
      uint32_t rec = aEdge + (sq & (ER - 1)) * NE * SZ;  // edge record of step x
      uint32_t fwb = aFw + (sq % SF) * 8;
      uint32_t fpar = (sq / SF) & 1;
      uint32_t eb = aStep + (eq % EB) * 8;
      uint32_t ob = aOut;  // out-record slot of step t (t % OR)
      T RB = T(0);         // own R of the plane below (0 outside the block)
      T r = T(0), lb = T(0), lw = T(0), ls = T(0), lp = T(0);  // prepared step
      T nf[F_NA];  // forward-pack values of the next step to prepare (LDG one step ahead)
#pragma unroll
      for (int a2 = 0; a2 < F_NA; ++a2) nf[a2] = T(0);
      const T* fw_cell = P.fw + td.slot * F_NA * kTT + p;
      auto ldg_next = [&](int xs) {
        const int k2 = xs - d;
        if (xs < NS && col && k2 >= 0 && k2 < nz) {
          const T* src = fw_cell + (long long)xs * F_NA * kTT;
#ifdef SIPB_EXP_NOLDG
#pragma unroll
          for (int a2 = 0; a2 < F_NA; ++a2) nf[a2] = T(0.01) * T(a2 + 1) + T(xs) * T(1e-9);
          (void)src;
#else
#pragma unroll
          for (int a2 = 0; a2 < F_NA; ++a2) nf[a2] = __ldg(src + a2 * kTT);
#endif
        }
      };
      // residual of step x (Listing-1 term order, a_nb = -A_nb)
      auto residual = [&](T fP, T fB, T fT, T fW, T fE, T fS, T fN) {
        T rr = -(nf[F_AE] * fE);
        rr -= nf[F_AW] * fW;
        rr -= nf[F_AN] * fN;
        rr -= nf[F_AS] * fS;
        rr -= nf[F_AT] * fT;
        rr -= nf[F_AB] * fB;
        rr += nf[F_Q];
        rr -= nf[F_AP] * fP;
        return rr;
      };
      T* gR = P.R + td.slot * kTT + p;
      // ---- step 0 preparation (only the (0,0) column is active at k = 0)
      ldg_next(0);
      mbar_wait_a(fwb, fpar, 21);
      bool act = col && d == 0 && nz > 0;
      {
        const uint32_t php = ring_next(ph0, aPh, SLICE, SP * SLICE);
        const T fP = lds<T>(ph0 + oP);
        const T fB = lds<T>(aGh + oP);
        const T fT = lds<T>((nz > 1 ? php : aGh + SLICE) + oP);
        const T fW = lds<T>(rec + offW), fE = lds<T>((inE ? php : rec) + offE);
        const T fS = lds<T>(rec + offS), fN = lds<T>((inN ? php : rec) + offN);
        const T rr = residual(fP, fB, fT, fW, fE, fS, fN);
        if (act) {
          nrm += fabs(static_cast<double>(rr));
          r = rr; lb = nf[F_LB]; lw = nf[F_LW]; ls = nf[F_LS]; lp = nf[F_LP];
        }
      }
      ldg_next(1);
      __syncwarp();
      if (lane == 0) mbar_arrive_a(eb);
      eb = ring_next(eb, aStep, 8, EB * 8);
      fwb = ring_next(fwb, aFw, 8, SF * 8);
      fpar ^= (fwb == aFw);
      ph0 = ring_next(ph0, aPh, SLICE, SP * SLICE);
      if (1 < NS) mbar_wait_a(fwb, fpar, 22);
      for (int t = 0; t < NS; ++t) {
        const int x = t + 1;
        // ---- shared loads of critical(t)
        const uint32_t sRm = aR + ((t - 1) & 1) * SLICE;
        const T RW = lds<T>((inW ? sRm : rec) + offRW);
        const T RS = lds<T>((inS ? sRm : rec) + offRS);
        // ---- shared loads of the residual of step x: slices x-1, x, x+1, record x
        const uint32_t recx = ring_next(rec, aEdge, NE * SZ, ER * NE * SZ);
        const uint32_t php = ring_next(ph0, aPh, SLICE, SP * SLICE);
        const uint32_t phm = ph0 == aPh ? ph0 + (SP - 1) * SLICE : ph0 - SLICE;
        const int k1 = x - d;
        const T fP = lds<T>(ph0 + oP);
        const T fB = lds<T>((k1 > 0 ? phm : aGh) + oP);
        const T fT = lds<T>((k1 + 1 < nz ? php : aGh + SLICE) + oP);
        const T fW = lds<T>((inW ? phm : recx) + offW);
        const T fE = lds<T>((inE ? php : recx) + offE);
        const T fS = lds<T>((inS ? phm : recx) + offS);
        const T fN = lds<T>((inN ? php : recx) + offN);
        // ---- critical(t): R = (((r - LB*R_B) - LW*R_W) - LS*R_S) * LP
        const T Rv = (((r - lb * RB) - lw * RW) - ls * RS) * lp;
        if (act) {
          RB = Rv;
          sts(aR + (t & 1) * SLICE + oP, Rv);
          if (oOutE != 0xFFFFFFFFu) sts(ob + oOutE, Rv);
          if (oOutN != 0xFFFFFFFFu) sts(ob + oOutN, Rv);
#ifndef SIPB_EXP_NOSTG
          gR[(long long)t * kTT] = Rv;  // consumed only by K3 (next launch)
#endif
        }
        // ---- residual of step x
        const bool act1 = x < NS && col && k1 >= 0 && k1 < nz;
        const T rr = residual(fP, fB, fT, fW, fE, fS, fN);
        if (act1) {
          nrm += fabs(static_cast<double>(rr));
          r = rr; lb = nf[F_LB]; lw = nf[F_LW]; ls = nf[F_LS]; lp = nf[F_LP];
        }
        ldg_next(x + 1);  // nf consumed above
        act = act1;
        __syncwarp();
        if (lane == 0) mbar_arrive_a(eb);  // E[x]: step t done, step x prepared
        eb = ring_next(eb, aStep, 8, EB * 8);
        fwb = ring_next(fwb, aFw, 8, SF * 8);
        fpar ^= (fwb == aFw);
        ph0 = php;
        rec = recx;
        ob = ring_next(ob, aOut, 32 * SZ, OR * 32 * SZ);
        if (x + 1 < NS) mbar_wait_a(fwb, fpar, 21);  // data of step x+1
        if (kStepTrace && P.trace && p == 0 && (tid == P.trace_tile || tid == P.trace_tile + 1))
          P.trace[8 * P.ntiles + 16 * t + (tid - P.trace_tile)] = gtime();  // slots 0, 1: tiles A, B
        bar_compute();
      }
    }
    sq += NS;
    eq += NS + 1;
    __syncthreads();  // publisher has published NS (all steps retired)
    if (P.trace && p == 0) P.trace[4 * tid + 1] = gtime();
    const double s = cta_sum(nrm, s_red);
    if (p == 0) {
      P.partial[tid] = s;
      __threadfence();
      s_last = (atomicAdd(P.state + 1, 1u) == (unsigned)P.ntiles - 1);
    }
    __syncthreads();
    if (s_last) {
      // finaliser: deterministic per-block norms, then reset the backward state
      __threadfence();
      const int nw = blockDim.x >> 5;
      for (int b = warp; b < P.nblocks; b += nw) {
        const BlockDesc bb = P.blocks[b];
        double v = 0.0;
        for (int x = lane; x < bb.ntiles; x += 32) v += __ldcg(P.partial + bb.tile0 + x);
#pragma unroll
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if (lane == 0) P.block_norms[b] = v;
      }
      __syncthreads();
      if (p == 0) {
        double v = 0.0;
        for (int b = 0; b < P.nblocks; ++b) v += P.block_norms[b];
        *P.norm = v;
      }
      for (int x = p; x < kProgOff + P.ntiles; x += blockDim.x) P.state_other[x] = 0u;
      if (p == 0) *P.epoch = epoch + 1;
    }
  }
}

// =============================================================================
// K3: backward substitution + phi update (backward3d); slices in reverse.
// Ring slot = {R, phi, UN, UE, UT} of one slice; edge record = delta of the
// E and N neighbour tiles (16 each).  Same warp roles and step pipeline as K2:
// prep(x) loads the slot into registers and forms UT*dT; the critical step is
// ((R - UN*dN) - UE*dE) - UT*dT after the barrier.
// =============================================================================
template <typename T, int SB>
struct BwdCfg {
  static constexpr int ER = 16, NE = 32, OR = 8, EB = 32;
  // R, phi, UN, UE, UT are own-cell data: LDG'd by each compute thread one
  // step ahead; shared memory holds only the delta exchange and edge records
  static constexpr size_t bytes = (size_t)2 * kTT * sizeof(T) +
                                  (size_t)(ER * NE + OR * 32) * sizeof(T) +
                                  (SB + EB) * sizeof(uint64_t);
};

template <typename T, int SB>
__global__ void __launch_bounds__(kThreads, 2) k_backward(const SweepParams<T> P) {
  using C = BwdCfg<T, SB>;
  constexpr int ER = C::ER, EB = C::EB, NE = C::NE, OR = C::OR;
  static_assert(EB > ER + SB && EB > OR + SB + 1, "barrier rings must cover the run-ahead");
  extern __shared__ __align__(128) unsigned char smem[];
  T* s_D = reinterpret_cast<T*>(smem);
  T* s_edge = s_D + 2 * kTT;
  T* s_out = s_edge + ER * NE;  // [OR][32]: delta of the W column (tj) and S row (16 + ti)
  // b_rg[u % SB] completes when slot u has landed AND edge record u is written
  uint64_t* b_rg = reinterpret_cast<uint64_t*>(s_out + OR * 32);
  uint64_t* b_step = b_rg + SB;  // E[x] as in K2
  __shared__ int s_tile, s_last, s_linked;

  const int p = threadIdx.x;
  const int warp = p >> 5, lane = p & 31;
  int ti = 0, tj = 0;
  if (warp < kComputeWarps) pos_to_tij(p, ti, tj);
  const int d = ti + tj;
  const int pE = ti < kTI - 1 ? tile_pos(ti + 1, tj) : 0;
  const int pN = tj < kTJ - 1 ? tile_pos(ti, tj + 1) : 0;
  unsigned* const prog = P.state + kProgOff;

  if (p == 0) {
    for (int b = 0; b < SB; ++b) mbar_init(&b_rg[b], 1);  // loader: edge record announced
    for (int b = 0; b < EB; ++b) mbar_init(&b_step[b], kCompute / 32);
    fence_mbar_init();
  }
  uint32_t sq = 0, eq = 0;
  const unsigned epoch = *P.epoch;

  for (;;) {
    __syncthreads();
    if (p == 0) {
      s_tile = atomicAdd(P.state, 1u);
      s_linked = 0;
    }
    __syncthreads();
    const int tk = s_tile;
    if (tk >= P.ntiles) break;
    const int tid = P.order[tk];
    const TileDesc td = P.tiles[tid];
    const int NS = td.ns, nz = td.nz;
    if (P.trace && p == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      P.trace[4 * tid + 0] = gtime();
      P.trace[4 * tid + 2] = smid;
      P.trace[4 * tid + 3] = blockIdx.x;
    }

    // no loader: compute threads LDG their own cells, the fetcher announces
    // edge records, the publisher keeps the slices warm in L2
    if (warp == kPublisherWarp) {
      // outgoing edge: lane c < 16 -> W column cell (0, c), lane >= 16 -> S row cell (c, 0)
      const bool we = lane < 16;
      const int c = lane & 15;
      const bool outok = we ? (td.nW >= 0 && c < td.wJ) : (td.nS >= 0 && c < td.wI);
      unsigned long long* outdst = (we ? P.tagA : P.tagB) + (td.edge + c) * kTagWords<T>;
      // keeps the slices kPFL steps ahead of the compute LDGs warm in L2 (the
      // publisher gates the compute warps through s_linked, so it cannot fall
      // a full E ring behind)
      constexpr int kL1 = kTT * (int)sizeof(T) / 128;  // lines per array slice
      const char* rb = reinterpret_cast<const char*>(P.R + td.slot * kTT);
      const char* pb = reinterpret_cast<const char*>(P.phi + td.slot * kTT);
      const char* ub = reinterpret_cast<const char*>(P.bw + td.slot * B_NA * kTT);
      auto pf = [&](int xs) {
        if (xs >= NS) return;
        const int ts = NS - 1 - xs;
        for (int l = lane; l < 5 * kL1; l += 32) {
          const char* a = l < kL1       ? rb + (long long)ts * kTT * sizeof(T) + 128 * l
                          : l < 2 * kL1 ? pb + (long long)ts * kTT * sizeof(T) + 128 * (l - kL1)
                                        : ub + (long long)ts * B_NA * kTT * sizeof(T) + 128 * (l - 2 * kL1);
          prefetch_line_l2(a);
        }
      };
      for (int xs = 0; xs <= kPFL; ++xs) pf(xs);
      int u = 0;
      while (u < NS) {
        {
          const uint32_t q = eq + u + 1;
          mbar_wait(&b_step[q % EB], (q / EB) & 1, 53);
        }
        int u_end = u + 1;
        while (u_end < NS) {
          const uint32_t q = eq + u_end + 1;
          if (!warp_test(&b_step[q % EB], (q / EB) & 1)) break;
          ++u_end;
        }
        for (; u < u_end; ++u) {
          const int k = (NS - 1 - u) - c;
          if (outok && k >= 0 && k < nz)
            put_tagged(outdst + (long long)k * 16 * kTagWords<T>, s_out[(u % OR) * 32 + lane],
                       edge_tag(epoch, k));
          pf(u + 1 + kPFL);
        }
        __syncwarp();
        if (lane == 0) st_release_cta_s(&s_linked, u);
      }
    } else if (warp == kFetcherWarp) {
      const bool we = lane < 16;
      const int c = lane & 15;
      const bool colok = we ? (c < td.wJ) : (c < td.wI);
      const int nB = we ? td.nE : td.nN;
      const long long edgeB = nB >= 0 ? P.tiles[nB].edge : 0;
      const unsigned long long* srcB = (we ? P.tagA : P.tagB) + (edgeB + c) * kTagWords<T>;
      const int offB = we ? (kTI - 1) + c : c + (kTJ - 1);  // edge cell (TI-1, c) / (c, TJ-1)
      // Poll tagged deltas into the deep ring (record s -> slot s % ER, reusable
      // once prep(s - ER + 1) is done) and announce record s on b_rg[s % SB]
      // once its previous phase is over (prep(s - SB) done).
      int e = 0, a = 0, freed = 0;
      Watchdog wd;
      constexpr int kB = 4;
      while (a < NS) {
        while (freed < NS) {
          const uint32_t q = eq + freed;
          if (!warp_test(&b_step[q % EB], (q / EB) & 1)) break;
          ++freed;
        }
        // compute step s writes out-record slot s % OR: the publisher must be past s - OR
        const int a_end = min(min(e, freed + SB), ld_relaxed_cta_s(&s_linked) + OR);
        if (a_end > a) {
          fence_cta();  // acquire the publisher's progress / order the record stores
          __syncwarp();
          if (lane == 0)
            for (int s2 = a; s2 < a_end; ++s2) mbar_arrive(&b_rg[(sq + s2) % SB]);
          a = a_end;
        }
        const int m = min(NS - 1, freed + ER - 2);
        if (e > m) {
          wd.idle(55);
          continue;
        }
        T v[kB];
        bool ok[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) {
          const int s2 = e + j;
          v[j] = T(0);
          ok[j] = true;
          if (s2 > m) continue;
          const int k = (NS - 1 - s2) - offB;
          if (nB >= 0 && colok && k >= 0 && k < nz)
            ok[j] = get_tagged(srcB + (long long)k * 16 * kTagWords<T>, edge_tag(epoch, k), v[j]);
        }
        int n = 0;
#pragma unroll
        for (int j = 0; j < kB; ++j) {
          if (n == j && e + j <= m && __all_sync(0xffffffffu, ok[j])) {
            s_edge[((sq + e + j) % ER) * NE + (we ? 0 : 16) + c] = v[j];
            n = j + 1;
          }
        }
        if (n == 0) {
          wd.idle(54);
          continue;
        }
        wd.progress();
        e += n;
      }
    } else if (warp < kComputeWarps) {
      const bool col = ti < td.wI && tj < td.wJ;
      const bool inE = ti + 1 < td.wI, inN = tj + 1 < td.wJ;
      T dT = T(0);
      T rr = T(0), ph = T(0), un = T(0), ue = T(0), utdt = T(0), dnx = T(0), dex = T(0);
      bool act = false;
      int kk = 0;
      const T* r_cell = P.R + td.slot * kTT + p;
      const T* ph_cell = P.phi + td.slot * kTT + p;
      const T* bw_cell = P.bw + td.slot * B_NA * kTT + p;
      T nb[5] = {T(0), T(0), T(0), T(0), T(0)};  // R, phi, UN, UE, UT of the next step
      auto ldg_next = [&](int xs) {
        const int ts = NS - 1 - xs, k2 = ts - d;
        if (xs < NS && col && k2 >= 0 && k2 < nz) {
#ifdef SIPB_EXP_NOLDG
          nb[0] = T(ts) * T(1e-9); nb[1] = T(0.5); nb[2] = T(0.1); nb[3] = T(0.2); nb[4] = T(0.3);
#else
          nb[0] = __ldg(r_cell + (long long)ts * kTT);
          nb[1] = __ldg(ph_cell + (long long)ts * kTT);
          const T* u = bw_cell + (long long)ts * B_NA * kTT;
          nb[2] = __ldg(u);
          nb[3] = __ldg(u + kTT);
          nb[4] = __ldg(u + 2 * kTT);
#endif
        }
      };
      auto prep = [&](int x) {
        const uint32_t q = sq + x;
        mbar_wait(&b_rg[q % SB], (q / SB) & 1, 31);  // edge record x announced
        const int t = NS - 1 - x;
        kk = t - d;
        act = col && kk >= 0 && kk < nz;
        if (act) {
          const T* rec = s_edge + (q % ER) * NE;
          rr = nb[0];
          ph = nb[1];
          un = nb[2];
          ue = nb[3];
          utdt = nb[4] * dT;
          dnx = rec[16 + ti];
          dex = rec[tj];
        }
        ldg_next(x + 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&b_step[(eq + x) % EB]);
      };
      ldg_next(0);
      prep(0);
      for (int u = 0; u < NS; ++u) {
        const int t = NS - 1 - u;
        const bool was = act;
        T phn = T(0);
        if (act) {
          const T dN = inN ? s_D[((u - 1) & 1) * kTT + pN] : dnx;
          const T dE = inE ? s_D[((u - 1) & 1) * kTT + pE] : dex;
          const T dl = ((rr - un * dN) - ue * dE) - utdt;
          dT = dl;
          phn = ph + dl;
          s_D[(u & 1) * kTT + p] = dl;
          if (ti == 0) s_out[(u % OR) * 32 + tj] = dl;
          if (tj == 0) s_out[(u % OR) * 32 + 16 + ti] = dl;
        }
        if (u + 1 < NS) {
          prep(u + 1);  // arrives E[u+1]
        } else {
          __syncwarp();
          if (lane == 0) mbar_arrive(&b_step[(eq + NS) % EB]);
        }
#ifndef SIPB_EXP_NOSTG
        if (was) P.phi[(td.slot + t) * kTT + p] = phn;
#endif
        bar_compute();
      }
    }
    sq += NS;
    eq += NS + 1;
    __syncthreads();
    if (P.trace && p == 0) P.trace[4 * tid + 1] = gtime();
    if (p == 0) {
      __threadfence();
      s_last = (atomicAdd(P.state + 1, 1u) == (unsigned)P.ntiles - 1);
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      for (int x = p; x < kProgOff + P.ntiles; x += blockDim.x) P.state_other[x] = 0u;
      if (p == 0) *P.epoch = epoch + 1;
    }
  }
}

// =============================================================================
// Static part of the K2 edge records: for every tile and step s, the old phi
// of the W / E / S / N neighbour cells the step reads (a neighbour tile's
// packed phi, or the block's ghost faces); [slot + s][64] in the shared
// record layout.  Runs after each halo exchange, before K2, so the forward
// sweep's fetcher only polls the R values that are produced during the sweep.
// =============================================================================
template <typename T>
__global__ void __launch_bounds__(256) k_edge_phi(const SweepParams<T> P) {
  const TileDesc td = P.tiles[blockIdx.x];
  const BlockDesc bd = P.blocks[td.block];
  const int NS = td.ns, nz = td.nz;
  const int q = threadIdx.x & 63;
  const bool we = q < 32, sideB = (q & 16) != 0;  // W, E, S, N = 16 each
  const int c = q & 15;
  const bool colok = we ? (c < td.wJ) : (c < td.wI);
  const int nbr = sideB ? (we ? td.nE : td.nN) : (we ? td.nW : td.nS);
  const long long slotN = nbr >= 0 ? P.tiles[nbr].slot : 0;
  const int lag = we ? kTI : kTJ;
  // neighbour cell (upstream: its E column / N row; downstream: its W column / S row)
  const int posN = sideB ? (we ? tile_pos(0, c) : tile_pos(c, 0))
                         : (we ? tile_pos(kTI - 1, c) : tile_pos(c, kTJ - 1));
  const int koff = sideB ? (we ? (td.wI - 1) + c : c + (td.wJ - 1)) : c;  // cell k = s - koff
  const long long sdelta = sideB ? -(lag - 1) : (lag - 1);                // neighbour slice = s + sdelta
  const T* g = P.ghost + ghost_face_offset(bd, sideB ? (we ? G_E : G_N) : (we ? G_W : G_S)) +
               (we ? td.j0 : td.i0) + c;
  const long long gstride = we ? bd.ny : bd.nx;
  for (int s = threadIdx.x >> 6; s < NS; s += blockDim.x >> 6) {
    const int k = s - koff;
    T v = T(0);
    if (colok && k >= 0 && k < nz)
      v = nbr >= 0 ? P.phi[(slotN + s + sdelta) * kTT + posN] : g[gstride * k];
    P.rec_phi[((long long)td.slot + s) * 64 + q] = v;
  }
}

// =============================================================================
// Layout / halo / utility kernels
// =============================================================================
__device__ __forceinline__ long long f3(int nx, int ny, int i, int j, int k) {
  return (long long)i + (long long)(nx + 2) * ((long long)j + (long long)(ny + 2) * k);
}

template <typename T>
__global__ void k_scatter(const double* __restrict__ src, const BlockDesc* blocks, int b, T* pack,
                          int na, int arr) {
  const BlockDesc bd = blocks[b];
  const long long n = (long long)bd.nx * bd.ny * bd.nz;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(c % bd.nx);
    const long long r = c / bd.nx;
    const int j = (int)(r % bd.ny), k = (int)(r / bd.ny);
    pack[pack_index(bd, na, arr, i, j, k)] = static_cast<T>(src[f3(bd.nx, bd.ny, i + 1, j + 1, k + 1)]);
  }
}

// plane coordinate (x0 fast, x1 slow) of face f -> 1-based Field3 cell
__device__ __forceinline__ void face_cell(const BlockDesc& bd, int f, int x0, int x1, bool ghost,
                                          int& i, int& j, int& k) {
  switch (f) {
    case G_W: i = ghost ? 0 : 1; j = x0 + 1; k = x1 + 1; break;
    case G_E: i = ghost ? bd.nx + 1 : bd.nx; j = x0 + 1; k = x1 + 1; break;
    case G_S: i = x0 + 1; j = ghost ? 0 : 1; k = x1 + 1; break;
    case G_N: i = x0 + 1; j = ghost ? bd.ny + 1 : bd.ny; k = x1 + 1; break;
    case G_B: i = x0 + 1; j = x1 + 1; k = ghost ? 0 : 1; break;
    default: i = x0 + 1; j = x1 + 1; k = ghost ? bd.nz + 1 : bd.nz; break;
  }
}
__device__ __forceinline__ void face_dims(const BlockDesc& bd, int f, int& n0, int& n1) {
  if (f <= G_E) { n0 = bd.ny; n1 = bd.nz; }
  else if (f <= G_N) { n0 = bd.nx; n1 = bd.nz; }
  else { n0 = bd.nx; n1 = bd.ny; }
}

template <typename T>
__global__ void k_ghost_in(const double* __restrict__ src, const BlockDesc* blocks, int b, T* ghost) {
  const BlockDesc bd = blocks[b];
  const int f = blockIdx.y;
  int n0, n1;
  face_dims(bd, f, n0, n1);
  const long long n = (long long)n0 * n1;
  T* g = ghost + ghost_face_offset(bd, f);
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    int i, j, k;
    face_cell(bd, f, (int)(c % n0), (int)(c / n0), true, i, j, k);
    g[c] = static_cast<T>(src[f3(bd.nx, bd.ny, i, j, k)]);
  }
}

template <typename T>
__global__ void k_gather(const T* __restrict__ pack, const T* __restrict__ ghost,
                         const BlockDesc* blocks, int b, int nbrmask, double* dst) {
  const BlockDesc bd = blocks[b];
  const long long n = (long long)bd.nx * bd.ny * bd.nz;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(c % bd.nx);
    const long long r = c / bd.nx;
    const int j = (int)(r % bd.ny), k = (int)(r / bd.ny);
    dst[f3(bd.nx, bd.ny, i + 1, j + 1, k + 1)] = static_cast<double>(pack[pack_index(bd, 1, 0, i, j, k)]);
  }
  // interface ghosts (faces with a neighbour block): values of the last exchange
  for (int f = 0; f < 6; ++f) {
    if (!((nbrmask >> f) & 1)) continue;
    int n0, n1;
    face_dims(bd, f, n0, n1);
    const long long m = (long long)n0 * n1;
    const T* g = ghost + ghost_face_offset(bd, f);
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < m;
         c += (long long)gridDim.x * blockDim.x) {
      int i, j, k;
      face_cell(bd, f, (int)(c % n0), (int)(c / n0), true, i, j, k);
      dst[f3(bd.nx, bd.ny, i, j, k)] = static_cast<double>(g[c]);
    }
  }
}

template <typename T>
__global__ void k_gather_any(const T* __restrict__ pack, int na, int arr, const BlockDesc* blocks,
                             int b, double* dst) {
  const BlockDesc bd = blocks[b];
  const long long n = (long long)bd.nx * bd.ny * bd.nz;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(c % bd.nx);
    const long long r = c / bd.nx;
    const int j = (int)(r % bd.ny), k = (int)(r / bd.ny);
    dst[f3(bd.nx, bd.ny, i + 1, j + 1, k + 1)] = static_cast<double>(pack[pack_index(bd, na, arr, i, j, k)]);
  }
}

// K4: face copies.  grid.y = copy index.  Source: interior plane `src_face`
// of local block src_block (phi pack) or buf_in; destination: ghost face
// dst_face of local block dst_block or buf_out.
template <typename T>
__global__ void k_face_copy(const FaceCopy* copies, const BlockDesc* blocks, const T* __restrict__ phi,
                            T* ghost, const T* buf_in, T* buf_out) {
  const FaceCopy fc = copies[blockIdx.y];
  const long long n = (long long)fc.n0 * fc.n1;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    const int x0 = (int)(c % fc.n0), x1 = (int)(c / fc.n0);
    T v;
    if (fc.src_block >= 0) {
      const BlockDesc sb = blocks[fc.src_block];
      int i, j, k;
      face_cell(sb, fc.src_face, x0, x1, false, i, j, k);
      v = phi[pack_index(sb, 1, 0, i - 1, j - 1, k - 1)];
    } else {
      v = buf_in[fc.buf + c];
    }
    if (fc.dst_block >= 0) {
      const BlockDesc db = blocks[fc.dst_block];
      ghost[ghost_face_offset(db, fc.dst_face) + c] = v;
    } else {
      buf_out[fc.buf + c] = v;
    }
  }
}

// residual_general of the device phi, Field3 fp64 output
template <typename T>
__global__ void k_residual(const BlockDesc* blocks, int b, const T* __restrict__ fw,
                           const T* __restrict__ phi, const T* __restrict__ ghost, double* out) {
  const BlockDesc bd = blocks[b];
  const long long n = (long long)bd.nx * bd.ny * bd.nz;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(c % bd.nx);
    const long long r = c / bd.nx;
    const int j = (int)(r % bd.ny), k = (int)(r / bd.ny);
    auto ph = [&](int ii, int jj, int kk) -> T {
      if (ii < 0) return ghost[ghost_face_offset(bd, G_W) + jj + (long long)bd.ny * kk];
      if (ii >= bd.nx) return ghost[ghost_face_offset(bd, G_E) + jj + (long long)bd.ny * kk];
      if (jj < 0) return ghost[ghost_face_offset(bd, G_S) + ii + (long long)bd.nx * kk];
      if (jj >= bd.ny) return ghost[ghost_face_offset(bd, G_N) + ii + (long long)bd.nx * kk];
      if (kk < 0) return ghost[ghost_face_offset(bd, G_B) + ii + (long long)bd.nx * jj];
      if (kk >= bd.nz) return ghost[ghost_face_offset(bd, G_T) + ii + (long long)bd.nx * jj];
      return phi[pack_index(bd, 1, 0, ii, jj, kk)];
    };
    auto A = [&](int arr) -> T { return fw[pack_index(bd, F_NA, arr, i, j, k)]; };
    T v = -(A(F_AE) * ph(i + 1, j, k));
    v -= A(F_AW) * ph(i - 1, j, k);
    v -= A(F_AN) * ph(i, j + 1, k);
    v -= A(F_AS) * ph(i, j - 1, k);
    v -= A(F_AT) * ph(i, j, k + 1);
    v -= A(F_AB) * ph(i, j, k - 1);
    v += A(F_Q);
    v -= A(F_AP) * ph(i, j, k);
    out[f3(bd.nx, bd.ny, i + 1, j + 1, k + 1)] = static_cast<double>(v);
  }
}

__global__ void k_convert(const double* __restrict__ src, float* __restrict__ dst, long long n) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x)
    dst[c] = static_cast<float>(src[c]);
}

// Synthetic generator; identical arithmetic to
// sip_generate_host (sip_gen.cpp).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double u01(uint64_t seed, uint32_t aid, uint64_t cell) {
  uint64_t h = mix64(seed ^ 0x5851F42D4C957F2DULL);
  h = mix64(h ^ ((uint64_t)(aid + 1) * 0x9E3779B97F4A7C15ULL));
  h = mix64(h ^ cell);
  return (double)(h >> 11) * 0x1.0p-53;
}
struct GenArgs {
  double* out[8];
  int g[3], o[3];
  int nx, ny, nz, kind;
  uint64_t seed;
};
__global__ void k_generate(const GenArgs A) {
  const long long n = (long long)A.nx * A.ny * A.nz;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(c % A.nx);
    const long long r = c / A.nx;
    const int j = (int)(r % A.ny), k = (int)(r / A.ny);
    const long long gi = A.o[0] + i, gj = A.o[1] + j, gk = A.o[2] + k;
    const uint64_t cell = (uint64_t)gi + (uint64_t)A.g[0] * ((uint64_t)gj + (uint64_t)A.g[1] * (uint64_t)gk);
    double aw, ae, as, an, ab, at;
    if (A.kind == 2) {
      const double m = 2.0 * u01(A.seed, 7, cell);
      ae = -1.0; aw = -1.0 - 1.0 * m;
      an = -10.0; as = -10.0 - 0.5 * m;
      at = -100.0; ab = -100.0 - 0.25 * m;
    } else {
      aw = -(1.0 + 0.5 * u01(A.seed, 0, cell));
      ae = -(1.0 + 0.5 * u01(A.seed, 1, cell));
      as = -(1.0 + 0.5 * u01(A.seed, 2, cell));
      an = -(1.0 + 0.5 * u01(A.seed, 3, cell));
      ab = -(1.0 + 0.5 * u01(A.seed, 4, cell));
      at = -(1.0 + 0.5 * u01(A.seed, 5, cell));
    }
    if (gi == 0) aw = 0.0;
    if (gi == A.g[0] - 1) ae = 0.0;
    if (gj == 0) as = 0.0;
    if (gj == A.g[1] - 1) an = 0.0;
    if (gk == 0) ab = 0.0;
    if (gk == A.g[2] - 1) at = 0.0;
    const double s = fabs(aw) + fabs(ae) + fabs(as) + fabs(an) + fabs(ab) + fabs(at);
    const long long x = f3(A.nx, A.ny, i + 1, j + 1, k + 1);
    A.out[0][x] = (A.kind == 2) ? s + 1e-3 : 1.01 * s;
    A.out[1][x] = aw; A.out[2][x] = ae; A.out[3][x] = as;
    A.out[4][x] = an; A.out[5][x] = ab; A.out[6][x] = at;
    A.out[7][x] = 2.0 * u01(A.seed, 6, cell) - 1.0;
  }
}

// ------------------------------------------------------------------ launchers
static int grid_for(long long n, int threads = 256) {
  long long g = (n + threads - 1) / threads;
  if (g > 148LL * 16) g = 148LL * 16;
  if (g < 1) g = 1;
  return (int)g;
}
static inline int cuda_status(cudaError_t e) { return e == cudaSuccess ? SIP_OK : SIP_ERR_CUDA; }

constexpr int kSF64 = 6, kSF32 = 6;  // forward slot ring depth (phi slices + edge records)
constexpr int kSB64 = 8, kSB32 = 8;  // backward record-announce ring depth

template <typename T> struct Rings;
template <> struct Rings<double> { static constexpr int SF = kSF64, SB = kSB64; };
template <> struct Rings<float> { static constexpr int SF = kSF32, SB = kSB32; };

int launch_factor(const FactorParams& p, int grid, void* stream) {
  k_factor<<<grid, kTT, 0, (cudaStream_t)stream>>>(p);
  return cuda_status(cudaGetLastError());
}

template <typename T>
int launch_forward(const SweepParams<T>& p, int grid, void* stream) {
  constexpr int SF = Rings<T>::SF;
  const size_t smem = FwdCfg<T, SF>::bytes;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_forward<T, SF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_forward<T, SF><<<grid, kThreads, smem, (cudaStream_t)stream>>>(p);
  return cuda_status(cudaGetLastError());
}

template <typename T>
int launch_backward(const SweepParams<T>& p, int grid, void* stream) {
  constexpr int SB = Rings<T>::SB;
  const size_t smem = BwdCfg<T, SB>::bytes;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_backward<T, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_backward<T, SB><<<grid, kThreads, smem, (cudaStream_t)stream>>>(p);
  return cuda_status(cudaGetLastError());
}

template <typename T>
int launch_edge_phi(const SweepParams<T>& p, void* stream) {
  if (p.ntiles <= 0) return SIP_OK;
  k_edge_phi<T><<<p.ntiles, 256, 0, (cudaStream_t)stream>>>(p);
  return cudaGetLastError() == cudaSuccess ? SIP_OK : SIP_ERR_CUDA;
}
template int launch_edge_phi<float>(const SweepParams<float>&, void*);
template int launch_edge_phi<double>(const SweepParams<double>&, void*);

int max_resident_ctas(int kind, int precision, int* grid) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaSuccess;
  if (kind == 0) {
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_factor, kTT, 0);
  } else if (kind == 1) {
    if (precision == SIP_PREC_DOUBLE) {
      constexpr int SF = Rings<double>::SF;
      cudaFuncSetAttribute(k_forward<double, SF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)FwdCfg<double, SF>::bytes);
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_forward<double, SF>, kThreads,
                                                        FwdCfg<double, SF>::bytes);
    } else {
      constexpr int SF = Rings<float>::SF;
      cudaFuncSetAttribute(k_forward<float, SF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)FwdCfg<float, SF>::bytes);
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_forward<float, SF>, kThreads,
                                                        FwdCfg<float, SF>::bytes);
    }
  } else {
    if (precision == SIP_PREC_DOUBLE) {
      constexpr int SB = Rings<double>::SB;
      cudaFuncSetAttribute(k_backward<double, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)BwdCfg<double, SB>::bytes);
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_backward<double, SB>, kThreads,
                                                        BwdCfg<double, SB>::bytes);
    } else {
      constexpr int SB = Rings<float>::SB;
      cudaFuncSetAttribute(k_backward<float, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)BwdCfg<float, SB>::bytes);
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_backward<float, SB>, kThreads,
                                                        BwdCfg<float, SB>::bytes);
    }
  }
  if (e != cudaSuccess || per < 1) return SIP_ERR_CUDA;
  *grid = per * sms;
  return SIP_OK;
}

template <typename T>
int launch_scatter(const double* src, const BlockDesc* d_blocks, int block, const BlockDesc& hb,
                   T* pack, int na, int arr, void* stream) {
  k_scatter<T><<<grid_for((long long)hb.nx * hb.ny * hb.nz), 256, 0, (cudaStream_t)stream>>>(
      src, d_blocks, block, pack, na, arr);
  return cuda_status(cudaGetLastError());
}
template <typename T>
int launch_ghost_in(const double* src, const BlockDesc* d_blocks, int block, const BlockDesc& hb,
                    T* ghost, void* stream) {
  long long m = (long long)hb.nx * hb.ny;
  if ((long long)hb.ny * hb.nz > m) m = (long long)hb.ny * hb.nz;
  if ((long long)hb.nx * hb.nz > m) m = (long long)hb.nx * hb.nz;
  dim3 g(grid_for(m) / 6 + 1, 6);
  k_ghost_in<T><<<g, 256, 0, (cudaStream_t)stream>>>(src, d_blocks, block, ghost);
  return cuda_status(cudaGetLastError());
}
template <typename T>
int launch_gather(const T* pack, const T* ghost, const BlockDesc* d_blocks, int block,
                  const BlockDesc& hb, const int* nbr6, double* dst, void* stream) {
  int mask = 0;
  for (int f = 0; f < 6; ++f)
    if (nbr6[f] >= 0) mask |= 1 << f;
  k_gather<T><<<grid_for((long long)hb.nx * hb.ny * hb.nz), 256, 0, (cudaStream_t)stream>>>(
      pack, ghost, d_blocks, block, mask, dst);
  return cuda_status(cudaGetLastError());
}
template <typename T>
int launch_face_copies(const FaceCopy* d_copies, int ncopies, int max_plane,
                       const BlockDesc* d_blocks, const T* phi, T* ghost, T* buf_in, T* buf_out,
                       void* stream) {
  if (ncopies <= 0) return SIP_OK;
  int gx = (max_plane + 255) / 256;
  if (gx > 64) gx = 64;
  dim3 g(gx, ncopies);
  k_face_copy<T><<<g, 256, 0, (cudaStream_t)stream>>>(d_copies, d_blocks, phi, ghost, buf_in, buf_out);
  return cuda_status(cudaGetLastError());
}
template <typename T>
int launch_residual(const BlockDesc* d_blocks, int block, const BlockDesc& hb, const T* fw,
                    const T* phi, const T* ghost, int symmetric, double* out, void* stream) {
  (void)symmetric;
  k_residual<T><<<grid_for((long long)hb.nx * hb.ny * hb.nz), 256, 0, (cudaStream_t)stream>>>(
      d_blocks, block, fw, phi, ghost, out);
  return cuda_status(cudaGetLastError());
}
template <typename T>
int launch_gather_any(const T* pack, int na, int arr, const BlockDesc* d_blocks, int block,
                      const BlockDesc& hb, double* dst, void* stream) {
  k_gather_any<T><<<grid_for((long long)hb.nx * hb.ny * hb.nz), 256, 0, (cudaStream_t)stream>>>(
      pack, na, arr, d_blocks, block, dst);
  return cuda_status(cudaGetLastError());
}
template int launch_gather_any<double>(const double*, int, int, const BlockDesc*, int,
                                       const BlockDesc&, double*, void*);
template int launch_gather_any<float>(const float*, int, int, const BlockDesc*, int,
                                      const BlockDesc&, double*, void*);

int launch_convert(const double* src, float* dst, long long n, void* stream) {
  k_convert<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(src, dst, n);
  return cuda_status(cudaGetLastError());
}
int launch_generate(int kind, uint64_t seed, const int g[3], const int o[3], int nx, int ny, int nz,
                    double* const* out8, void* stream) {
  GenArgs a;
  for (int x = 0; x < 8; ++x) a.out[x] = out8[x];
  for (int x = 0; x < 3; ++x) { a.g[x] = g[x]; a.o[x] = o[x]; }
  a.nx = nx; a.ny = ny; a.nz = nz; a.kind = kind; a.seed = seed;
  k_generate<<<grid_for((long long)nx * ny * nz), 256, 0, (cudaStream_t)stream>>>(a);
  return cuda_status(cudaGetLastError());
}

#define SIPB_INST(T)                                                                              \
  template int launch_forward<T>(const SweepParams<T>&, int, void*);                              \
  template int launch_backward<T>(const SweepParams<T>&, int, void*);                             \
  template int launch_scatter<T>(const double*, const BlockDesc*, int, const BlockDesc&, T*, int, \
                                 int, void*);                                                     \
  template int launch_ghost_in<T>(const double*, const BlockDesc*, int, const BlockDesc&, T*,     \
                                  void*);                                                         \
  template int launch_gather<T>(const T*, const T*, const BlockDesc*, int, const BlockDesc&,      \
                                const int*, double*, void*);                                      \
  template int launch_face_copies<T>(const FaceCopy*, int, int, const BlockDesc*, const T*, T*,   \
                                     T*, T*, void*);                                              \
  template int launch_residual<T>(const BlockDesc*, int, const BlockDesc&, const T*, const T*,    \
                                  const T*, int, double*, void*);
SIPB_INST(double)
SIPB_INST(float)

}  // namespace sipb
