// sip_kernels.cu -- sm_100a kernels of the SIP hot path.
//
//   K1 k_factor    Stone ILU factor          brick wavefront, fp64
//   K2 k_forward   residual + L1 norm + forward substitution   brick wavefront
//                  (resforward3d, SPEC.md:155 + SPEC.md:173)
//   K3 k_backward  backward substitution + phi update          brick wavefront
//                  (backward3d)
//   K4 k_face_copy face-halo copies / pack / unpack (exvec)
//   K7 k_tile_xfer / k_phi_in / k_gather  Field3 <-> brick-slice layout (interior tiled, ghost faces)
//   k_residual     residual_general / residual_symmetric
//
// Wavefront scheme (DESIGN.md sections 4-5): a brick of kW x kL columns is
// swept by ONE recurrence warp; persistent CTAs (one brick at a time) claim
// bricks through an atomic ticket in topological order.  Lane jl owns row
// j0 + jl and walks its cells c = k * kW + il one per step, jl steps behind
// lane 0, so at slice tau = c + jl:
//   * the W neighbour (c - 1) is the lane's own previous step (register),
//   * the S neighbour (lane jl - 1, same c) is one __shfl_up of the previous step,
//   * the B neighbour (c - kW) is the lane's own step tau - kW (register window).
// The recurrence therefore needs no barrier at all: its critical path per step
// is shfl + 4 dependent floating-point operations.  The other warps of the CTA
// are specialised: a producer streams the packs by TMA bulk copies
// (cp.async.bulk + mbarrier complete_tx) into a ring of D stages of kStage
// slices and drains the results, a mailbox warp fetches the neighbour bricks'
// edge values, and (K2) a residual warp computes the 8-term residuals ahead of
// the recurrence.  Across bricks, the producer stores self-validating tagged
// words (value + launch epoch) to a mailbox; the consumer's mailbox warp
// re-polls only while the epoch does not match.  No grid barrier, no counter.
//
// Bitwise parity: every cell performs the oracle's operations in the oracle's
// order (oracle/sip_oracle.c header); this file is compiled with
// --fmad=false and IEEE division, so no contraction changes the rounding.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>

#include "sip_internal.h"

namespace sipb {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// A value the compiler cannot re-derive: keeps the shared-window base in a
// register (otherwise it is rematerialised with S2R SR_CgaCtaId + LEA in
// every stage of the chain warps' loops).
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
  asm volatile("" : "+r"(x));
  return x;
}
// shared loads / stores by 32-bit shared address (volatile: kept in program
// order relative to the mbarrier waits / arrives that guard the slot)
template <typename T>
__device__ __forceinline__ T lds(uint32_t a);
template <>
__device__ __forceinline__ double lds<double>(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
template <>
__device__ __forceinline__ float lds<float>(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void sts(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
// Watchdog: a spin that makes no progress for kWatchdogNs aborts the kernel
// (__trap -> the launch fails with an error instead of hanging the GPU).
constexpr unsigned long long kWatchdogNs = 4000000000ULL;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __noinline__ void watchdog_fire(int where) {
  printf("sip watchdog: block %d thread %d stalled at site %d\n", blockIdx.x, threadIdx.x, where);
  __trap();
}
struct Watchdog {
  unsigned long long t0 = 0;
  int n = 0;
  __device__ __forceinline__ void idle(int where) {
    if ((++n & 255) == 0) {
      if (t0 == 0) t0 = gtime();
      else if (gtime() - t0 > kWatchdogNs) watchdog_fire(where);
    }
  }
};

// mbarrier + TMA bulk copies (1D, global -> shared)
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity, int where) {
  if (mbar_try(bar, parity)) return;
  Watchdog wd;
  while (!mbar_try(bar, parity)) wd.idle(where);
}
__device__ __forceinline__ void tma_1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ int pmod(int a, int q) {
  const int r = a % q;
  return r < 0 ? r + q : r;
}

// ---- tagged words: value bits + 32-bit epoch tag, single-copy atomic 64-bit words
template <typename T>
constexpr int kTagWords = sizeof(T) / 4;  // 64-bit words per tagged value
template <typename T>
struct Tagged;
template <>
struct Tagged<double> {
  unsigned long long w0 = ~0ull, w1 = ~0ull;
  __device__ __forceinline__ void load(const unsigned long long* src) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(src) : "memory");
  }
  __device__ __forceinline__ bool ok(uint32_t tag) const {
    return (uint32_t)(w0 >> 32) == tag && (uint32_t)(w1 >> 32) == tag;
  }
  __device__ __forceinline__ double value() const {
    return __longlong_as_double((long long)((w0 << 32) | (w1 & 0xFFFFFFFFull)));
  }
};
template <>
struct Tagged<float> {
  unsigned long long w0 = ~0ull;
  __device__ __forceinline__ void load(const unsigned long long* src) {
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w0) : "l"(src) : "memory");
  }
  __device__ __forceinline__ bool ok(uint32_t tag) const { return (uint32_t)(w0 >> 32) == tag; }
  __device__ __forceinline__ float value() const { return __uint_as_float((uint32_t)w0); }
};
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
// Predicated tagged store (no branch: a branch around an asm store would split
// the unrolled steps into basic blocks).
__device__ __forceinline__ void put_tagged_if(bool p, unsigned long long* dst, float v, uint32_t tag) {
  const unsigned long long w = ((unsigned long long)tag << 32) | __float_as_uint(v);
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.relaxed.gpu.global.u64 [%0], %1;\n}\n" ::"l"(dst),
               "l"(w), "r"((unsigned)p)
               : "memory");
}
__device__ __forceinline__ void put_tagged_if(bool p, unsigned long long* dst, double v, uint32_t tag) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned long long w0 = ((unsigned long long)tag << 32) | (b >> 32);
  const unsigned long long w1 = ((unsigned long long)tag << 32) | (b & 0xFFFFFFFFull);
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n @q st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};\n}\n" ::"l"(dst),
      "l"(w0), "l"(w1), "r"((unsigned)p)
      : "memory");
}
// Value of a tagged word loaded earlier; re-polls (L2) until the tag matches.
template <typename T>
__device__ __forceinline__ T take_tagged(Tagged<T> v, const unsigned long long* src, uint32_t tag,
                                         int where) {
  if (!v.ok(tag)) {
    Watchdog wd;
    do {
      v.load(src);
      wd.idle(where);
    } while (!v.ok(tag));
  }
  return v.value();
}

template <bool B>
struct BoolC {
  static constexpr bool value = B;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// Ticket of the next brick of this CTA (one warp): lane 0 claims, all agree.
__device__ __forceinline__ int claim(unsigned* state) {
  int t = 0;
  if (threadIdx.x == 0) t = (int)atomicAdd(state, 1u);
  return __shfl_sync(0xffffffffu, t, 0);
}

// Brick done: returns true (all lanes) in the CTA that finished the last brick.
// Called by one whole warp (its lane 0 counts).
__device__ __forceinline__ bool brick_done(unsigned* state, int nbricks) {
  int last = 0;
  if ((threadIdx.x & 31) == 0) {
    __threadfence();
    last = atomicAdd(state + 1, 1u) == (unsigned)nbricks - 1;
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (last) __threadfence();
  return last != 0;
}

__device__ __forceinline__ void trace_begin(unsigned long long* trace, int bid) {
  if (trace && (threadIdx.x & 31) == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    trace[4 * bid + 0] = gtime();
    trace[4 * bid + 2] = smid;
  }
}
__device__ __forceinline__ void trace_end(unsigned long long* trace, int bid) {
  if (trace && (threadIdx.x & 31) == 0) trace[4 * bid + 1] = gtime();
}

// =============================================================================
// K1: Stone factorisation, SPEC.md:146 -- once per system revision.  Same
// brick wavefront as K2 (the factor of a cell needs UN/UE/UT of its B, W and S
// neighbours); the coefficients are read with plain loads one stage at a time
// (not on the measured path).  Factors are computed in fp64 and stored in T.
// Mailbox entries carry (UN, UE, UT) as three tagged fp64 values.
// =============================================================================
template <typename T>
__global__ void __launch_bounds__(32) k_factor(const FactorParams<T> P) {
  const int lane = threadIdx.x;
  const uint32_t tag = *P.epoch;
  const double alpha = P.alpha;
  constexpr int MW = 3 * kTagWords<double>;  // words per mailbox entry
  for (;;) {
    const int tk = claim(P.state);
    if (tk >= P.nbricks) break;
    const int bid = P.order[tk];
    const BrickDesc bd = P.bricks[bid];
    const BlockDesc bk = P.blocks[bd.block];
    const int NST = bd.ns / kStage, nzW = bd.nz * kW;
    const bool lane_ok = lane < bd.wJ;
    double unP = 0.0, ueP = 0.0, utP = 0.0;  // own previous step (W neighbour)
    double wU[kW][3];                         // own steps tau - kW (B neighbour)
#pragma unroll
    for (int s = 0; s < kW; ++s) wU[s][0] = wU[s][1] = wU[s][2] = 0.0;
    for (int n = 0; n < NST; ++n) {
      // coefficients of the stage
      double a[kStage][7];
#pragma unroll
      for (int s = 0; s < kStage; ++s) {
        const double* src = P.coef + ((bd.slot + (long long)n * kStage + s) * P.coef_na) * kL + lane;
#pragma unroll
        for (int x = 0; x < 7; ++x) a[s][x] = __ldg(src + x * kL);
      }
      // cross-brick values of the stage: W column (lane jl at its il == 0 step),
      // S row (lanes 0..7 hold lane 0's steps s)
      double mw[3] = {0.0, 0.0, 0.0}, ms[3] = {0.0, 0.0, 0.0};
      {
        const int k = n - (lane >> 3);
        if (bd.mWe >= 0 && lane_ok && k >= 0 && k < bd.nz) {
          const unsigned long long* src = P.mA + (bd.mWe + (long long)k * kL + lane) * MW;
#pragma unroll
          for (int x = 0; x < 3; ++x) {
            Tagged<double> v;
            v.load(src + 2 * x);
            mw[x] = take_tagged(v, src + 2 * x, tag, 11);
          }
        }
        const int c = n * kStage + lane;
        if (lane < kStage && bd.mSr >= 0 && c < nzW && lane < bd.wI) {
          const unsigned long long* src = P.mB + (bd.mSr + c) * MW;
#pragma unroll
          for (int x = 0; x < 3; ++x) {
            Tagged<double> v;
            v.load(src + 2 * x);
            ms[x] = take_tagged(v, src + 2 * x, tag, 12);
          }
        }
      }
#pragma unroll
      for (int s = 0; s < kStage; ++s) {
        const int tau = n * kStage + s;
        const int c = tau - lane;
        const int il = (s - lane) & (kW - 1);
        const bool valid = lane_ok && c >= 0 && c < nzW && il < bd.wI;
        const bool wedge = il == 0;
        const double unB = wU[s][0], ueB = wU[s][1], utB = wU[s][2];
        const double unW = wedge ? mw[0] : unP, ueW = wedge ? mw[1] : ueP, utW = wedge ? mw[2] : utP;
        const double un1 = __shfl_up_sync(0xffffffffu, unP, 1);
        const double ue1 = __shfl_up_sync(0xffffffffu, ueP, 1);
        const double ut1 = __shfl_up_sync(0xffffffffu, utP, 1);
        const double s0 = __shfl_sync(0xffffffffu, ms[0], s);
        const double s1 = __shfl_sync(0xffffffffu, ms[1], s);
        const double s2 = __shfl_sync(0xffffffffu, ms[2], s);
        const double unS = lane == 0 ? s0 : un1, ueS = lane == 0 ? s1 : ue1, utS = lane == 0 ? s2 : ut1;
        const double ap = a[s][0], aw = a[s][1], ae = a[s][2], as = a[s][3], an = a[s][4];
        const double ab = a[s][5], at = a[s][6];
        // SPEC.md:146 with m_nb = A_nb, operation order of oracle/sip_oracle.c
        const double lb = ab / (1.0 + alpha * (unB + ueB));
        const double lw = aw / (1.0 + alpha * (unW + utW));
        const double ls = as / (1.0 + alpha * (ueS + utS));
        const double p1 = alpha * (lb * unB + lw * unW);
        const double p2 = alpha * (lb * ueB + ls * ueS);
        const double p3 = alpha * (lw * utW + ls * utS);
        const double den = ap + p1 + p2 + p3 - lb * utB - lw * ueW - ls * unS;
        const int k = c >> 3;
        if (valid && !(fabs(den) >= 1e-30)) {
          const long long cell = (long long)(bd.i0 + il + 1) +
                                 (long long)(bk.nx + 2) * ((long long)(bd.j0 + lane + 1) +
                                                           (long long)(bk.ny + 2) * (k + 1));
          atomicMin(P.bad, ((unsigned long long)bk.id << 40) | (unsigned long long)cell);
        }
        const double lp = 1.0 / den;
        double un = (an - p1) * lp, ue = (ae - p2) * lp, ut = (at - p3) * lp;
        if (!valid) un = ue = ut = 0.0;
        if (valid) {
          T* f = P.fw + ((bd.slot + tau) * F_NA) * kL + lane;
          f[F_LB * kL] = static_cast<T>(lb);
          f[F_LW * kL] = static_cast<T>(lw);
          f[F_LS * kL] = static_cast<T>(ls);
          f[F_LP * kL] = static_cast<T>(lp);
          T* u = P.bw + ((bd.slot + tau) * B_NA) * kL + lane;
          u[B_UN * kL] = static_cast<T>(un);
          u[B_UE * kL] = static_cast<T>(ue);
          u[B_UT * kL] = static_cast<T>(ut);
          if (il == kW - 1 && bd.mEe >= 0) {
            unsigned long long* dst = P.mA + (bd.medge + (long long)k * kL + lane) * MW;
            put_tagged(dst, un, tag);
            put_tagged(dst + 2, ue, tag);
            put_tagged(dst + 4, ut, tag);
          }
          if (lane == kL - 1 && bd.mNr >= 0) {
            unsigned long long* dst = P.mB + (bd.mrow + c) * MW;
            put_tagged(dst, un, tag);
            put_tagged(dst + 2, ue, tag);
            put_tagged(dst + 4, ut, tag);
          }
        }
        wU[s][0] = un; wU[s][1] = ue; wU[s][2] = ut;
        unP = un; ueP = ue; utP = ut;
      }
    }
    if (brick_done(P.state, P.nbricks) && lane == 0) *P.epoch = tag + 1;
  }
}

// =============================================================================
// K2: residual + L1 norm + forward substitution.  One CTA of five warps per
// brick, warp-specialised around a ring of D stage slots (mbarriers):
//   warp 0 "producer":   TMA bulk copies of the stage's forward pack slices and
//                        the next phi chunk, cp.async of the stage's W / E / S
//                        / N neighbour phi values        -> full[q]
//   warp 1 "residual":   r = -(AE*phiE) - AW*phiW - AN*phiN - AS*phiS - AT*phiT
//                        - AB*phiB + Q - AP*phiP, |r|    -> ready[q], empty[q]
//   warp 2 "recurrence": t1 = r - LB*R_B, R = ((t1 - LW*R_W) - LS*R_S) * LP
//                                                        -> rdone[q], empty[q]
//   warp 3 "mailbox":    polls the W brick's E column / S brick's N row
//                        (tagged words) for the stage    -> ready[q]
//   warp 4 "drain":      the E column / N row publishes and the R stores of a
//                        finished stage (smem -> HBM)    -> drained[q]
// The recurrence warp's per-step critical path is one shfl plus three
// dependent fp operations; everything else runs in the other warps.  phi
// chunks live in a mirrored ring (slices 8n-8 .. 8n+15 of stage n are
// contiguous: the B / T / W / E / S / N neighbours inside the brick are fixed
// offsets).
// =============================================================================
#ifndef SIPB_K2_D64
#define SIPB_K2_D64 3
#endif
#ifndef SIPB_K2_D32
#define SIPB_K2_D32 7  // measured 293 -> 291 us at 256^3 vs 5
#endif
#ifndef SIPB_K3_D
#define SIPB_K3_D 4  // even: slot q is always served by compute warp q & 1
#endif
#ifndef SIPB_K3_D32
#define SIPB_K3_D32 6  // fp32 (even); measured 235 -> 232 us at 256^3 vs 4
#endif
template <typename T>
struct K2Cfg {
  static constexpr int D = sizeof(T) == 8 ? SIPB_K2_D64 : SIPB_K2_D32;
  static constexpr int QP = D + 2;  // phi chunks in the ring (+2 mirror slots)
  static constexpr int kFw = kStage * F_NA * kL;  // forward pack elements per stage
  static constexpr int kCh = kStage * kL;          // one slice row per step
  // slot (T units): fw (TMA) | r (residual -> recurrence) | R (recurrence ->
  // producer) | edge phi phW[32] phE[32] phS[8] phN[8] (cp.async) | mailbox rW[32] eR[8]
  static constexpr int o_r = kFw, o_R = kFw + kCh, o_ed = kFw + 2 * kCh, o_mb = o_ed + 2 * kL + 2 * kStage;
  static constexpr size_t slot_bytes = (sizeof(T) * (o_mb + kL + kStage) + 127) / 128 * 128;
  static constexpr size_t off_ph = D * slot_bytes;
  static constexpr size_t off_bar = off_ph + sizeof(T) * (QP + 2) * kCh;
  static constexpr size_t off_misc = off_bar + 8 * 5 * D;  // full ready mbx rdone empty
  static constexpr size_t bytes = off_misc + 16;
  static constexpr int kThreads = 160;  // producer, residual, recurrence, mailbox, drain
};

// phase parity bit of slot q for one barrier kind, flipped after each wait
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t& phases, int q, int where) {
  mbar_wait(bar, (phases >> q) & 1u, where);
  phases ^= 1u << q;
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// arrive on `bar` once every cp.async this thread issued so far has landed
__device__ __forceinline__ void cp_async_arrive(uint32_t bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(dst), "l"(src), "n"(N) : "memory");
}
// whole warp: wait for a tagged word (already loaded once) to carry `tag`
template <typename T>
__device__ __forceinline__ T settle(Tagged<T> v, bool need, const unsigned long long* src, uint32_t tag,
                                   int where) {
  if (need && !v.ok(tag)) {
    Watchdog wd;
    do {
      v.load(src);
      wd.idle(where);
    } while (!v.ok(tag));
  }
  return need ? v.value() : T(0);
}

// Mailbox reads of the next stage are issued as soon as the current stage's
// settled (kLook = 1: read-ahead of 2 or 4 stages measured 6 % / 21 % slower
// at 256^3 -- stale in-flight reads of lines being written).
constexpr int kLook = 1;

template <typename T>
__global__ void __launch_bounds__(160) k_forward(const SweepParams<T> P) {
  using C = K2Cfg<T>;
  constexpr int D = C::D, QP = C::QP;
  extern __shared__ __align__(128) unsigned char smem[];
  auto slot = [&](int q) { return reinterpret_cast<T*>(smem + q * C::slot_bytes); };
  T* const s_ph = reinterpret_cast<T*>(smem + C::off_ph);
  const uint32_t sb = opaque(saddr(smem));
  const uint32_t full0 = sb + (uint32_t)C::off_bar, ready0 = full0 + 8 * D, mbx0 = ready0 + 8 * D,
                 rdone0 = mbx0 + 8 * D, empty0 = rdone0 + 8 * D;
  int* const s_brick = reinterpret_cast<int*>(smem + C::off_misc);
  double* const s_nrm = reinterpret_cast<double*>(smem + C::off_misc + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (*(volatile unsigned*)P.ctl) return;  // target reached by an earlier sweep
  const uint32_t tag = *P.epoch;
  if (threadIdx.x == 0) {
    for (int q = 0; q < D; ++q) {
      mbar_init(full0 + 8 * q, 33);  // producer lane 0 expect_tx + 32 cp.async arrivals
      mbar_init(ready0 + 8 * q, 2);  // residual warp (r) + mailbox warp (cross-brick R)
      mbar_init(mbx0 + 8 * q, kL);   // drained: every drain-warp lane (slot free for the producer)
      mbar_init(rdone0 + 8 * q, kL);      // recurrence warp, every lane: R of the stage in the slot
      mbar_init(empty0 + 8 * q, 1 + kL);  // residual (lane 0) + recurrence (every lane): inputs consumed
    }
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t ph_a = 0, ph_b = 0, ph_c = 0;  // per-warp parity bits of the barriers it waits on
  long long g = 0;                        // stages run by this CTA (all bricks)
  const int wedge_s = lane & (kW - 1);             // step of a stage with il == 0
  const int eedge_s = (lane + kW - 1) & (kW - 1);  // step with il == kW - 1
  constexpr uint32_t kFwBytes = sizeof(T) * C::kFw, kChBytes = sizeof(T) * C::kCh;

  for (;;) {
    if (threadIdx.x == 0) *s_brick = (int)atomicAdd(P.state, 1u);
    __syncthreads();
    const int tk = *s_brick;
    __syncthreads();
    if (tk >= P.nbricks) break;
    const int bid = P.order[tk];
    const BrickDesc bd = P.bricks[bid];
    const int NST = bd.ns / kStage, nzW = bd.nz * kW;
    const bool lane_ok = lane < bd.wJ;
#ifdef SIPB_STAGE_MARKS
    // pipeline timing of brick trace_brick (clock64, one SM; tools/k2_pipe.py):
    // region 2, per stage: 0 TMA issued, 1 residual past full, 2 residual
    // ready, 3 mailbox ready, 4 recurrence past ready, 5 recurrence rdone
    unsigned long long* const pmk =
        P.trace && bid == (P.trace_brick & 0xFFFFF) ? P.trace + 8ull * P.nbricks + 2 * kTraceStages * kTraceMarks
                                                    : nullptr;
    auto pm = [&](int n, int k) {
      if (pmk && (threadIdx.x & 31) == 0 && n < kTraceStages) pmk[n * kTraceMarks + k] = clock64();
    };
#else
    auto pm = [](int, int) {};
#endif

    if (warp == 0) {
      // ------------------------------------------------------------ producer
      const T* const fw_src = P.fw + bd.slot * F_NA * kL;
      const T* const ph_src = P.phi + bd.pslot * kL;
      const T* const phW_src = P.phi + (bd.pW + kW - 1) * kL + lane;
      const T* const phE_src = P.phi + (bd.pE - (kW - 1)) * kL + lane;
      const T* const phX_src = lane < kStage ? P.phi + (bd.pS + kL - 1 + lane) * kL + (kL - 1)
                                             : P.phi + (bd.pN - (kL - 1) + lane - kStage) * kL;
      auto put_chunk = [&](int c, uint32_t bar) {
        const int r = pmod(c, QP);
        const T* src = ph_src + (long long)c * C::kCh;
        tma_1d(saddr(s_ph + (r + 1) * C::kCh), src, kChBytes, bar);
        if (r == QP - 1) tma_1d(saddr(s_ph), src, kChBytes, bar);
        if (r == 0) tma_1d(saddr(s_ph + (QP + 1) * C::kCh), src, kChBytes, bar);
      };
      auto chunk_copies = [&](int c) { const int r = pmod(c, QP); return 1 + (r == QP - 1) + (r == 0); };
      int q = (int)(g % D);
      for (int n = 0; n < NST; ++n, ++g, q = q + 1 == D ? 0 : q + 1) {
        if (g >= D) {
          bar_wait(empty0 + 8 * q, ph_b, q, 40);
          bar_wait(mbx0 + 8 * q, ph_c, q, 45);  // the slot's previous stage drained
        }
        const uint32_t full = full0 + 8 * q;
        T* const ed = slot(q) + C::o_ed;
        const long long tb = (long long)n * kStage;
        cp_async<sizeof(T)>(saddr(ed + lane), phW_src + (tb + wedge_s) * kL);
        cp_async<sizeof(T)>(saddr(ed + kL + lane), phE_src + (tb + eedge_s) * kL);
        if (lane < 2 * kStage) cp_async<sizeof(T)>(saddr(ed + 2 * kL + lane), phX_src + tb * kL);
        if (lane == 0) {
          int nch = chunk_copies(n + 1);
          if (n == 0) nch += chunk_copies(-1) + chunk_copies(0);
          mbar_expect_tx(full, kFwBytes + (uint32_t)nch * kChBytes);
          tma_1d(saddr(slot(q)), fw_src + (long long)n * C::kFw, kFwBytes, full);
          if (n == 0) {
            put_chunk(-1, full);
            put_chunk(0, full);
          }
          put_chunk(n + 1, full);
        }
        cp_async_arrive(full);
        pm(n, 0);
      }
    } else if (warp == 1) {
      // ------------------------------------------------------------ residual
      double nrm = 0.0;
      int q = (int)(g % D);
      for (int n = 0; n < NST; ++n, ++g, q = q + 1 == D ? 0 : q + 1) {
        bar_wait(full0 + 8 * q, ph_a, q, 41);
        pm(n, 1);
        const T* const F = slot(q) + lane;
        const T* const ed = slot(q) + C::o_ed;
        const T* const Pw = s_ph + pmod(n, QP) * C::kCh + lane;  // slice 8n - 8
        T* const rout = slot(q) + C::o_r + lane;
        const T phW = ed[lane], phE = ed[kL + lane];
        // r of the 8 steps stays in registers until all are computed: a shared
        // store inside the loop may alias the next step's shared loads and
        // would serialise the 8 independent residual chains
        T rs[kStage];
        auto body = [&](auto masked) {
          constexpr bool M = decltype(masked)::value;
#pragma unroll
          for (int s = 0; s < kStage; ++s) {
            const T* f = F + s * F_NA * kL;
            const T* p = Pw + (kStage + s) * kL;  // slice tau = 8n + s
            // branch-free selects (a branch would split the unrolled steps)
            const T phiW = (s == wedge_s) ? phW : p[-kL];
            const T phiE = (s == eedge_s) ? phE : p[kL];
            const T phiS = *(lane == 0 ? ed + 2 * kL + s : p - kL - 1);
            const T phiN = *(lane == kL - 1 ? ed + 2 * kL + kStage + s : p + kL + 1);
            // residual_general, Listing-1 term order
            T r = -(f[F_AE * kL] * phiE);
            r -= f[F_AW * kL] * phiW;
            r -= f[F_AN * kL] * phiN;
            r -= f[F_AS * kL] * phiS;
            r -= f[F_AT * kL] * p[kW * kL];
            r -= f[F_AB * kL] * p[-kW * kL];
            r += f[F_Q * kL];
            r -= f[F_AP * kL] * p[0];
            if (M) {
              const int c = n * kStage + s - lane;
              const bool v = lane_ok && (unsigned)c < (unsigned)nzW && ((s - lane) & (kW - 1)) < bd.wI;
              nrm += v ? fabs(static_cast<double>(r)) : 0.0;
            } else {
              nrm += fabs(static_cast<double>(r));
            }
            rs[s] = r;
          }
        };
        const bool interior = bd.wI == kW && bd.wJ == kL && n >= kL / kStage && n + kL / kStage < NST;
        if (interior) body(BoolC<false>{});
        else body(BoolC<true>{});
#pragma unroll
        for (int s = 0; s < kStage; ++s) rout[s * kL] = rs[s];
        if (n == NST - 1) {
          const double v = warp_sum(nrm);
          if (lane == 0) *s_nrm = v;
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(ready0 + 8 * q);
          mbar_arrive(empty0 + 8 * q);
        }
        pm(n, 2);
      }
    } else if (warp == 2) {
      // ---------------------------------------------------------- recurrence
      trace_begin(P.trace, bid);
#ifdef SIPB_STAGE_MARKS
      unsigned long long* const marks =
          (P.trace && bid == P.trace_brick) ? P.trace + 8ull * P.nbricks : nullptr;
      auto mark = [&](int n, int m) {
        if (marks && lane == 0 && n < kTraceStages) marks[n * kTraceMarks + m] = clock64();
      };
#else
      auto mark = [](int, int) {};
#endif
      T Rprev = T(0);
      T win[kW];
#pragma unroll
      for (int s = 0; s < kW; ++s) win[s] = T(0);
      int q = (int)(g % D);
      g += NST;
      for (int n = 0; n < NST; ++n, q = q + 1 == D ? 0 : q + 1) {
        mark(n, 0);
        // ready = the residual warp's r (it waited for the TMA data of the
        // slot, so its release covers it) + the mailbox warp's values
        bar_wait(ready0 + 8 * q, ph_b, q, 43);
        mark(n, 1);
        pm(n, 4);
        constexpr uint32_t E = sizeof(T);
        const uint32_t sq = sb + (uint32_t)q * (uint32_t)C::slot_bytes, sl = sq + E * lane;
        const T rW = lds<T>(sl + E * C::o_mb);
        T rin[kStage], lb[kStage], lw[kStage], ls[kStage], lp[kStage], eR[kStage];
#pragma unroll
        for (int s = 0; s < kStage; ++s) {
          const uint32_t f = sl + E * (s * F_NA * kL);
          rin[s] = lds<T>(sl + E * (C::o_r + s * kL));
          lb[s] = lds<T>(f + E * (F_LB * kL));
          lw[s] = lds<T>(f + E * (F_LW * kL));
          ls[s] = lds<T>(f + E * (F_LS * kL));
          lp[s] = lds<T>(f + E * (F_LP * kL));
          eR[s] = lds<T>(sq + E * (C::o_mb + kL + s));
        }
        mbar_arrive(empty0 + 8 * q);  // slot inputs now in registers (every lane)
        // the recurrence; no masking on the chain: a valid
        // cell's W / S inputs are valid cells (or the mailbox), padding cells
        // compute exact zeros from the zero-filled packs
#pragma unroll
        for (int s = 0; s < kStage; ++s) {
          const T RS1 = __shfl_up_sync(0xffffffffu, Rprev, 1);
          const T RW = (s == wedge_s) ? rW : Rprev;
          const T RS = lane == 0 ? eR[s] : RS1;
          const T t1 = rin[s] - lb[s] * win[s];  // R_B: previous stage's step s
          const T R = ((t1 - lw[s] * RW) - ls[s] * RS) * lp[s];
          win[s] = R;
          Rprev = R;
        }
        mark(n, 2);
        // (masked) R into the slot: the producer stores it and publishes the
        // E column / N row; the masked copy is also the register window
        const bool interior = bd.wI == kW && bd.wJ == kL && n >= kL / kStage && n + kL / kStage < NST;
        if (!interior) {
#pragma unroll
          for (int s = 0; s < kStage; ++s) {
            const int c = n * kStage + s - lane;
            const bool v = lane_ok && (unsigned)c < (unsigned)nzW && ((s - lane) & (kW - 1)) < bd.wI;
            win[s] = v ? win[s] : T(0);
          }
        }
#pragma unroll
        for (int s = 0; s < kStage; ++s) sts(sl + E * (C::o_R + s * kL), win[s]);
        mbar_arrive(rdone0 + 8 * q);
        pm(n, 5);
        mark(n, 3);
#ifdef SIPB_STAGE_MARKS
        if (n == kL / kStage && P.trace && lane == 0) P.trace[4 * bid + 3] = gtime();
#endif
      }
      trace_end(P.trace, bid);
      // the residual warp's brick norm (written before its last ready arrive)
      if (lane == 0) P.partial[bid] = *s_nrm;
      if (brick_done(P.state, P.nbricks)) {
        // finaliser: deterministic per-block norms, then reset the backward state
        const unsigned it = *(volatile unsigned*)P.norm_it;
        double* bnorms = P.bnorms_base + (size_t)it * P.nblocks;
        double tot = 0.0;
        for (int b = 0; b < P.nblocks; ++b) {
          const BlockDesc bb = P.blocks[b];
          double v = 0.0;
          for (int x = lane; x < bb.nbricks; x += 32) v += __ldcg(P.partial + bb.brick0 + x);
          v = warp_sum(v);
          tot += v;  // blocks in ascending (local) order
          if (lane == 0) bnorms[b] = v;
        }
        if (lane == 0) {
          P.norms_base[it] = tot;
          *P.norm_it = it + 1;
          P.state_other[0] = 0u;
          P.state_other[1] = 0u;
          *P.epoch = tag + 1;
          P.ctl[1] = 1u;  // this sweep's K3 runs
          if (P.xseq) *P.xseq += 1u;  // K3's stamp value (split exchange)
          if (P.target > 0.0) {  // same test as the host loop: n0 == 0 or n / n0 <= target
            const double n0 = it == 0 ? tot : P.norms_base[0];
            if (n0 == 0.0 || tot / n0 <= P.target) P.ctl[0] = 1u;
          }
        }
      }
    } else if (warp == 4) {
      // --------------------------------------------------------------- drain
      // R of stage n (slot q) -> HBM once the recurrence warp is done with it,
      // and the cross-brick publishes: each lane's E-column value (its
      // il == kW-1 step) and, lanes 0..7, lane 31's N-row value of step lane;
      // then the slot is free for the producer (drained)
      T* const R_dst = P.R + bd.slot * kL + lane;
      int q = (int)(g % D);
      g += NST;
      for (int n = 0; n < NST; ++n, q = q + 1 == D ? 0 : q + 1) {
        bar_wait(rdone0 + 8 * q, ph_c, q, 44);
        const T* src = slot(q) + C::o_R;
        T v[kStage];
#pragma unroll
        for (int s = 0; s < kStage; ++s) v[s] = src[s * kL + lane];
        const T vE = src[eedge_s * kL + lane];
        const T vN = src[(lane & (kStage - 1)) * kL + (kL - 1)];
        // the neighbours' values first (on the wavefront's critical path)
        const int cE = n * kStage + eedge_s - lane;
        const bool pe = bd.mEe >= 0 && lane_ok && (unsigned)cE < (unsigned)nzW && ((cE & (kW - 1)) < bd.wI);
        put_tagged_if(pe, P.mA + (bd.medge + (long long)(pe ? cE >> 3 : 0) * kL + lane) * kTagWords<T>, vE, tag);
        const int cN = n * kStage + lane - (kL - 1);
        const bool pn = bd.mNr >= 0 && lane < kStage && bd.wJ == kL && (unsigned)cN < (unsigned)nzW &&
                        ((cN & (kW - 1)) < bd.wI);
        put_tagged_if(pn, P.mB + (bd.mrow + (pn ? cN : 0)) * kTagWords<T>, vN, tag);
        mbar_arrive(mbx0 + 8 * q);  // slot read out: the producer may refill it
#pragma unroll
        for (int s = 0; s < kStage; ++s) R_dst[((long long)n * kStage + s) * kL] = v[s];
      }
    } else {
      // ------------------------------------------------------------- mailbox
      // R of the W brick's E column at this lane's il == 0 step (lane jl:
      // entry k = n - jl / 8) and, lanes 16..23, of the S brick's N row at
      // lane 0's step lane - 16; read kLook stages ahead (only where a lane
      // needs a value), re-polled until this launch's tag shows, then
      // deposited in the slot (0 across a block boundary)
      if constexpr (sizeof(T) == 8) {
        // fp64 (HBM-bound): one read per stage, issued once the slot is free
        // (measured 5 % faster than the read-ahead below at 256^3; fp32, which
        // is hand-off bound, is 4 % faster with the read-ahead)
        int q = (int)(g % D);
        for (int n = 0; n < NST; ++n, ++g, q = q + 1 == D ? 0 : q + 1) {
          if (g >= D) bar_wait(empty0 + 8 * q, ph_a, q, 46);
          const int k = n - (lane >> 3);
          const bool needA = bd.mWe >= 0 && lane_ok && k >= 0 && k < bd.nz;
          const unsigned long long* aA = needA ? P.mA + (bd.mWe + (long long)k * kL + lane) * kTagWords<T> : P.mA;
          const int c = n * kStage + (lane - 2 * kStage);
          const bool needB =
              lane >= 2 * kStage && lane < 3 * kStage && bd.mSr >= 0 && c < nzW && (c & (kW - 1)) < bd.wI;
          const unsigned long long* aB = needB ? P.mB + (bd.mSr + c) * kTagWords<T> : P.mB;
          Tagged<T> tA, tB;
          tA.load(aA);
          tB.load(aB);
          const T vA = settle(tA, needA, aA, tag, 21);
          const T vB = settle(tB, needB, aB, tag, 22);
          T* const mb = slot(q) + C::o_mb;
          mb[lane] = vA;
          if (lane >= 2 * kStage && lane < 3 * kStage) mb[kL + lane - 2 * kStage] = vB;
          __syncwarp();
          if (lane == 0) mbar_arrive(ready0 + 8 * q);
          pm(n, 3);
        }
      } else {
        struct Req {
          const unsigned long long *aA, *aB;
          bool needA, needB;
        };
        auto req = [&](int n) {
          const int k = n - (lane >> 3);
          const int c = n * kStage + (lane - 2 * kStage);
          Req r;
          r.needA = n < NST && bd.mWe >= 0 && lane_ok && k >= 0 && k < bd.nz;
          r.needB = n < NST && lane >= 2 * kStage && lane < 3 * kStage && bd.mSr >= 0 && c < nzW &&
                    (c & (kW - 1)) < bd.wI;
          r.aA = r.needA ? P.mA + (bd.mWe + (long long)k * kL + lane) * kTagWords<T> : P.mA;
          r.aB = r.needB ? P.mB + (bd.mSr + c) * kTagWords<T> : P.mB;
          return r;
        };
        Tagged<T> tA[kLook], tB[kLook];
        auto issue = [&](int j, int n) {
          const Req r = req(n);
          tA[j] = Tagged<T>{};
          tB[j] = Tagged<T>{};
          if (r.needA) tA[j].load(r.aA);
          if (r.needB) tB[j].load(r.aB);
        };
#pragma unroll
        for (int j = 0; j < kLook; ++j) issue(j, j);
        int q = (int)(g % D);
        for (int n0 = 0; n0 < NST; n0 += kLook) {
#pragma unroll
          for (int j = 0; j < kLook; ++j) {
            const int n = n0 + j;
            if (n < NST) {
              if (g >= D) bar_wait(empty0 + 8 * q, ph_a, q, 46);
              const Req r = req(n);
              const T vA = settle(tA[j], r.needA, r.aA, tag, 21);
              const T vB = settle(tB[j], r.needB, r.aB, tag, 22);
              issue(j, n + kLook);
              T* const mb = slot(q) + C::o_mb;
              mb[lane] = vA;
              if (lane >= 2 * kStage && lane < 3 * kStage) mb[kL + lane - 2 * kStage] = vB;
              __syncwarp();
              if (lane == 0) mbar_arrive(ready0 + 8 * q);
              pm(n, 3);
              ++g;
              q = q + 1 == D ? 0 : q + 1;
            }
          }
        }
      }
    }
    __syncthreads();  // brick done in all roles before the next claim
  }
}

// =============================================================================
// K3: backward substitution + phi update (backward3d), slices in
// reverse:  delta = ((R - UN*dN) - UE*dE) - UT*dT,  phi += delta.
// dE: own previous step (or the E brick's W column, tagged), dN: lane + 1's
// previous step (shfl_down; lane 31: the N brick's S row), dT: own step
// tau + kW.  Five warps per brick: producer (TMA of R, phi, UN, UE, UT of a
// stage, D stages ahead), two compute warps taking alternate stages (the
// chain state handed over through shared memory), mailbox, and drain (phi +=
// delta of a finished stage -> HBM, the tagged publishes).
// =============================================================================
#ifndef SIPB_K3_MINB
#define SIPB_K3_MINB (sizeof(T) == 8 ? 3 : 4)  // resident CTAs per SM K3 is compiled for
#endif
template <typename T>
struct K3Cfg {
  static constexpr int D = sizeof(T) == 8 ? SIPB_K3_D : SIPB_K3_D32;
  static constexpr int kBw = kStage * B_NA * kL, kCh = kStage * kL;
  // slot (T units): bw | R | phi (TMA) | phi new (compute -> producer) | mailbox dE[32] eN[8]
  static constexpr int o_R = kBw, o_ph = kBw + kCh, o_pn = kBw + 2 * kCh, o_mb = kBw + 3 * kCh;
  static constexpr size_t slot_bytes = (sizeof(T) * (o_mb + kL + kStage) + 127) / 128 * 128;
  static constexpr size_t off_bar = D * slot_bytes;
  static constexpr size_t off_misc = off_bar + 8 * 4 * D;  // full mbx cdone empty
  // chain state handed between the two compute warps: [warp][kW + 1][kL]
  // (the masked window of the stage, then the last step's delta)
  static constexpr size_t off_hand = off_misc + 16;
  static constexpr size_t bytes = off_hand + sizeof(T) * 2 * (kW + 1) * kL;
  static constexpr int kThreads = 160;  // producer, compute x2, mailbox, drain
  static_assert(D % 2 == 0, "slot parity selects the compute warp");
};

template <typename T>
__global__ void __launch_bounds__(160, SIPB_K3_MINB) k_backward(const SweepParams<T> P) {
  using C = K3Cfg<T>;
  constexpr int D = C::D;
  extern __shared__ __align__(128) unsigned char smem[];
  auto slot = [&](int q) { return reinterpret_cast<T*>(smem + q * C::slot_bytes); };
  const uint32_t sb = opaque(saddr(smem));
  const uint32_t full0 = sb + (uint32_t)C::off_bar, mbx0 = full0 + 8 * D, cdone0 = mbx0 + 8 * D,
                 empty0 = cdone0 + 8 * D;
  int* const s_brick = reinterpret_cast<int*>(smem + C::off_misc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (!*(volatile unsigned*)(P.ctl + 1)) return;  // the sweep's K2 did not run (target reached)
  const uint32_t tag = *P.epoch;
  const unsigned xs = P.xflag ? *(volatile unsigned*)P.xseq : 0u;
  if (threadIdx.x == 0) {
    for (int q = 0; q < D; ++q) {
      mbar_init(full0 + 8 * q, 2);    // producer expect_tx + mailbox warp
      mbar_init(mbx0 + 8 * q, kL);    // drained: every drain-warp lane (slot free for the producer)
      mbar_init(cdone0 + 8 * q, kL);  // every lane of the slot's compute warp
      mbar_init(empty0 + 8 * q, kL);  // every lane of the slot's compute warp
    }
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t ph_a = 0, ph_b = 0, ph_c = 0;
  long long g = 0;
  constexpr uint32_t kBwBytes = sizeof(T) * C::kBw, kChBytes = sizeof(T) * C::kCh;
  const int eedge_s = (kW - (lane & (kW - 1))) & (kW - 1);  // step with il == kW - 1
  const int wedge_b = kW - 1 - (lane & (kW - 1));           // step with il == 0

  for (;;) {
    if (threadIdx.x == 0) *s_brick = (int)atomicAdd(P.state, 1u);
    __syncthreads();
    const int tk = *s_brick;
    __syncthreads();
    if (tk >= P.nbricks) break;
    const int bid = P.order[tk];
    const BrickDesc bd = P.bricks[bid];
    const int NST = bd.ns / kStage, nzW = bd.nz * kW;
    const bool lane_ok = lane < bd.wJ;
#ifdef SIPB_STAGE_MARKS
    // hand-off timing (globaltimer): region 3 = brick trace_brick + 1 (the E
    // neighbour), region 4 = brick trace_brick; marks: 0 mailbox poll start,
    // 1 mailbox value seen, 2 compute past full, 3 compute cdone, 4 published
    // (trace_brick: low 20 bits the brick, high bits the upstream offset, 0 = 1)
    const int tb = P.trace_brick & 0xFFFFF, tup = (P.trace_brick >> 20) ? (P.trace_brick >> 20) : 1;
    unsigned long long* const hm =
        P.trace && (bid == tb || bid == tb + tup)
            ? P.trace + 4ull * P.nbricks + (bid == tb ? 4 : 3) * kTraceStages * kTraceMarks
            : nullptr;
#ifdef SIPB_K3_CMARKS
    // compute-warp timeline (clock64, one SM; tools/k3_cmarks.py): 0 ready
    // at the hand-over barrier, 3 hand-over arrived (chain done), 5 past full
    auto hmark = [](int, int) {};
    auto cmark = [&](int m, int k) {
      if (hm && bid == tb && lane == 0 && m < kTraceStages) hm[m * kTraceMarks + k] = clock64();
    };
#else
    auto hmark = [&](int m, int k) {
      if (hm && lane == 0 && m < kTraceStages) hm[m * kTraceMarks + k] = gtime();
    };
    auto cmark = [](int, int) {};
#endif
#else
    auto cmark = [](int, int) {};
    auto hmark = [](int, int) {};
#endif

    if (warp == 0) {
      // ------------------------------------------------------------ producer
      // TMA copies only: stage m's UN UE UT, R and phi once the slot's inputs
      // were consumed (empty) and its previous stage was drained
      int q = (int)(g % D);
      for (int m = 0; m < NST; ++m, ++g, q = q + 1 == D ? 0 : q + 1) {
        if (g >= D) {
          bar_wait(empty0 + 8 * q, ph_b, q, 50);
          bar_wait(mbx0 + 8 * q, ph_c, q, 51);
        }
        if (lane == 0) {
          const int n = NST - 1 - m;  // stage m covers slices 8n .. 8n + 7
          const uint32_t full = full0 + 8 * q;
          const long long sl = bd.slot + (long long)n * kStage;
          T* const d = slot(q);
          mbar_expect_tx(full, kBwBytes + 2 * kChBytes);
          tma_1d(saddr(d), P.bw + sl * B_NA * kL, kBwBytes, full);
          tma_1d(saddr(d + C::o_R), P.R + sl * kL, kChBytes, full);
          tma_1d(saddr(d + C::o_ph), P.phi + (bd.pslot + (long long)n * kStage) * kL, kChBytes, full);
        }
      }
    } else if (warp == 4) {
      // --------------------------------------------------------------- drain
      // stage m (slices 8n .. 8n+7, n = NST-1-m) once its compute warp is
      // done: phi += delta on the valid cells (padding cells keep their
      // ghost values bit for bit) -> HBM, and the cross-brick publishes: each
      // lane's W-column delta (its il == 0 step) and, lanes 0..7, lane 0's
      // S-row delta of slice 8n + lane; then the slot is free (drained)
      T* const P_dst = P.phi + bd.pslot * kL + lane;
      const int wedge_o = lane & (kW - 1);  // slice offset of this lane's il == 0 step
      int q = (int)(g % D);
      g += NST;
      for (int m = 0; m < NST; ++m, q = q + 1 == D ? 0 : q + 1) {
        bar_wait(cdone0 + 8 * q, ph_c, q, 54);
        const int n = NST - 1 - m;
        const T* dsrc = slot(q) + C::o_pn;  // delta, slice-major
        const T* psrc = slot(q) + C::o_ph;  // old phi
        T v[kStage];
#pragma unroll
        for (int o = 0; o < kStage; ++o) {
          const int c = n * kStage + o - lane;
          const bool ok = lane_ok && (unsigned)c < (unsigned)nzW && ((o - lane) & (kW - 1)) < bd.wI;
          const T p = psrc[o * kL + lane];
          v[o] = ok ? p + dsrc[o * kL + lane] : p;
        }
        const T vW = dsrc[wedge_o * kL + lane];
        const T vS = dsrc[(lane & (kStage - 1)) * kL];
        // the neighbours' values first (on the wavefront's critical path)
        const int cW = n * kStage + wedge_o - lane;
        const bool pw = bd.mWe >= 0 && lane_ok && (unsigned)cW < (unsigned)nzW && ((cW & (kW - 1)) < bd.wI);
        put_tagged_if(pw, P.mA + (bd.medge + (long long)(pw ? cW >> 3 : 0) * kL + lane) * kTagWords<T>, vW, tag);
        const int cS = n * kStage + lane;
        const bool ps = bd.mSr >= 0 && lane < kStage && bd.wJ > 0 && (unsigned)cS < (unsigned)nzW &&
                        ((cS & (kW - 1)) < bd.wI);
        put_tagged_if(ps, P.mB + (bd.mrow + (ps ? cS : 0)) * kTagWords<T>, vS, tag);
        hmark(m, 4);
        mbar_arrive(mbx0 + 8 * q);  // slot read out: the producer may refill it
        // ghost / padding cells inside the brick's slices are written back
        // bit for bit, except the B ghost plane (c < 0, stages n < kL / kStage,
        // lanes with il + jl >= kW): the comm stream's face copies may write it
        // while this sweep runs (split exchange)
        if (n >= kL / kStage) {
#pragma unroll
          for (int o = 0; o < kStage; ++o) P_dst[((long long)n * kStage + o) * kL] = v[o];
        } else {
#pragma unroll
          for (int o = 0; o < kStage; ++o)
            if (n * kStage + o >= lane) P_dst[((long long)n * kStage + o) * kL] = v[o];
        }
        if (P.xflag && (m == NST - bd.nz || m == NST - 1)) {
          // stage NST - nz completes the brick's k = nz - 1 plane (its slices
          // 8(nz-1) ...), stage NST - 1 the brick: stamp for the face copies
          __threadfence();
          __syncwarp();
          if (lane == 0) {
            if (m == NST - bd.nz) *(volatile unsigned*)(P.xflag + 2 * bid) = xs;
            if (m == NST - 1) *(volatile unsigned*)(P.xflag + 2 * bid + 1) = xs;
          }
        }
      }
    } else if (warp == 1 || warp == 3) {
      // ------------------------------------------------------------- compute
      // Two compute warps take alternate stages (slot parity): while one runs
      // its stage's 8-step chain, the other loads the next stage's inputs and
      // stores its deltas, so only the chain and the hand-over of its state
      // (the masked window + the last delta, 9 values per lane, through
      // shared memory and a named barrier) are serial.  Per stage: wait for
      // the slot (TMA data + the mailbox warp's values), inputs -> registers,
      // release the slot, the chain, delta -> slot.  Every lane arrives on
      // empty / cdone (count 32).
      const int cw = warp == 1 ? 0 : 1;
      constexpr uint32_t E = sizeof(T);
      // hand-over rows through the opaque shared base (a generic pointer here
      // made the compiler rebuild the address with S2UR SR_CgaCtaId on the
      // chain's critical path every stage)
      const uint32_t hand_rx = sb + (uint32_t)C::off_hand + E * (uint32_t)(cw * (kW + 1) * kL + lane);
      const uint32_t hand_tx = sb + (uint32_t)C::off_hand + E * (uint32_t)((cw ^ 1) * (kW + 1) * kL + lane);
      const int q0 = (int)(g % D), qlast = (int)((g + NST - 1) % D);
      if (cw == (q0 & 1)) trace_begin(P.trace, bid);
      int q = q0;
      g += NST;
      for (int m = 0; m < NST; ++m, q = q + 1 == D ? 0 : q + 1) {
        if ((q & 1) != cw) continue;
        const int n = NST - 1 - m;
        bar_wait(full0 + 8 * q, ph_a, q, 33);
        hmark(m, 2);
        cmark(m, 5);
        const uint32_t sq = sb + (uint32_t)q * (uint32_t)C::slot_bytes, sl = sq + E * lane;
        const T dE = lds<T>(sl + E * C::o_mb);
        T rr[kStage], un[kStage], ue[kStage], ut[kStage], eN[kStage];
#pragma unroll
        for (int s = 0; s < kStage; ++s) {
          const int o = kStage - 1 - s;  // slice tau = 8n + o
          un[s] = lds<T>(sl + E * ((o * B_NA + B_UN) * kL));
          ue[s] = lds<T>(sl + E * ((o * B_NA + B_UE) * kL));
          ut[s] = lds<T>(sl + E * ((o * B_NA + B_UT) * kL));
          rr[s] = lds<T>(sl + E * (C::o_R + o * kL));
          eN[s] = lds<T>(sq + E * (C::o_mb + kL + s));
        }
        mbar_arrive(empty0 + 8 * q);  // slot inputs now in registers
        // chain state: zero at the brick's first stage, else from the other warp
        T dprev = T(0);
        T win[kW];
        if (m == 0) {
#pragma unroll
          for (int s = 0; s < kW; ++s) win[s] = T(0);
        } else {
          // named barrier 1 + cw: the other warp's bar.arrive + this warp's
          // bar.sync (64 threads, membar.cta semantics); the hand-overs
          // strictly alternate, so a barrier is never over-arrived (an
          // mbarrier hand-over measured ~6 % slower, a polled flag ~4 %)
          cmark(m, 0);
          asm volatile("bar.sync %0, 64;" ::"r"(1 + cw) : "memory");
          dprev = lds<T>(hand_rx + E * (kW * kL));
#pragma unroll
          for (int s = 0; s < kW; ++s) win[s] = lds<T>(hand_rx + E * (s * kL));
        }
#ifdef SIPB_K3_CMARKS
        // chain start: after dprev (the hand-over) is in a register
        if (dprev == T(1.2345e30)) asm volatile("");
        cmark(m, 1);
#endif
        // delta = ((R - UN*dN) - UE*dE) - UT*dT, dT = the
        // previous stage's step s (win); padding cells compute exact zeros
        // (zero-filled packs), stored copies masked below
#pragma unroll
        for (int s = 0; s < kStage; ++s) {
          const T utdt = ut[s] * win[s];
          const T dN1 = __shfl_down_sync(0xffffffffu, dprev, 1);
          const T dEv = (s == eedge_s) ? dE : dprev;
          const T dN = lane == kL - 1 ? eN[s] : dN1;
          const T d = ((rr[s] - un[s] * dN) - ue[s] * dEv) - utdt;
          win[s] = d;
          dprev = d;
        }
#ifdef SIPB_K3_CMARKS
        if (dprev == T(1.2345e30)) asm volatile("");  // chain end: the last step's delta computed
        cmark(m, 2);
#endif
        // the masked copy is the next stage's window and the slot's delta
        const bool interior = bd.wI == kW && bd.wJ == kL && n >= kL / kStage && n + kL / kStage < NST;
        if (!interior) {
#pragma unroll
          for (int s = 0; s < kStage; ++s) {
            const int o = kStage - 1 - s, c = n * kStage + o - lane;
            const bool v = lane_ok && (unsigned)c < (unsigned)nzW && ((o - lane) & (kW - 1)) < bd.wI;
            win[s] = v ? win[s] : T(0);
          }
        }
        if (m + 1 < NST) {  // hand the chain state to the other warp first
          sts(hand_tx + E * (kW * kL), dprev);
#pragma unroll
          for (int s = 0; s < kW; ++s) sts(hand_tx + E * (s * kL), win[s]);
          asm volatile("bar.arrive %0, 64;" ::"r"(1 + (cw ^ 1)) : "memory");
          cmark(m, 3);
        }
#pragma unroll
        for (int s = 0; s < kStage; ++s) sts(sl + E * (C::o_pn + (kStage - 1 - s) * kL), win[s]);
        mbar_arrive(cdone0 + 8 * q);
        hmark(m, 3);
#ifdef SIPB_STAGE_MARKS
        if (m == kL / kStage && P.trace && lane == 0) P.trace[4 * bid + 3] = gtime();
#endif
      }
      if (cw == (qlast & 1)) {  // the warp that ran the brick's last stage closes it
        trace_end(P.trace, bid);
        if (brick_done(P.state, P.nbricks) && lane == 0) {
          P.state_other[0] = 0u;
          P.state_other[1] = 0u;
          *P.epoch = tag + 1;
          P.ctl[1] = 0u;
        }
      }
    } else {
      // ------------------------------------------------------------- mailbox
      // delta of the E brick's W column at this lane's il == kW-1 step and,
      // lanes 24..31, of the N brick's S row at lane 31's step lane - 24;
      // reads issued kLook stages ahead, re-polled until this launch's tag
      struct Req {
        const unsigned long long *aA, *aB;
        bool needA, needB;
      };
      auto req = [&](int m) {
        const int n = NST - 1 - m;
        const int k = n - ((lane + kW - 1) >> 3);
        const int c = n * kStage - 3 * kStage - (lane - 3 * kStage);
        Req r;
        r.needA = m < NST && bd.mEe >= 0 && lane_ok && k >= 0 && k < bd.nz;
        r.needB = m < NST && lane >= 3 * kStage && bd.mNr >= 0 && c >= 0 && c < nzW && (c & (kW - 1)) < bd.wI;
        r.aA = r.needA ? P.mA + (bd.mEe + (long long)k * kL + lane) * kTagWords<T> : P.mA;
        r.aB = r.needB ? P.mB + (bd.mNr + c) * kTagWords<T> : P.mB;
        return r;
      };
      Tagged<T> tA[kLook], tB[kLook];
      auto issue = [&](int j, int m) {
        const Req r = req(m);
        tA[j] = Tagged<T>{};
        tB[j] = Tagged<T>{};
        if (r.needA) tA[j].load(r.aA);
        if (r.needB) tB[j].load(r.aB);
      };
#pragma unroll
      for (int j = 0; j < kLook; ++j) issue(j, j);
      int q = (int)(g % D);
      for (int m0 = 0; m0 < NST; m0 += kLook) {
#pragma unroll
        for (int j = 0; j < kLook; ++j) {
          const int m = m0 + j;
          if (m < NST) {
            if (g >= D) bar_wait(empty0 + 8 * q, ph_a, q, 56);
            hmark(m, 0);
            const Req r = req(m);
            const T vA = settle(tA[j], r.needA, r.aA, tag, 31);
            const T vB = settle(tB[j], r.needB, r.aB, tag, 32);
            hmark(m, 1);
            issue(j, m + kLook);
            T* const mb = slot(q) + C::o_mb;
            mb[lane] = vA;
            if (lane >= 3 * kStage) mb[kL + lane - 3 * kStage] = vB;
            __syncwarp();
            if (lane == 0) mbar_arrive(full0 + 8 * q);
            ++g;
            q = q + 1 == D ? 0 : q + 1;
          }
        }
      }
    }
    __syncthreads();
  }
}

// =============================================================================
// Layout / halo / utility kernels
// =============================================================================
__device__ __forceinline__ long long f3(int nx, int ny, int i, int j, int k) {
  return (long long)i + (long long)(nx + 2) * ((long long)j + (long long)(ny + 2) * k);
}
// linear interior cell -> (i, j, k), 0-based (blocks < 2^32 cells)
__device__ __forceinline__ void cell_ijk(const BlockDesc& bd, long long c, int& i, int& j, int& k) {
  const unsigned cu = (unsigned)c, r = cu / (unsigned)bd.nx;
  i = (int)(cu - r * (unsigned)bd.nx);
  j = (int)(r % (unsigned)bd.ny);
  k = (int)(r / (unsigned)bd.ny);
}

// Interior Field3 <-> brick layout, tiled (one CTA per brick x kXK k-levels):
// the brick's cells of the chunk go through shared memory, so Field3 is read
// (written) in 64 B row pieces (8 cells along i) and the brick array in 256 B
// slice rows (32 lanes).  A slice row holds cells of different k (lane jl is
// jl slices behind lane 0); each cell belongs to the chunk of its own k, so
// rows at chunk boundaries are shared between two CTAs, lane by lane.
// Brick element (slice tau, lane jl) of brick r: phi (PHI) or pack array arr.
constexpr int kXK = 16;
template <typename T, bool PHI>
__device__ __forceinline__ long long brick_elem(const BlockDesc& bd, int r, int tau, int na, int arr, int jl) {
  if (PHI) return (phi_slot(bd, r) + tau) * kL + jl;
  return ((bd.slot0 + (long long)r * bd.ns + tau) * na + arr) * kL + jl;
}
template <typename T, bool PHI, bool TO_BRICK>
__global__ void __launch_bounds__(256) k_tile_xfer(const BlockDesc* blocks, int b, const double* f3in, double* f3out,
                                                   const T* bin, T* bout, int na, int arr) {
  __shared__ double tile[kXK][kL][kW + 1];  // +1: no bank conflicts on the i-row accesses
  const BlockDesc bd = blocks[b];
  const int r = blockIdx.x, bi = r % bd.BX, bj = r / bd.BX, k0 = blockIdx.y * kXK;
  const int i0 = bi * kW, j0 = bj * kL, kn = min(kXK, bd.nz - k0);
  const int t = threadIdx.x, il = t & (kW - 1), jr = t >> 3;  // 8 x 32 cells per pass
  const bool rowok = i0 + il < bd.nx && j0 + jr < bd.ny;
  const int w = t >> 5, lane = t & 31;
  const bool lane_ok = j0 + lane < bd.ny;
  if (TO_BRICK) {
    for (int kk = 0; kk < kn; ++kk)
      if (rowok) tile[kk][jr][il] = f3in[f3(bd.nx, bd.ny, i0 + il + 1, j0 + jr + 1, k0 + kk + 1)];
    __syncthreads();
    // rows tau = k0 * kW .. (k0 + kn) * kW + kL - 2: lane's cell c = tau - lane
    for (int tau = k0 * kW + w; tau < (k0 + kn) * kW + kL - 1; tau += 8) {
      const int c = tau - lane, k = c >> 3, ci = c & (kW - 1);
      if (c >= k0 * kW && k < k0 + kn && lane_ok && i0 + ci < bd.nx)
        bout[brick_elem<T, PHI>(bd, r, tau, na, arr, lane)] = static_cast<T>(tile[k - k0][lane][ci]);
    }
  } else {
    for (int tau = k0 * kW + w; tau < (k0 + kn) * kW + kL - 1; tau += 8) {
      const int c = tau - lane, k = c >> 3, ci = c & (kW - 1);
      if (c >= k0 * kW && k < k0 + kn && lane_ok && i0 + ci < bd.nx)
        tile[k - k0][lane][ci] = static_cast<double>(bin[brick_elem<T, PHI>(bd, r, tau, na, arr, lane)]);
    }
    __syncthreads();
    for (int kk = 0; kk < kn; ++kk)
      if (rowok) f3out[f3(bd.nx, bd.ny, i0 + il + 1, j0 + jr + 1, k0 + kk + 1)] = tile[kk][jr][il];
  }
}
template <typename T, bool PHI, bool TO_BRICK>
static void launch_tile_xfer(const BlockDesc& hb, const BlockDesc* d_blocks, int b, const double* f3in, double* f3out,
                             const T* bin, T* bout, int na, int arr, cudaStream_t st) {
  if (hb.nbricks == 0 || hb.nz == 0) return;
  dim3 g(hb.nbricks, (hb.nz + kXK - 1) / kXK);
  k_tile_xfer<T, PHI, TO_BRICK><<<g, 256, 0, st>>>(d_blocks, b, f3in, f3out, bin, bout, na, arr);
}

__device__ __forceinline__ void face_cell(const BlockDesc& bd, int f, int x0, int x1, bool ghost,
                                          int& i, int& j, int& k) {
  switch (f) {
    case G_W: i = ghost ? -1 : 0; j = x0; k = x1; break;
    case G_E: i = ghost ? bd.nx : bd.nx - 1; j = x0; k = x1; break;
    case G_S: i = x0; j = ghost ? -1 : 0; k = x1; break;
    case G_N: i = x0; j = ghost ? bd.ny : bd.ny - 1; k = x1; break;
    case G_B: i = x0; j = x1; k = ghost ? -1 : 0; break;
    default: i = x0; j = x1; k = ghost ? bd.nz : bd.nz - 1; break;
  }
}
__device__ __forceinline__ void face_dims(const BlockDesc& bd, int f, int& n0, int& n1) {
  if (f <= G_E) { n0 = bd.ny; n1 = bd.nz; }
  else if (f <= G_N) { n0 = bd.nx; n1 = bd.nz; }
  else { n0 = bd.nx; n1 = bd.ny; }
}

// Field3 -> phi ghost faces (blockIdx.y = face; the interior: k_tile_xfer)
template <typename T>
__global__ void k_phi_in(const double* __restrict__ src, const BlockDesc* blocks, int b, T* phi) {
  const BlockDesc bd = blocks[b];
  const int f = blockIdx.y;  // ghost face (the interior: k_tile_xfer)
  int n0, n1;
  face_dims(bd, f, n0, n1);
  const long long n = (long long)n0 * n1;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    int i, j, k;
    face_cell(bd, f, (int)(c % n0), (int)(c / n0), true, i, j, k);
    phi[phi_index(bd, i, j, k)] = static_cast<T>(src[f3(bd.nx, bd.ny, i + 1, j + 1, k + 1)]);
  }
}

// phi -> Field3: interior, plus the ghost faces whose bit is set in nbrmask
// (faces written by the halo plan).  blockIdx.y: 6 = interior, else face.
template <typename T>
__global__ void k_gather(const T* __restrict__ phi, const BlockDesc* blocks, int b, int nbrmask,
                         double* dst) {
  const BlockDesc bd = blocks[b];
  const int f = blockIdx.y;  // ghost face (the interior: k_tile_xfer)
  if (!((nbrmask >> f) & 1)) return;
  int n0, n1;
  face_dims(bd, f, n0, n1);
  const long long m = (long long)n0 * n1;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < m;
       c += (long long)gridDim.x * blockDim.x) {
    int i, j, k;
    face_cell(bd, f, (int)(c % n0), (int)(c / n0), true, i, j, k);
    dst[f3(bd.nx, bd.ny, i + 1, j + 1, k + 1)] = static_cast<double>(phi[phi_index(bd, i, j, k)]);
  }
}

template <typename T>
__global__ void k_gather_any(const T* __restrict__ pack, int na, int arr, const BlockDesc* blocks,
                             int b, double* dst) {
  const BlockDesc bd = blocks[b];
  const long long n = (long long)bd.nx * bd.ny * bd.nz;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    int i, j, k;
    cell_ijk(bd, c, i, j, k);
    const long long x = na > 0 ? pack_index(bd, na, arr, i, j, k) : phi_index(bd, i, j, k);
    dst[f3(bd.nx, bd.ny, i + 1, j + 1, k + 1)] = static_cast<double>(pack[x]);
  }
}

// K4: face copies.  grid.y = copy index.  Source: interior plane `src_face`
// of local block src_block (phi) or buf_in; destination: ghost face dst_face
// of local block dst_block (phi ghost cells) or buf_out.
template <typename T>
__global__ void k_face_copy(const FaceCopy* copies, const BlockDesc* blocks, T* phi, const T* buf_in,
                            T* buf_out) {
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
      v = phi[phi_index(sb, i, j, k)];
    } else {
      v = buf_in[fc.buf + c];
    }
    if (fc.dst_block >= 0) {
      const BlockDesc db = blocks[fc.dst_block];
      int i, j, k;
      face_cell(db, fc.dst_face, x0, x1, true, i, j, k);
      phi[phi_index(db, i, j, k)] = v;
    } else {
      buf_out[fc.buf + c] = v;
    }
  }
}

// K4, split exchange phase 1: the copies whose source is an E,
// N or T interior plane, launched on the comm stream as soon as K2 finished,
// i.e. while K3 runs (K3 completes those planes early: it starts at the
// block's E / N / T corner, and each brick's k = nz - 1 slices come first).
// One work item = the part of a plane one brick holds; CTA b of G (half the
// SMs: K3 always keeps SMs of its own) takes items b, b + G, ... (the host orders them by when K3 finishes them) and waits for
// the brick's stamp from K3 (this iteration's value) before copying.  The
// wait points one way only (K3 never waits on this kernel), and the CTAs are
// small (64 threads, <= 64 registers: the 4096 registers three fp64 K3 CTAs
// leave free), so each fits next to K3's resident CTAs on its SM: no
// deadlock for any residency, and K3 keeps its occupancy.  Each thread keeps
// 8 independent loads in flight.
constexpr int kXCopyThreads = 64;
template <typename T>
__global__ void __launch_bounds__(kXCopyThreads, 16)
    k_face_copy_after(const FaceCopy* copies, const XItem* items, int nitems, const BlockDesc* blocks,
                      T* phi, T* buf_out, const unsigned* xflag, const unsigned* xseq,
                      unsigned long long* xtrace) {
  const unsigned want = *(const volatile unsigned*)xseq;
  // debug timeline (tools/xsplit_timeline.py): this CTA's first item start, last item end
  if (xtrace && threadIdx.x == 0 && blockIdx.x < nitems) xtrace[2 * blockIdx.x] = gtime();
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const XItem xi = items[it];
    // descriptors first (independent of the stamp), then thread 0's wait
    const FaceCopy fc = copies[xi.entry];
    const BlockDesc sb = blocks[fc.src_block];
    const BlockDesc db = blocks[fc.dst_block >= 0 ? fc.dst_block : fc.src_block];
    if (threadIdx.x == 0) {
      const unsigned* f = xflag + 2ll * xi.brick + xi.sel;
      Watchdog wd;
      while (ld_acquire_u32(f) != want) {
        __nanosleep(100);
        wd.idle(60);
      }
    }
    __syncthreads();  // thread 0's acquire orders the CTA's phi reads after K3's stores
    const int w = xi.x0e - xi.x0b, n = w * (xi.x1e - xi.x1b);
    constexpr int U = 8;
    for (int c0 = 0; c0 < n; c0 += U * kXCopyThreads) {
      T v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * kXCopyThreads + threadIdx.x;
        if (c < n) {
          int i, j, k;
          face_cell(sb, fc.src_face, xi.x0b + c % w, xi.x1b + c / w, false, i, j, k);
          v[u] = phi[phi_index(sb, i, j, k)];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * kXCopyThreads + threadIdx.x;
        if (c < n) {
          const int x0 = xi.x0b + c % w, x1 = xi.x1b + c / w;
          if (fc.dst_block >= 0) {
            int i, j, k;
            face_cell(db, fc.dst_face, x0, x1, true, i, j, k);
            phi[phi_index(db, i, j, k)] = v[u];
          } else {
            buf_out[fc.buf + x0 + (long long)fc.n0 * x1] = v[u];
          }
        }
      }
    }
  }
  if (xtrace && threadIdx.x == 0 && blockIdx.x < nitems) xtrace[2 * blockIdx.x + 1] = gtime();
}

// residual_general or, with SYM, residual_symmetric
// (Listing PAPER.md:503-518): the W / S / B couplings are
// read as the E / N / T coefficients of the W / S / B neighbour cell (5
// coefficient arrays instead of 8); at the block's first interior cell the
// neighbour is the ghost cell, whose AE (AN, AT) equals this cell's AW (AS,
// AB) by the symmetry invariant, so AW (AS, AB) is read there.
template <typename T, bool SYM>
__global__ void k_residual(const BlockDesc* blocks, int b, const T* __restrict__ fw,
                           const T* __restrict__ phi, double* out) {
  const BlockDesc bd = blocks[b];
  const long long n = (long long)bd.nx * bd.ny * bd.nz;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    int i, j, k;
    cell_ijk(bd, c, i, j, k);
    auto ph = [&](int ii, int jj, int kk) -> T { return phi[phi_index(bd, ii, jj, kk)]; };
    auto A = [&](int arr) -> T { return fw[pack_index(bd, F_NA, arr, i, j, k)]; };
    T aw, as, ab;
    if (SYM) {
      aw = i > 0 ? fw[pack_index(bd, F_NA, F_AE, i - 1, j, k)] : A(F_AW);
      as = j > 0 ? fw[pack_index(bd, F_NA, F_AN, i, j - 1, k)] : A(F_AS);
      ab = k > 0 ? fw[pack_index(bd, F_NA, F_AT, i, j, k - 1)] : A(F_AB);
    } else {
      aw = A(F_AW);
      as = A(F_AS);
      ab = A(F_AB);
    }
    T v = -(A(F_AE) * ph(i + 1, j, k));
    v -= aw * ph(i - 1, j, k);
    v -= A(F_AN) * ph(i, j + 1, k);
    v -= as * ph(i, j - 1, k);
    v -= A(F_AT) * ph(i, j, k + 1);
    v -= ab * ph(i, j, k - 1);
    v += A(F_Q);
    v -= A(F_AP) * ph(i, j, k);
    out[f3(bd.nx, bd.ny, i + 1, j + 1, k + 1)] = static_cast<double>(v);
  }
}

// Symmetry invariant of a StencilSystem on the fp64 coefficients:
// AE(i) == AW(i+1), AN(j) == AS(j+1), AT(k) == AB(k+1) exactly; counts violations.
__global__ void k_check_symmetric(const BlockDesc* blocks, int b, const double* __restrict__ cf,
                                  int na, unsigned long long* bad) {
  const BlockDesc bd = blocks[b];
  const long long n = (long long)bd.nx * bd.ny * bd.nz;
  unsigned long long cnt = 0;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    int i, j, k;
    cell_ijk(bd, c, i, j, k);
    if (i + 1 < bd.nx && cf[pack_index(bd, na, F_AE, i, j, k)] != cf[pack_index(bd, na, F_AW, i + 1, j, k)]) ++cnt;
    if (j + 1 < bd.ny && cf[pack_index(bd, na, F_AN, i, j, k)] != cf[pack_index(bd, na, F_AS, i, j + 1, k)]) ++cnt;
    if (k + 1 < bd.nz && cf[pack_index(bd, na, F_AT, i, j, k)] != cf[pack_index(bd, na, F_AB, i, j, k + 1)]) ++cnt;
  }
  if (cnt) atomicAdd(bad, cnt);
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
    } else if (A.kind == 3) {  // symmetric: one coefficient per face (sip_gen.cpp)
      const uint64_t sy = (uint64_t)A.g[0], sz = (uint64_t)A.g[0] * (uint64_t)A.g[1];
      ae = -(1.0 + 0.5 * u01(A.seed, 1, cell));
      an = -(1.0 + 0.5 * u01(A.seed, 3, cell));
      at = -(1.0 + 0.5 * u01(A.seed, 5, cell));
      aw = gi > 0 ? -(1.0 + 0.5 * u01(A.seed, 1, cell - 1)) : 0.0;
      as = gj > 0 ? -(1.0 + 0.5 * u01(A.seed, 3, cell - sy)) : 0.0;
      ab = gk > 0 ? -(1.0 + 0.5 * u01(A.seed, 5, cell - sz)) : 0.0;
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

template <typename T>
int launch_factor(const FactorParams<T>& p, int grid, void* stream) {
  k_factor<T><<<grid, 32, 0, (cudaStream_t)stream>>>(p);
  return cuda_status(cudaGetLastError());
}
template int launch_factor<double>(const FactorParams<double>&, int, void*);
template int launch_factor<float>(const FactorParams<float>&, int, void*);

template <typename T>
static bool sweep_attrs() {
  static bool done = [] {
    cudaFuncSetAttribute(k_forward<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K2Cfg<T>::bytes);
    cudaFuncSetAttribute(k_backward<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K3Cfg<T>::bytes);
    return true;
  }();
  return done;
}

// The symmetric (Listing-1) forward variant is not separate here: the general
// kernel computes the same values with the same rounding on a symmetric system.
template <typename T>
int launch_forward(const SweepParams<T>& p, int grid, void* stream) {
  sweep_attrs<T>();
  k_forward<T><<<grid, K2Cfg<T>::kThreads, K2Cfg<T>::bytes, (cudaStream_t)stream>>>(p);
  return cuda_status(cudaGetLastError());
}

template <typename T>
int launch_backward(const SweepParams<T>& p, int grid, void* stream) {
  sweep_attrs<T>();
  k_backward<T><<<grid, K3Cfg<T>::kThreads, K3Cfg<T>::bytes, (cudaStream_t)stream>>>(p);
  return cuda_status(cudaGetLastError());
}

int max_resident_ctas(int kind, int precision, int* grid) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaSuccess;
  const bool dbl = precision == SIP_PREC_DOUBLE;
  if (dbl) sweep_attrs<double>(); else sweep_attrs<float>();
  if (kind == 0) {
    e = dbl ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_factor<double>, 32, 0)
            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_factor<float>, 32, 0);
  } else if (kind == 1) {
    e = dbl ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_forward<double>, K2Cfg<double>::kThreads, K2Cfg<double>::bytes)
            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_forward<float>, K2Cfg<float>::kThreads, K2Cfg<float>::bytes);
  } else {
    e = dbl ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_backward<double>, K3Cfg<double>::kThreads, K3Cfg<double>::bytes)
            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_backward<float>, K3Cfg<float>::kThreads, K3Cfg<float>::bytes);
  }
  if (e != cudaSuccess || per < 1) return SIP_ERR_CUDA;
  *grid = per * sms;
  return SIP_OK;
}

template <typename T>
int launch_scatter(const double* src, const BlockDesc* d_blocks, int block, const BlockDesc& hb,
                   T* pack, int na, int arr, void* stream) {
  launch_tile_xfer<T, false, true>(hb, d_blocks, block, src, nullptr, nullptr, pack, na, arr, (cudaStream_t)stream);
  return cuda_status(cudaGetLastError());
}
template <typename T>
int launch_phi_in(const double* src, const BlockDesc* d_blocks, int block, const BlockDesc& hb,
                  T* phi, void* stream) {
  // interior tiled; the six ghost faces (blockIdx.y 0..5) by k_phi_in
  launch_tile_xfer<T, true, true>(hb, d_blocks, block, src, nullptr, nullptr, phi, 1, 0, (cudaStream_t)stream);
  dim3 g(grid_for((long long)hb.nx * hb.ny * hb.nz) / 4 + 1, 6);
  k_phi_in<T><<<g, 256, 0, (cudaStream_t)stream>>>(src, d_blocks, block, phi);
  return cuda_status(cudaGetLastError());
}
template <typename T>
int launch_gather(const T* phi, const BlockDesc* d_blocks, int block, const BlockDesc& hb,
                  const int* nbr6, double* dst, void* stream) {
  int mask = 0;
  for (int f = 0; f < 6; ++f)
    if (nbr6[f] >= 0) mask |= 1 << f;
  // interior tiled; the ghost faces the plan writes (blockIdx.y 0..5) by k_gather
  launch_tile_xfer<T, true, false>(hb, d_blocks, block, nullptr, dst, phi, nullptr, 1, 0, (cudaStream_t)stream);
  dim3 g(grid_for((long long)hb.nx * hb.ny * hb.nz) / 4 + 1, 6);
  k_gather<T><<<g, 256, 0, (cudaStream_t)stream>>>(phi, d_blocks, block, mask, dst);
  return cuda_status(cudaGetLastError());
}
template <typename T>
int launch_face_copies(const FaceCopy* d_copies, int ncopies, int max_plane,
                       const BlockDesc* d_blocks, T* phi, const T* buf_in, T* buf_out,
                       void* stream) {
  if (ncopies <= 0) return SIP_OK;
  int gx = (max_plane + 255) / 256;
  if (gx > 64) gx = 64;
  dim3 g(gx, ncopies);
  k_face_copy<T><<<g, 256, 0, (cudaStream_t)stream>>>(d_copies, d_blocks, phi, buf_in, buf_out);
  return cuda_status(cudaGetLastError());
}
template <typename T>
int launch_face_copies_after(const FaceCopy* d_copies, const XItem* d_items, int nitems,
                             const BlockDesc* d_blocks, T* phi, T* buf_out, const unsigned* xflag,
                             const unsigned* xseq, unsigned long long* xtrace, void* stream) {
  if (nitems <= 0) return SIP_OK;
  static int grid = 0;
  if (grid == 0) {
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    grid = std::max(1, nsm / 2);
    // keep the SMs that host a copy CTA in the large-shared configuration K3
    // needs (a CTA without shared memory would otherwise let its SM switch to
    // a small carveout, and K3's CTAs could not join it until the copy CTA
    // exits -- with a copy CTA on every SM, K3 would never start)
    cudaFuncSetAttribute(k_face_copy_after<T>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         (int)cudaSharedmemCarveoutMaxShared);
  }
  k_face_copy_after<T><<<grid, kXCopyThreads, 0, (cudaStream_t)stream>>>(
      d_copies, d_items, nitems, d_blocks, phi, buf_out, xflag, xseq, xtrace);
  return cuda_status(cudaGetLastError());
}
template <typename T>
int launch_residual(const BlockDesc* d_blocks, int block, const BlockDesc& hb, const T* fw,
                    const T* phi, int symmetric, double* out, void* stream) {
  const int g = grid_for((long long)hb.nx * hb.ny * hb.nz);
  if (symmetric)
    k_residual<T, true><<<g, 256, 0, (cudaStream_t)stream>>>(d_blocks, block, fw, phi, out);
  else
    k_residual<T, false><<<g, 256, 0, (cudaStream_t)stream>>>(d_blocks, block, fw, phi, out);
  return cuda_status(cudaGetLastError());
}
int launch_check_symmetric(const BlockDesc* d_blocks, int block, const BlockDesc& hb,
                           const double* coef, int coef_na, unsigned long long* bad, void* stream) {
  k_check_symmetric<<<grid_for((long long)hb.nx * hb.ny * hb.nz), 256, 0, (cudaStream_t)stream>>>(
      d_blocks, block, coef, coef_na, bad);
  return cuda_status(cudaGetLastError());
}
template <typename T>
int launch_gather_any(const T* pack, int na, int arr, const BlockDesc* d_blocks, int block,
                      const BlockDesc& hb, double* dst, void* stream) {
  k_gather_any<T><<<grid_for((long long)hb.nx * hb.ny * hb.nz), 256, 0, (cudaStream_t)stream>>>(
      pack, na, arr, d_blocks, block, dst);
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
  template int launch_phi_in<T>(const double*, const BlockDesc*, int, const BlockDesc&, T*,      \
                                void*);                                                           \
  template int launch_gather<T>(const T*, const BlockDesc*, int, const BlockDesc&, const int*,    \
                                double*, void*);                                                  \
  template int launch_face_copies<T>(const FaceCopy*, int, int, const BlockDesc*, T*, const T*,   \
                                     T*, void*);                                                  \
  template int launch_face_copies_after<T>(const FaceCopy*, const XItem*, int, const BlockDesc*,   \
                                           T*, T*, const unsigned*, const unsigned*,              \
                                           unsigned long long*, void*);                           \
  template int launch_residual<T>(const BlockDesc*, int, const BlockDesc&, const T*, const T*,    \
                                  int, double*, void*);                                           \
  template int launch_gather_any<T>(const T*, int, int, const BlockDesc*, int, const BlockDesc&,  \
                                    double*, void*);
SIPB_INST(double)
SIPB_INST(float)

}  // namespace sipb
