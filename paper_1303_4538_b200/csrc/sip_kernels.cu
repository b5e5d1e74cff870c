// sip_kernels.cu -- sm_100a kernels of the SIP hot path.
//
//   K1 k_factor    Stone ILU factor          wavefront, fp64
//   K2 k_forward   residual + L1 norm + forward substitution   wavefront, critical /
//                  (resforward3d, SPEC.md:155 + SPEC.md:173)    residual thread groups
//   K3 k_backward  backward substitution + phi update          wavefront
//                  (backward3d)
//   k_edge_phi     static edge records of K2 (old neighbour phi / ghosts per step)
//   K4 k_face_copy face-halo copies / pack / unpack (exvec)
//   K5 k_convert   fp64 -> fp32 (Field3::cast, field.hpp:61-68)
//   K7 k_scatter / k_gather / k_ghost_in   Field3 <-> tile-slice layout
//   k_residual     residual_general / residual_symmetric
//
// Wavefront scheme: a persistent CTA owns a 16x16-column
// tile at a time and walks the tile's hyperplanes t = k + ti + tj.  Inside a
// tile the W/S (forward) or E/N (backward) neighbours of a cell were produced
// one step earlier by neighbouring threads (shared memory, one barrier per
// step); the B/T neighbour is the thread's own previous value (register).
// Across tiles, the edge threads store self-validating tagged words to global
// memory and the consuming edge threads poll them ahead of use, so there is no
// grid-wide barrier and no progress counter.  Tiles are claimed through an
// atomic ticket in topological order: deadlock-free for any residency.
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
// Watchdog: a spin that makes no progress for kWatchdogNs aborts the kernel
// (__trap -> the launch fails with an error instead of hanging the GPU).
constexpr unsigned long long kWatchdogNs = 4000000000ULL;

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
// Idle-loop watchdog of polling loops (reset whenever progress was made).
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

// Named barriers of the split forward sweep (id 0 = __syncthreads).
__device__ __forceinline__ void nbar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
// L2 prefetch of a contiguous range by the TMA engine (one instruction).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
#ifdef SIPB_EXP_NOPF
  return;
#endif
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// LSU-side L2 prefetch of one 128-byte line (does not use the TMA engine)
__device__ __forceinline__ void prefetch_line_l2(const void* p) {
#ifdef SIPB_EXP_NOPF
  return;
#endif
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
#ifdef SIPB_EXP_PFL
constexpr int kPFL = SIPB_EXP_PFL;
#else
constexpr int kPFL = 2;  // L2 prefetch distance (steps) beyond the loads it covers
#endif
// Progress counter of the publisher (slots of the out-record ring it has
// read): a relaxed shared store.  A release here (MEMBAR.ALL.CTA) would wait
// for the publisher's just-issued global edge stores; the only hazard it
// guards is shared (its reads of out-record slots, whose values its issued
// stores have already consumed, against the compute warps' later rewrite,
// ordered through the fetcher's mbarrier arrive and the compute's wait).
// Spin until *p >= need with cheap relaxed loads, then one CTA fence (the
// relaxed load that observed the released value + fence = acquire pattern).

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
// Warp-collective test of a step-done barrier: complete only if every lane
// observed completion (each such lane holds its own acquire).

// =============================================================================
// K2 / K3: one CTA of 256 threads per 16x16-column tile, persistent, tiles
// taken in topological ticket order (an upstream tile always holds an
// earlier ticket, so spinning on it cannot deadlock).  Each thread owns one
// column and walks the tile's hyperplanes; per step it meets the other 255
// threads at one barrier, nothing else.
//   * own data (forward pack, phi, R / backward pack) are LDG'd by each
//     thread two or more steps ahead into registers (coalesced: the pack is
//     slice-major, anti-diagonal positions);
//   * in-tile neighbour values go through small shared rings (phi slices,
//     the static edge-phi record, R / delta of the previous step);
//   * cross-tile values: the producing edge threads store tagged words
//     (value + (epoch, k) tag) straight to global memory; the consuming edge
//     threads issue the poll load two steps ahead and re-poll only if the tag
//     does not match yet.  No service warps, no counters, no fences.
// Iteration t of K2 computes critical(t) and the residual of step t+1: both
// sets of shared loads are issued first, so the residual fills the latency
// of the recurrence.
// =============================================================================

// Poll words of one tagged value: issued early, decoded when consumed.
template <typename T>
struct TagPoll;
template <>
struct TagPoll<double> {
  unsigned long long w0 = ~0ull, w1 = ~0ull;
  __device__ __forceinline__ void issue(const unsigned long long* src) {
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
struct TagPoll<float> {
  unsigned long long w0 = ~0ull;
  __device__ __forceinline__ void issue(const unsigned long long* src) {
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w0) : "l"(src) : "memory");
  }
  __device__ __forceinline__ bool ok(uint32_t tag) const { return (uint32_t)(w0 >> 32) == tag; }
  __device__ __forceinline__ float value() const { return __uint_as_float((uint32_t)w0); }
};
__device__ __forceinline__ void cp_async8(uint32_t dst_smem, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst_smem), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst_smem, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst_smem), "l"(src) : "memory");
}
__device__ __forceinline__ void async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// Consume a poll: spin (re-issue) until the tag matches.
template <typename T>
__device__ __forceinline__ T poll_take(TagPoll<T>& pl, const unsigned long long* src, uint32_t tag,
                                       int where, unsigned long long* stall = nullptr) {
  if (!pl.ok(tag)) {
    Watchdog wd;
    const unsigned long long t0 = kStepTrace ? gtime() : 0;
    do {
      pl.issue(src);
      wd.idle(where);
    } while (!pl.ok(tag));
    if (kStepTrace && stall) atomicAdd(stall, (1ull << 40) + (gtime() - t0));  // events, ns
  }
  return pl.value();
}

// Edge warp of K2 / K3: the 32 cross-tile cells of a tile, one lane each.
// Lane c < 16 polls the upstream neighbour in i (cell d = dPoll of row c) and
// publishes the own downstream cell of row c; lane 16 + c does the same in j.
// At step u (between the group barriers of steps u-1 and u) it publishes the
// value of step u-1 (s_val[(u-1) & 1][pub_pos], written by the tile's
// columns before barrier u-1) and deposits the polled value of step u+1 into
// s_rec[(u+1) & 1][lane], which the columns read after barrier u.  Polls are
// issued kPD - 1 steps before their deposit (ring q[v % kPD]): under full
// load an L2 round trip to a peer tile's words takes up to ~1 us.  Forward
// sweeps run plane k = u - d at step u, backward sweeps k = NS - 1 - u - d.
template <typename T>
struct EdgeLane {
  bool fwd, poll, pub;
  int d_poll, d_pub, pub_pos, NS, nz, lane;
  const unsigned long long* src;  // polled words of this lane's upstream cell (plane 0)
  unsigned long long* dst;        // published words of this lane's downstream cell
  __device__ __forceinline__ int k_of(int u, int dd) const { return fwd ? u - dd : (NS - 1 - u) - dd; }
};
// sync(u): the group barrier that ends step u (u = -1: the prologue barrier).
template <typename T, int kPD, typename Sync>
__device__ __forceinline__ void edge_warp_run(const EdgeLane<T>& e, const T (*s_val)[kTT], T (*s_rec)[32],
                                              unsigned epoch, Sync sync, unsigned long long* stall) {
  constexpr int TW = kTagWords<T>;
  TagPoll<T> q[kPD];
  auto issue = [&](TagPoll<T>& qq, int u) {
    const int k = e.k_of(u, e.d_poll);
    if (e.poll && u < e.NS && k >= 0 && k < e.nz) qq.issue(e.src + (long long)k * 16 * TW);
  };
  auto deposit = [&](TagPoll<T>& qq, int u) {
    const int k = e.k_of(u, e.d_poll);
    T v = T(0);
    if (e.poll && u < e.NS && k >= 0 && k < e.nz)
      v = poll_take(qq, e.src + (long long)k * 16 * TW, edge_tag(epoch, k), 64, stall);
    s_rec[u & 1][e.lane] = v;
  };
  auto publish = [&](int u) {
    const int k = e.k_of(u, e.d_pub);
    if (e.pub && u >= 0 && k >= 0 && k < e.nz)
      put_tagged(e.dst + (long long)k * 16 * TW, s_val[u & 1][e.pub_pos], edge_tag(epoch, k));
  };
#pragma unroll
  for (int v = 0; v < kPD; ++v) issue(q[v], v);
  deposit(q[0], 0);
  issue(q[0], kPD);
  sync(-1);  // prologue barrier: record of step 0 in place
  auto estep = [&](int u, TagPoll<T>& qq) {
    publish(u - 1);
    deposit(qq, u + 1);
    issue(qq, u + 1 + kPD);
    sync(u);
  };
  int u = 0;
  for (; u + kPD - 1 < e.NS; u += kPD) {
#pragma unroll
    for (int j = 0; j < kPD; ++j) estep(u + j, q[(j + 1) % kPD]);
  }
#pragma unroll
  for (int j = 0; j < kPD - 1; ++j)
    if (u + j < e.NS) estep(u + j, q[(j + 1) % kPD]);
  publish(e.NS - 1);
}

#if defined(SIPB_EXP_PD64)
constexpr int kPollK3 = SIPB_EXP_PD64, kPollK3f = 12;
#elif defined(SIPB_EXP_PD)
constexpr int kPollK3 = 8, kPollK3f = SIPB_EXP_PD;
#else
// K3 poll rings: issued kPoll - 1 steps ahead (tile step ~0.3 us fp64,
// ~0.2 us fp32 under load; an L2 round trip to a peer tile ~1 us)
constexpr int kPollK3 = 8, kPollK3f = 12;
#endif
constexpr int kPrep = 4;  // prepared-step ring between the residual and critical groups
constexpr int kRingR = 8; // phi-slice / record ring of the split K2 (two slices per iteration)
constexpr int kBarCrit = 1, kBarRes = 2, kBarFull = 3, kBarEmpty = kBarFull + kPrep;

// SYM: symmetric-system fast path (Listing 1; SURVEY.md
// 8(f) row 1): the residual reads AW / AS / AB of a cell as AE / AN / AT of its
// W / S / B neighbour -- the W / S values are the lines the neighbour threads
// stream one step earlier (L1 / L2 hits), AB is the thread's own AT of the
// plane below -- so the AW, AS and AB arrays are not streamed from HBM (11
// instead of 14 array touches per cell).  The coefficient values, hence every
// operation and its rounding, are the general path's (the symmetry invariant
// is checked exactly by sip_set_symmetric).
// fp32 general path: the critical group's cross-tile polls / publishes run in
// an edge warp (threads 512..543, edge_warp_run) -- 6 % faster at 256^3.  fp64
// and the symmetric path keep them in the critical threads: a 17th warp caps
// the kernel at 96 registers (fp64: the residual group spills; fp32 SYM:
// measured 6 % slower).
template <typename T, bool SYM>
__host__ __device__ constexpr bool k2_edge_warp() { return sizeof(T) == 4 && !SYM; }
#ifdef SIPB_EXP_PD2
constexpr int kPollK2 = SIPB_EXP_PD2;
#else
constexpr int kPollK2 = 2;  // K2 edge-warp poll ring (tile step ~0.5-0.9 us; 2: -1 % vs 3)
#endif

template <typename T, bool SYM>
__global__ void __launch_bounds__(2 * kTT + (k2_edge_warp<T, SYM>() ? 32 : 0), 1)
    k_forward(const SweepParams<T> P) {
  // Two threads per column.  Threads 0..255 ("critical"): the recurrence
  // R = (((r - LB*R_B) - LW*R_W) - LS*R_S) * LP of step t, cross-tile R
  // stores / polls (fp32: done by the edge warp, see k2_edge_warp).
  // Threads 256..511 ("residual"): everything that does
  // not depend on R -- the residual r of each step and its factors (handed
  // over through the s_prep ring of kPrep slots), the phi / edge-record
  // rings, the forward-pack LDGs and the L2 prefetch front.  The two groups
  // are decoupled by named barriers (producer/consumer FULL / EMPTY per prep
  // slot), so the residual group runs up to kPrep steps ahead; each group
  // meets only itself once per step (its own shared-ring exchange).
  __shared__ __align__(16) T s_ph[kRingR][kTT];  // own-column phi of slice y in slot y % kRingR
  __shared__ __align__(16) T s_rec[kRingR][64];  // static edge record of step y (phiW/E/S/N)
  __shared__ __align__(16) T s_R[2][kTT];       // R of steps t-1 / t
  __shared__ __align__(16) T s_eR[2][32];       // edge warp: polled R of the W column / S row
  __shared__ __align__(16) T s_gh[2][kTT];      // ghost phi below / above each column
  __shared__ __align__(16) T s_prep[kPrep][kTT];  // residual r of prepared steps
  __shared__ double s_red[2 * kTT / 32 + 1];
  constexpr bool kEdge = k2_edge_warp<T, SYM>();
  constexpr int kCritBar = kTT + (kEdge ? 32 : 0);  // critical-group barrier (+ edge warp)
  // FULL(slot of step t): residual threads arrive when r(t) is in s_prep; the
  // critical threads (and the edge warp) sync on it at the end of step t-1,
  // so one barrier both publishes R(t-1) to the group and admits step t
  constexpr int kFullBar = 2 * kTT + (kEdge ? 32 : 0);
  __shared__ int s_tile, s_last;
  __shared__ unsigned long long s_stall;  // debug (SIPB_STEP_TRACE): poll stalls of the tile
  constexpr int TW = kTagWords<T>;

  const int p = threadIdx.x;
  const bool crit = p < kTT, edgew = p >= 2 * kTT;
  const int q = p & (kTT - 1);  // column position
  int ti, tj;
  pos_to_tij(q, ti, tj);
  const int d = ti + tj;
  const int pW = ti > 0 ? tile_pos(ti - 1, tj) : q;
  const int pE = ti < kTI - 1 ? tile_pos(ti + 1, tj) : q;
  const int pS = tj > 0 ? tile_pos(ti, tj - 1) : q;
  const int pN = tj < kTJ - 1 ? tile_pos(ti, tj + 1) : q;
  const unsigned epoch = *P.epoch;  // stable for this launch (bumped by the finaliser)

  for (;;) {
    __syncthreads();
    if (p == 0) {
      s_tile = atomicAdd(P.state, 1u);
      s_stall = 0;
    }
    __syncthreads();
    const int tk = s_tile;
    if (tk >= P.ntiles) break;
    const int tid = P.order[tk];
    const TileDesc td = P.tiles[tid];
    const BlockDesc bd = P.blocks[td.block];
    const int NS = td.ns, nz = td.nz;
    if (P.trace && p == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      P.trace[4 * tid + 0] = gtime();
      P.trace[4 * tid + 2] = smid;
      P.trace[4 * tid + 3] = blockIdx.x;
    }
    const bool col = ti < td.wI && tj < td.wJ;
    const bool inW = ti > 0, inE = ti + 1 < td.wI, inS = tj > 0, inN = tj + 1 < td.wJ;
    double nrm = 0.0;
    if (crit) {
      // ------------------------------------------------------------ critical
      const bool pollW = col && ti == 0 && td.nW >= 0, pollS = col && tj == 0 && td.nS >= 0;
      const bool pubE = col && ti == kTI - 1 && td.nE >= 0, pubN = col && tj == kTJ - 1 && td.nN >= 0;
      const unsigned long long* srcW = P.tagA + ((pollW ? P.tiles[td.nW].edge : 0) + tj) * TW;
      const unsigned long long* srcS = P.tagB + ((pollS ? P.tiles[td.nS].edge : 0) + ti) * TW;
      unsigned long long* dstE = P.tagA + (td.edge + tj) * TW;
      unsigned long long* dstN = P.tagB + (td.edge + ti) * TW;
      T* gR = P.R + td.slot * kTT + q;
      auto poll_issue = [&](TagPoll<T>& pw, TagPoll<T>& ps, int s) {
        const int k = s - d;
        if (!kEdge && k >= 0 && k < nz && s < NS) {
          if (pollW) pw.issue(srcW + (long long)k * 16 * TW);
          if (pollS) ps.issue(srcS + (long long)k * 16 * TW);
        }
      };
      TagPoll<T> pw0, ps0, pw1, ps1;  // R polls of even / odd steps
      poll_issue(pw0, ps0, 0);
      poll_issue(pw1, ps1, 1);
      // own factor coefficients LB, LW, LS, LP, LDG'd two steps ahead
      const T* lf_cell = P.fw + td.slot * F_NA * kTT + F_LB * kTT + q;
      auto ldg_lf = [&](T* lf, int s) {
        const int k = s - d;
        if (s < NS && col && k >= 0 && k < nz) {
          const T* src = lf_cell + (long long)s * F_NA * kTT;
#pragma unroll
          for (int a = 0; a < 4; ++a) lf[a] = __ldg(src + a * kTT);
        }
      };
      T lf0[4] = {T(0), T(0), T(0), T(0)}, lf1[4] = {T(0), T(0), T(0), T(0)};
      ldg_lf(lf0, 0);
      ldg_lf(lf1, 1);
      nbar_sync(kBarFull, kFullBar);  // prologue: step 0 prepared (and its edge record in place)
      T RB = T(0);  // own R of the plane below (0 outside the block)
      auto iter = [&](const int t, TagPoll<T>& pw, TagPoll<T>& ps, T* lf) {
        const int k = t - d;
        const int sl = t & (kPrep - 1);
        if (kStepTrace && P.trace && p == 0 && tid == P.trace_tile)
          P.trace[8 * P.ntiles + 16 * t + 7] = gtime();  // slot 7: step t starts (tile A, thread 0)
        const T r = s_prep[sl][q];  // step t prepared (FULL barrier that ended step t-1)
        const T lb = lf[0], lw = lf[1], ls = lf[2], lp = lf[3];
        if (t + kPrep < NS) nbar_arrive(kBarEmpty + sl, 2 * kTT);  // slot free for step t + kPrep
        const T RWi = s_R[(t - 1) & 1][pW], RSi = s_R[(t - 1) & 1][pS];
        if (col && k >= 0 && k < nz) {
          const uint32_t tag = edge_tag(epoch, k);
          T RW, RS;
          if constexpr (kEdge) {
            RW = inW ? RWi : s_eR[t & 1][tj];  // 0 at a block face
            RS = inS ? RSi : s_eR[t & 1][16 + ti];
          } else {
            RW = inW ? RWi : (pollW ? poll_take(pw, srcW + (long long)k * 16 * TW, tag, 61, &s_stall) : T(0));
            RS = inS ? RSi : (pollS ? poll_take(ps, srcS + (long long)k * 16 * TW, tag, 62, &s_stall) : T(0));
          }
          const T Rv = (((r - lb * RB) - lw * RW) - ls * RS) * lp;
          RB = Rv;
          s_R[t & 1][q] = Rv;
          if (!kEdge && pubE) put_tagged(dstE + (long long)k * 16 * TW, Rv, tag);
          if (!kEdge && pubN) put_tagged(dstN + (long long)k * 16 * TW, Rv, tag);
#ifndef SIPB_EXP_NOSTG
          gR[(long long)t * kTT] = Rv;  // consumed only by K3 (next launch)
#endif
        }
        poll_issue(pw, ps, t + 2);
        ldg_lf(lf, t + 2);
        if (kStepTrace && P.trace && p == 0 && (tid == P.trace_tile || tid == P.trace_tile + 1))
          P.trace[8 * P.ntiles + 16 * t + (tid - P.trace_tile)] = gtime();  // slots 0, 1: tiles A, B
        // R of step t visible to the group (and the edge warp); step t+1 prepared
        if (t + 1 < NS)
          nbar_sync(kBarFull + ((t + 1) & (kPrep - 1)), kFullBar);
        else
          nbar_sync(kBarCrit, kCritBar);
      };
      int t = 0;
      for (; t + 1 < NS; t += 2) {
        iter(t, pw0, ps0, lf0);
        iter(t + 1, pw1, ps1, lf1);
      }
      if (t < NS) iter(t, pw0, ps0, lf0);
    } else if (edgew) {
      if constexpr (kEdge) {
        // ---------------------------------------------------------- edge warp
        // lane c < 16: poll the W tile's E column (cell (0, c) here), publish
        // cell (15, c); lane 16 + c: S tile's N row (cell (c, 0)), publish (c, 15)
        const int lane = p & 31, c = lane & 15;
        const bool wi = lane < 16;
        EdgeLane<T> e;
        const int nPoll = wi ? td.nW : td.nS, nPub = wi ? td.nE : td.nN;
        const bool colok = wi ? (c < td.wJ) : (c < td.wI);
        const bool full = wi ? (td.wI == kTI) : (td.wJ == kTJ);  // the published cell exists
        e.fwd = true;
        e.poll = colok && nPoll >= 0;
        e.pub = colok && full && nPub >= 0;
        e.d_poll = c;
        e.d_pub = c + (wi ? kTI - 1 : kTJ - 1);
        e.pub_pos = wi ? tile_pos(kTI - 1, c) : tile_pos(c, kTJ - 1);
        e.NS = NS;
        e.nz = nz;
        e.lane = lane;
        e.src = (wi ? P.tagA : P.tagB) + ((e.poll ? P.tiles[nPoll].edge : 0) + c) * TW;
        e.dst = (wi ? P.tagA : P.tagB) + (td.edge + c) * TW;
        edge_warp_run<T, kPollK2>(
            e, s_R, s_eR, epoch,
            [&](int u) {
              if (u + 1 < NS)
                nbar_sync(kBarFull + ((u + 1) & (kPrep - 1)), kFullBar);
              else
                nbar_sync(kBarCrit, kCritBar);
            },
            &s_stall);
      }
    } else {
      // ------------------------------------------------------------ residual
      // Two steps per iteration (two independent residual chains interleave,
      // one group barrier per two steps).  Iteration m prepares steps 2m+1
      // and 2m+2, refills ring slices 2m+4 and 2m+5 (ring of kRingR slots).
      const int rW = tj, rE = 16 + tj, rS = 32 + ti, rN = 48 + ti;
      {
        const int gi = td.i0 + ti, gj = td.j0 + tj;
        T gb = T(0), gt = T(0);
        if (col) {
          gb = P.ghost[ghost_face_offset(bd, G_B) + gi + (long long)bd.nx * gj];
          gt = P.ghost[ghost_face_offset(bd, G_T) + gi + (long long)bd.nx * gj];
        }
        s_gh[0][q] = gb;
        s_gh[1][q] = gt;
      }
      const T* fw_cell = P.fw + td.slot * F_NA * kTT + q;
      const T* ph_cell = P.phi + td.slot * kTT + q;
      const T* rp_cell = P.rec_phi + td.slot * 64 + (q & 63);
      // SYM: per-thread bases, linear in the step x, of the W neighbour's AE
      // and the S neighbour's AN (in-tile: slice x-1; neighbour tile: its edge
      // cell, slice x+15; block boundary: own AW / AS, equal by symmetry)
      constexpr long long kSl = (long long)F_NA * kTT;
      const T* symW = fw_cell;
      const T* symS = fw_cell;
      if (SYM) {
        symW = ti > 0 ? P.fw + (td.slot - 1) * kSl + F_AE * kTT + pW
               : td.nW >= 0 ? P.fw + (P.tiles[td.nW].slot + kTI - 1) * kSl + F_AE * kTT + tile_pos(kTI - 1, tj)
                            : fw_cell + F_AW * kTT;
        symS = tj > 0 ? P.fw + (td.slot - 1) * kSl + F_AN * kTT + pS
               : td.nS >= 0 ? P.fw + (P.tiles[td.nS].slot + kTJ - 1) * kSl + F_AN * kTT + tile_pos(ti, kTJ - 1)
                            : fw_cell + F_AS * kTT;
      }
      auto ldg_fw = [&](T* nf, int x) {  // the 8 residual coefficients (AP .. AT, Q)
        const int k = x - d;
        if (x < NS && col && k >= 0 && k < nz) {
          const T* src = fw_cell + (long long)x * F_NA * kTT;
#ifdef SIPB_EXP_NOLDG
#pragma unroll
          for (int a = 0; a < F_LB; ++a) nf[a] = T(0.01) * T(a + 1) + T(x) * T(1e-9);
          (void)src;
#else
          if (SYM) {
            nf[F_AP] = __ldg(src + F_AP * kTT);
            nf[F_AE] = __ldg(src + F_AE * kTT);
            nf[F_AN] = __ldg(src + F_AN * kTT);
            nf[F_AT] = __ldg(src + F_AT * kTT);
            nf[F_Q] = __ldg(src + F_Q * kTT);
            nf[F_AW] = __ldg(symW + (long long)x * kSl);
            nf[F_AS] = __ldg(symS + (long long)x * kSl);
            if (k == 0) nf[F_AB] = __ldg(src + F_AB * kTT);  // else: own AT of the plane below
          } else {
#pragma unroll
            for (int a = 0; a < F_LB; ++a) nf[a] = __ldg(src + a * kTT);
          }
#endif
        }
      };
      auto ldg_phi = [&](int y) -> T {
        const int k = y - d;
        return (y < NS && col && k >= 0 && k < nz) ? __ldg(ph_cell + (long long)y * kTT) : T(0);
      };
      auto ldg_rec = [&](int y) -> T { return (y < NS && q < 64) ? __ldg(rp_cell + (long long)y * 64) : T(0); };
      // residual of step x (Listing-1 term order, a_nb = -A_nb)
      auto residual = [&](const T* nf, T fP, T fB, T fT, T fW, T fE, T fS, T fN) {
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
      auto publish = [&](int x, T rr) {  // hand the residual of step x to the critical group
        const int sl = x & (kPrep - 1);
        if (x >= kPrep) nbar_sync(kBarEmpty + sl, 2 * kTT);  // step x - kPrep consumed
        s_prep[sl][q] = rr;
        if (kStepTrace && P.trace && q == 0 && tid == P.trace_tile)
          P.trace[8 * P.ntiles + 16 * x + 6] = gtime();  // slot 6: residual of step x published (tile A)
        nbar_arrive(kBarFull + sl, kFullBar);
      };
      constexpr int kFwLines = F_NA * kTT * (int)sizeof(T) / 128, kPhLines = kTT * (int)sizeof(T) / 128;
      constexpr int kArrLines = kTT * (int)sizeof(T) / 128;  // lines per array slice
      // SYM: the AW / AS / AB lines are never loaded, so not prefetched either
      const bool pf_skip = SYM && q < kFwLines &&
                           ((q / kArrLines) == F_AW || (q / kArrLines) == F_AS || (q / kArrLines) == F_AB);
      auto pf_step = [&](int x) {  // L2 prefetch front: one 128-byte line per thread
        if (x >= NS || pf_skip) return;
        if (q < kFwLines)
          prefetch_line_l2(reinterpret_cast<const char*>(P.fw + (td.slot + x) * F_NA * kTT) + 128 * q);
        else if (q < kFwLines + kPhLines)
          prefetch_line_l2(reinterpret_cast<const char*>(P.phi + (td.slot + x) * kTT) + 128 * (q - kFwLines));
      };
      // operands of the residual of step x from ring slots of slices x-1, x, x+1
      struct Ops { T fP, fB, fT, fW, fE, fS, fN; };
      auto load_ops = [&](int x) {
        Ops o;
        const int k1 = x - d;
        const int sm = (x - 1) & (kRingR - 1), s0 = x & (kRingR - 1), sp = (x + 1) & (kRingR - 1);
        const int rr = x & (kRingR - 1);
        o.fP = s_ph[s0][q];
        o.fB = k1 > 0 ? s_ph[sm][q] : s_gh[0][q];
        o.fT = k1 + 1 < nz ? s_ph[sp][q] : s_gh[1][q];
        o.fW = inW ? s_ph[sm][pW] : s_rec[rr][rW];
        o.fE = inE ? s_ph[sp][pE] : s_rec[rr][rE];
        o.fS = inS ? s_ph[sm][pS] : s_rec[rr][rS];
        o.fN = inN ? s_ph[sp][pN] : s_rec[rr][rN];
        return o;
      };
      auto active = [&](int x) { const int k1 = x - d; return x < NS && col && k1 >= 0 && k1 < nz; };
      // ---- prologue: slices / records 0..3 into the ring, 4..7 in flight
      for (int y = 0; y < 4; ++y) {
        s_ph[y][q] = ldg_phi(y);
        if (q < 64) s_rec[y][q] = ldg_rec(y);
      }
      T phA[2] = {ldg_phi(4), ldg_phi(5)}, phB[2] = {ldg_phi(6), ldg_phi(7)};
      T rcA[2] = {ldg_rec(4), ldg_rec(5)}, rcB[2] = {ldg_rec(6), ldg_rec(7)};
      T nfO[F_LB], nfE[F_LB];  // residual coefficients of odd / even steps
#pragma unroll
      for (int a = 0; a < F_LB; ++a) nfO[a] = nfE[a] = T(0);
      ldg_fw(nfE, 0);
      ldg_fw(nfO, 1);
      for (int x = 0; x <= kPFL; ++x) pf_step(x + 8);
      nbar_sync(kBarRes, kTT);  // prologue: ring filled
      T atPrev = T(0);  // SYM: own AT of the last prepared step (= AB of the next plane)
      {
        const Ops o = load_ops(0);
        const T rr = residual(nfE, o.fP, o.fB, o.fT, o.fW, o.fE, o.fS, o.fN);
        if (active(0)) nrm += fabs(static_cast<double>(rr));
        publish(0, rr);
        atPrev = nfE[F_AT];
      }
      ldg_fw(nfE, 2);
      auto iter = [&](const int m, T* phb, T* rcb) {
        const int x0 = 2 * m + 1, x1 = x0 + 1;
        const Ops o0 = load_ops(x0);
        const Ops o1 = load_ops(x1);
        if (SYM) {
          if (x0 - d != 0) nfO[F_AB] = atPrev;
          if (x1 - d != 0) nfE[F_AB] = nfO[F_AT];
          atPrev = nfE[F_AT];
        }
        const T r0 = residual(nfO, o0.fP, o0.fB, o0.fT, o0.fW, o0.fE, o0.fS, o0.fN);
        const T r1 = residual(nfE, o1.fP, o1.fB, o1.fT, o1.fW, o1.fE, o1.fS, o1.fN);
        if (active(x0)) nrm += fabs(static_cast<double>(r0));
        if (active(x1)) nrm += fabs(static_cast<double>(r1));
        if (x0 < NS) publish(x0, r0);
        if (x1 < NS) publish(x1, r1);
        ldg_fw(nfO, x0 + 2);  // consumed above
        ldg_fw(nfE, x1 + 2);
        // refill: slices / records 2m+4, 2m+5 (slots of slices 2m-4, 2m-3, last read in iteration m-2)
        const int y = 2 * m + 4;
        s_ph[y & (kRingR - 1)][q] = phb[0];
        s_ph[(y + 1) & (kRingR - 1)][q] = phb[1];
        if (q < 64) {
          s_rec[y & (kRingR - 1)][q] = rcb[0];
          s_rec[(y + 1) & (kRingR - 1)][q] = rcb[1];
        }
        phb[0] = ldg_phi(y + 4);
        phb[1] = ldg_phi(y + 5);
        rcb[0] = ldg_rec(y + 4);
        rcb[1] = ldg_rec(y + 5);
        pf_step(y + 4 + kPFL);
        pf_step(y + 5 + kPFL);
        nbar_sync(kBarRes, kTT);  // ring slices 2m+4, 2m+5 visible to the group
      };
      // iterations m while 2m+1 < NS
      int m = 0;
      for (; 2 * m + 3 < NS; m += 2) {
        iter(m, phA, rcA);
        iter(m + 1, phB, rcB);
      }
      if (2 * m + 1 < NS) iter(m, phA, rcA);
    }

    if (P.trace && p == 0) P.trace[4 * tid + 1] = gtime();
    if (kStepTrace && P.trace) {
      __syncthreads();
      if (p == 0) P.trace[4 * tid + 3] = s_stall;  // (events << 40) + stalled ns
    }
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
      const unsigned it = *P.norm_it;  // iteration index (written by the previous launch)
      double* bnorms = P.bnorms_base + (size_t)it * P.nblocks;
      const int warp = p >> 5, nw = blockDim.x >> 5;
      for (int b = warp; b < P.nblocks; b += nw) {
        const BlockDesc bb = P.blocks[b];
        double v = 0.0;
        for (int x2 = (p & 31); x2 < bb.ntiles; x2 += 32) v += __ldcg(P.partial + bb.tile0 + x2);
#pragma unroll
        for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if ((p & 31) == 0) bnorms[b] = v;
      }
      __syncthreads();
      if (p == 0) {
        double v = 0.0;
        for (int b = 0; b < P.nblocks; ++b) v += bnorms[b];
        P.norms_base[it] = v;
        *P.norm_it = it + 1;
      }
      for (int x2 = p; x2 < kProgOff + P.ntiles; x2 += blockDim.x) P.state_other[x2] = 0u;
      if (p == 0) *P.epoch = epoch + 1;
    }
  }
}

// =============================================================================
// K3: backward substitution + phi update (backward3d); slices in reverse.
// delta = ((R - UN*dN) - UE*dE) - UT*dT with R, phi, UN, UE, UT LDG'd two
// steps ahead, dN / dE from the previous step's shared delta or polled from
// the E / N neighbour tiles (their W column / S row, tagged).
// =============================================================================
template <typename T>
__global__ void __launch_bounds__(kTT + 32, 1) k_backward(const SweepParams<T> P) {
  // threads 0..255: one per tile column, no cross-tile code at all;
  // warp 8 ("edge warp"): publishes the tile's W column / S row delta one
  // step after it is computed and polls the E / N neighbours' values three
  // steps ahead, depositing each step's 32 edge values into s_rec before the
  // columns need them.  All 288 threads meet at one barrier per step.
  __shared__ __align__(16) T s_D[2][kTT];
  __shared__ __align__(16) T s_rec[2][32];  // [step & 1]: dE (c < 16), dN (16 + c)
  // own R, phi, UN, UE, UT of steps u % 4, copied 4 steps ahead with
  // cp.async (under full load the HBM latency exceeds two tile steps; a
  // register double buffer measured slower, 8 steps no faster)
  constexpr int kNbD = 4;  // cp.async depth (steps)
  __shared__ __align__(16) T s_nb[kNbD][5][kTT];
  __shared__ int s_tile, s_last;
  __shared__ unsigned long long s_stall;  // debug (SIPB_STEP_TRACE): poll stalls of the tile
  constexpr int TW = kTagWords<T>;

  const int p = threadIdx.x;
  const bool edge_warp = p >= kTT;
  const int lane = p & 31;
  int ti = 0, tj = 0;
  if (!edge_warp) pos_to_tij(p, ti, tj);
  const int d = ti + tj;
  const int pE = ti < kTI - 1 ? tile_pos(ti + 1, tj) : p;
  const int pN = tj < kTJ - 1 ? tile_pos(ti, tj + 1) : p;
  const unsigned epoch = *P.epoch;

  for (;;) {
    __syncthreads();
    if (p == 0) {
      s_tile = atomicAdd(P.state, 1u);
      s_stall = 0;
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
    if (edge_warp) {
      // ------------------------------------------------------------ edge warp
      // lane c < 16: poll the E tile's W column (cell (15, c) here), publish
      // cell (0, c); lane 16 + c: N tile's S row (cell (c, 15)), publish (c, 0)
      EdgeLane<T> e;
      const bool we = lane < 16;
      const int c = lane & 15;
      const bool colok = we ? (c < td.wJ) : (c < td.wI);
      const int nPoll = we ? td.nE : td.nN, nPub = we ? td.nW : td.nS;
      e.fwd = false;
      e.poll = colok && nPoll >= 0;
      e.pub = colok && nPub >= 0;
      e.d_poll = we ? (kTI - 1) + c : c + (kTJ - 1);
      e.d_pub = c;
      e.pub_pos = we ? tile_pos(0, c) : tile_pos(c, 0);
      e.NS = NS;
      e.nz = nz;
      e.lane = lane;
      e.src = (we ? P.tagA : P.tagB) + ((e.poll ? P.tiles[nPoll].edge : 0) + c) * TW;
      e.dst = (we ? P.tagA : P.tagB) + (td.edge + c) * TW;
      edge_warp_run<T, sizeof(T) == 8 ? kPollK3 : kPollK3f>(
          e, s_D, s_rec, epoch, [](int) { nbar_sync(1, kTT + 32); }, &s_stall);
    } else {
    // -------------------------------------------------------------- columns
    const bool col = ti < td.wI && tj < td.wJ;
    const bool inE = ti + 1 < td.wI, inN = tj + 1 < td.wJ;
    const T* r_cell = P.R + td.slot * kTT + p;
    T* ph_cell = P.phi + td.slot * kTT + p;
    const T* bw_cell = P.bw + td.slot * B_NA * kTT + p;
    auto pf = [&](int u) {  // three bulk L2 prefetches (R, phi, U slices of step u), thread 0
      if (u >= NS || p != 0) return;
      const long long ts = td.slot + NS - 1 - u;
      prefetch_l2(P.R + ts * kTT, kTT * sizeof(T));
      prefetch_l2(P.phi + ts * kTT, kTT * sizeof(T));
      prefetch_l2(P.bw + ts * B_NA * kTT, B_NA * kTT * sizeof(T));
    };
    T nb0[5], nb1[5];  // R, phi, UN, UE, UT of even / odd steps
#pragma unroll
    for (int a = 0; a < 5; ++a) nb0[a] = nb1[a] = T(0);
    auto acp = [&](int xs) {
      const int ts = NS - 1 - xs, k2 = ts - d;
      if (xs < NS && col && k2 >= 0 && k2 < nz) {
        const T* srcs[5] = {r_cell + (long long)ts * kTT, ph_cell + (long long)ts * kTT,
                            bw_cell + (long long)ts * B_NA * kTT, bw_cell + (long long)ts * B_NA * kTT + kTT,
                            bw_cell + (long long)ts * B_NA * kTT + 2 * kTT};
#pragma unroll
        for (int a = 0; a < 5; ++a) {
          if (sizeof(T) == 8) cp_async8(saddr(&s_nb[xs & (kNbD - 1)][a][p]), srcs[a]);
          else cp_async4(saddr(&s_nb[xs & (kNbD - 1)][a][p]), srcs[a]);
        }
      }
      async_commit();
    };
    for (int x = 0; x < kNbD; ++x) acp(x);
    for (int u = 0; u < kNbD + 3; ++u) pf(u);
    nbar_sync(1, kTT + 32);  // prologue barrier (edge record of step 0)
    T dT = T(0);  // own delta of the plane above (0 outside the block)
    auto iter = [&](const int u, T* nb) {
      const int t = NS - 1 - u, k = t - d;
      async_wait<kNbD - 1>();  // this thread's copies of step u (issued kNbD iterations ago) landed
#pragma unroll
      for (int a = 0; a < 5; ++a) nb[a] = s_nb[u & (kNbD - 1)][a][p];
      // in-tile neighbours from the previous step, tile-edge ones from the edge record
      const T dN = inN ? s_D[(u - 1) & 1][pN] : s_rec[u & 1][16 + ti];
      const T dE = inE ? s_D[(u - 1) & 1][pE] : s_rec[u & 1][tj];
      if (col && k >= 0 && k < nz) {
        const T utdt = nb[4] * dT;
        const T dl = ((nb[0] - nb[2] * dN) - nb[3] * dE) - utdt;
        dT = dl;
        s_D[u & 1][p] = dl;
#ifndef SIPB_EXP_NOSTG
        ph_cell[(long long)t * kTT] = nb[1] + dl;
#endif
      }
      acp(u + kNbD);  // into the slot just consumed
      pf(u + kNbD + 3);  // L2 prefetch three steps beyond the copies
      if (kStepTrace && P.trace && p == 0 && (tid == P.trace_tile || tid == P.trace_tile - 1))
        P.trace[8 * P.ntiles - 4 * P.ntiles + 16 * u + 2 + (P.trace_tile - tid)] = gtime();  // K3 slots 2, 3
      nbar_sync(1, kTT + 32);
    };
    int u = 0;
    for (; u + 1 < NS; u += 2) {
      iter(u, nb0);
      iter(u + 1, nb1);
    }
    if (u < NS) iter(u, nb0);
    }  // columns

    if (P.trace && p == 0) P.trace[4 * tid + 1] = gtime();
    if (kStepTrace && P.trace) {
      __syncthreads();
      if (p == 0) P.trace[4 * tid + 3] = s_stall;  // (events << 40) + stalled ns
    }
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
__global__ void __launch_bounds__(1024) k_edge_phi(const SweepParams<T> P) {
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
#pragma unroll 4
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
    const unsigned cu = (unsigned)c, r = cu / (unsigned)bd.nx;  // blocks < 2^32 cells
    const int i = (int)(cu - r * (unsigned)bd.nx), j = (int)(r % (unsigned)bd.ny), k = (int)(r / (unsigned)bd.ny);
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
    const unsigned cu = (unsigned)c, r = cu / (unsigned)bd.nx;  // blocks < 2^32 cells
    const int i = (int)(cu - r * (unsigned)bd.nx), j = (int)(r % (unsigned)bd.ny), k = (int)(r / (unsigned)bd.ny);
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
    const unsigned cu = (unsigned)c, r = cu / (unsigned)bd.nx;  // blocks < 2^32 cells
    const int i = (int)(cu - r * (unsigned)bd.nx), j = (int)(r % (unsigned)bd.ny), k = (int)(r / (unsigned)bd.ny);
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
// residual_general or, with SYM, residual_symmetric
// (Listing PAPER.md:503-518): the W / S / B couplings are
// read as the E / N / T coefficients of the W / S / B neighbour cell (5
// coefficient arrays instead of 8); at the block's first interior cell the
// neighbour is the ghost cell, whose AE (AN, AT) equals this cell's AW (AS,
// AB) by the symmetry invariant, so AW (AS, AB) is read there.
template <typename T, bool SYM>
__global__ void k_residual(const BlockDesc* blocks, int b, const T* __restrict__ fw,
                           const T* __restrict__ phi, const T* __restrict__ ghost, double* out) {
  const BlockDesc bd = blocks[b];
  const long long n = (long long)bd.nx * bd.ny * bd.nz;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    const unsigned cu = (unsigned)c, r = cu / (unsigned)bd.nx;  // blocks < 2^32 cells
    const int i = (int)(cu - r * (unsigned)bd.nx), j = (int)(r % (unsigned)bd.ny), k = (int)(r / (unsigned)bd.ny);
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

// Symmetry invariant of a StencilSystem on the fp64 pack:
// AE(i) == AW(i+1), AN(j) == AS(j+1), AT(k) == AB(k+1) exactly; counts violations.
__global__ void k_check_symmetric(const BlockDesc* blocks, int b, const double* __restrict__ fw,
                                  unsigned long long* bad) {
  const BlockDesc bd = blocks[b];
  const long long n = (long long)bd.nx * bd.ny * bd.nz;
  unsigned long long cnt = 0;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    const unsigned cu = (unsigned)c, r = cu / (unsigned)bd.nx;  // blocks < 2^32 cells
    const int i = (int)(cu - r * (unsigned)bd.nx), j = (int)(r % (unsigned)bd.ny), k = (int)(r / (unsigned)bd.ny);
    if (i + 1 < bd.nx && fw[pack_index(bd, F_NA, F_AE, i, j, k)] != fw[pack_index(bd, F_NA, F_AW, i + 1, j, k)]) ++cnt;
    if (j + 1 < bd.ny && fw[pack_index(bd, F_NA, F_AN, i, j, k)] != fw[pack_index(bd, F_NA, F_AS, i, j + 1, k)]) ++cnt;
    if (k + 1 < bd.nz && fw[pack_index(bd, F_NA, F_AT, i, j, k)] != fw[pack_index(bd, F_NA, F_AB, i, j, k + 1)]) ++cnt;
  }
  if (cnt) atomicAdd(bad, cnt);
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

int launch_factor(const FactorParams& p, int grid, void* stream) {
  k_factor<<<grid, kTT, 0, (cudaStream_t)stream>>>(p);
  return cuda_status(cudaGetLastError());
}

template <typename T>
int launch_forward(const SweepParams<T>& p, int grid, void* stream) {
  // The symmetric fast path (identical values, identical rounding) saves HBM
  // reads; it pays in fp64 (1.4 % at 256^3) but not in fp32, whose forward
  // sweep is latency- rather than bandwidth-bound (the neighbour-line reads
  // lengthen the residual chain: 6.9 % slower), so fp32 always runs the
  // general kernel.
  if constexpr (sizeof(T) == 8) {
    if (p.symmetric) {
      k_forward<T, true><<<grid, 2 * kTT, 0, (cudaStream_t)stream>>>(p);
      return cuda_status(cudaGetLastError());
    }
  }
  k_forward<T, false><<<grid, 2 * kTT + (k2_edge_warp<T, false>() ? 32 : 0), 0, (cudaStream_t)stream>>>(p);
  return cuda_status(cudaGetLastError());
}

template <typename T>
int launch_backward(const SweepParams<T>& p, int grid, void* stream) {
  k_backward<T><<<grid, kTT + 32, 0, (cudaStream_t)stream>>>(p);
  return cuda_status(cudaGetLastError());
}

template <typename T>
int launch_edge_phi(const SweepParams<T>& p, void* stream) {
  if (p.ntiles <= 0) return SIP_OK;
  k_edge_phi<T><<<p.ntiles, 1024, 0, (cudaStream_t)stream>>>(p);
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
    e = precision == SIP_PREC_DOUBLE
            ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_forward<double, false>, 2 * kTT, 0)
            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_forward<float, false>, 2 * kTT + 32, 0);
  } else {
    e = precision == SIP_PREC_DOUBLE
            ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_backward<double>, kTT + 32, 0)
            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_backward<float>, kTT + 32, 0);
    // one tile per SM: a second co-resident tile halves both tiles' pace
    // (the sweep is step-latency bound) -- measured 4-8 % faster at 256^3
    per = per > 0 ? 1 : per;
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
  const int g = grid_for((long long)hb.nx * hb.ny * hb.nz);
  if (symmetric)
    k_residual<T, true><<<g, 256, 0, (cudaStream_t)stream>>>(d_blocks, block, fw, phi, ghost, out);
  else
    k_residual<T, false><<<g, 256, 0, (cudaStream_t)stream>>>(d_blocks, block, fw, phi, ghost, out);
  return cuda_status(cudaGetLastError());
}
int launch_check_symmetric(const BlockDesc* d_blocks, int block, const BlockDesc& hb,
                           const double* fw, unsigned long long* bad, void* stream) {
  k_check_symmetric<<<grid_for((long long)hb.nx * hb.ny * hb.nz), 256, 0, (cudaStream_t)stream>>>(
      d_blocks, block, fw, bad);
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
