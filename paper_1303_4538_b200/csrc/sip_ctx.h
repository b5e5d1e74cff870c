// sip_ctx.h -- the library context behind the opaque sip_ctx handle and the
// host helpers shared by the C-ABI translation units (sip_api.cu: system,
// factor, sweep and halo entry points; sip_flow.cu: the pressure-correction
// caller).  Host code only.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <array>
#include <string>
#include <tuple>
#include <vector>

#include "sip_internal.h"

namespace sipb {

// NCCL is resolved at run time (dlopen), only when a multi-rank lattice is
// built: a host process that already loaded an NCCL (e.g. torch's bundled
// libnccl.so.2) shares it, and single-GPU use needs no NCCL at all.
struct NcclApi {
  bool ok = false;
  std::string err;
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};
NcclApi& nccl();

struct Peer {
  int rank = -1;
  std::vector<FaceCopy> pack, unpack;  // plane -> send buffer, recv buffer -> ghost
  long long count = 0;                 // elements each way
  FaceCopy* d_pack = nullptr;
  FaceCopy* d_unpack = nullptr;
  void* sbuf = nullptr;  // into sip_ctx::x_sbuf / x_rbuf at soff / roff
  void* rbuf = nullptr;
  int max_plane = 0;
  // SIP exchange: the first s1 (r1) elements of the message are the early
  // (E / N / T source plane) transfers, sent in phase 1
  long long soff = 0, roff = 0, s1 = 0, r1 = 0;
};
// One pending sip_solve_async: its norms (pinned host copy, delivered to
// `out` when it completes), the caller's phi buffers and one event per
// downloaded chunk of each (the next solve's upload of the same buffer
// follows them chunk by chunk).
constexpr int kAsyncChunks = 8;
struct AsyncSolve {
  int iters = 0;
  double* out = nullptr;
  double* h_norms = nullptr;
  int h_cap = 0;
  std::vector<double*> phi;
  std::vector<cudaEvent_t> chunk_ev;
  cudaEvent_t done = nullptr, h2d = nullptr;
};
}  // namespace sipb

using namespace sipb;  // internal header: the context is built from sipb types

struct sip_ctx {
  int device = 0, precision = 0, rank = 0, nranks = 1;
  size_t esize = 8;
  Lattice L;
  std::vector<int> rank_of, local, local_of;
  std::vector<BlockDesc> hblocks;
  std::vector<BrickDesc> hbricks;
  std::vector<int> order_f, order_b;
  BlockDesc* d_blocks = nullptr;
  BrickDesc* d_bricks = nullptr;
  int* d_order_f = nullptr;
  int* d_order_b = nullptr;
  // packs (brick-slice layout, sip_internal.h): forward (F_NA arrays), backward
  // (B_NA), R; phi with its ghost cells (porches + ghost bricks)
  void *fw = nullptr, *bw = nullptr, *phi = nullptr, *R = nullptr;
  // fp64 AP..AT for the factorisation: the forward pack itself in double
  // mode (coef_na = F_NA), a C_NA-array pack in single mode (no fp64 factors
  // are kept: K1 stores the fp32 factors directly)
  double* coef64 = nullptr;
  int coef_na = F_NA;
  std::vector<char> symmetric;  // per local block: system flagged symmetric
  // per local block, kernel face order: >= 0 where the installed halo plan
  // writes that ghost face (store_phi returns those ghosts)
  std::vector<std::array<int, 6>> plan_ghosts;
  // cross-brick mailboxes (tagged words): [0] K2 E col, [1] K2 N row, [2] K3 W col,
  // [3] K3 S row, [4] K1 E col, [5] K1 N row
  unsigned long long* mbox[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  size_t mbox_bytes[6] = {0, 0, 0, 0, 0, 0};
  unsigned* epochs = nullptr;           // [0] K2, [1] K3, [2] K1 launch counters
  unsigned *st_f = nullptr, *st_b = nullptr, *st_fac = nullptr;
  double* partial = nullptr;
  double* d_norms = nullptr;
  double* d_bnorms = nullptr;
  int norm_cap = 0, n_done = 0;
  unsigned long long* d_bad = nullptr;
  double* staging = nullptr;  // 8 x Gmax doubles (generator needs all 8)
  size_t gmax = 0;
  double* phi_stage = nullptr;       // per local block Field3 fp64 mirror of phi (load/store)
  std::vector<size_t> phi_stage_off;
  long long total_slices = 0, total_phi_slices = 0, total_edge = 0, total_row = 0;
  int grid_f = 1, grid_b = 1, grid_fac = 1;
  cudaStream_t own_stream = nullptr, stream = nullptr;
  long long revision = 0, factor_stamp = -1;
  bool factored = false;
  double alpha = 0.92;
  std::vector<FaceCopy> local_copies;
  FaceCopy* d_local_copies = nullptr;
  int local_max_plane = 0;
  std::vector<sipb::Peer> peers;
  // SIP face-halo exchange lists (install_plan): local copies + packs, early
  // entries (source plane E / N / T: final while K3 still runs) first; unpacks,
  // early (ghost W / S / B) first.  Pack / unpack offsets index x_sbuf / x_rbuf.
  FaceCopy *d_x = nullptr, *d_ux = nullptr;
  int x_early = 0, x_late = 0, ux_early = 0, ux_late = 0, x_max_plane = 0;
  void *x_sbuf = nullptr, *x_rbuf = nullptr;
  // split exchange (opt-in, env SIPB_XSPLIT=1): phase 1 on the
  // comm stream xstream from the end of K2 (waits on K3's per-brick stamps),
  // phase 2 after K3; the next K2 waits on ev_x
  bool xsplit = false;
  cudaStream_t xstream = nullptr;
  cudaEvent_t ev_k2 = nullptr, ev_k3 = nullptr, ev_x = nullptr;
  unsigned* d_xflag = nullptr;  // [2 * nbricks] K3 stamps (SweepParams::xflag)
  unsigned* d_xseq = nullptr;   // bumped by K2's finaliser
  XItem* d_xitems = nullptr;    // phase 1 work items (per brick of each early plane)
  int n_xitems = 0;
  // pipelined solves (sip_set_source_async / sip_solve_async): copy stream,
  // two staging slots per local block for the source (Field3 doubles), the
  // event of each slot's H2D and of the scatter that last read it; up to two
  // solves in flight (AsyncSolve), the second with its own phi mirror
  cudaStream_t cstream = nullptr;
  double* q_stage = nullptr;
  std::vector<int> q_slot;
  std::vector<std::array<cudaEvent_t, 2>> ev_qcopy, ev_qscat;
  double* phi_stage2 = nullptr;
  sipb::AsyncSolve async[2];
  int async_head = 0, async_count = 0;
  ncclComm_t comm = nullptr;
  bool prof = false;
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> events;  // kind 0 fwd, 1 bwd, 2 halo
  double t_fwd = 0, t_bwd = 0, t_halo = 0;
  long long launches = 0, prof_launches = 0;
  long long factor_count = 0;  // K1 launches (SPEC.md:185 factorisation counter)
  unsigned long long* trace = nullptr;  // debug: per-brick timestamps of the last F/B sweeps
  int trace_brick = -1;                 // debug: brick with per-stage marks (env SIPB_TRACE_BRICK)
  // pressure-correction caller (sip_flow.cu): grid of the assembled Poisson
  // system, boundary kinds per face (W,E,S,N,B,T) and the pinned cell
  bool poisson = false;
  double h[3] = {1.0, 1.0, 1.0};
  int bc[6] = {0, 0, 0, 0, 0, 0};
  int pin_local = -1;  // local block holding global cell (0,0,0), or -1
  // test mode (env SIPB_NCCL_SELF=1, single rank): local face transfers go
  // through the NCCL pack / send / recv / unpack path to this rank itself
  bool nccl_self = false;
  long long plan_gen = 0;  // bumped by install_plan (flows are bound to one plan)
  unsigned* d_norm_it = nullptr;  // device iteration counter (== n_done between calls)
  unsigned* d_ctl = nullptr;      // [0] target reached (K2 skips), [1] K3 pending (SweepParams::ctl)
  double solve_target = 0.0;      // > 0 while a single-rank target solve is enqueued
  // a sweep launch failed part-way: the device counters (ticket / done state,
  // norm slot, stop flags) may be out of step with the host; iterate refuses
  // until sip_load_phi resets them
  bool failed = false;
  // CUDA graph of one sip_iterate(iters) call (single rank, no profiling,
  // opt-in): kernels of `iters` iterations captured once and replayed
  cudaGraphExec_t graph_exec = nullptr;
  int graph_iters = -1;
  long long graph_plan = -1, graph_launches = 0;
  const void* graph_norms = nullptr;
  cudaStream_t graph_stream = nullptr;
  int graph_sym = -1;
  bool use_graphs = false;  // opt-in: env SIPB_GRAPH=1 at context creation
  double* d_gather = nullptr;  // multi-rank norm all-gather buffers (sip_read_norms)
  size_t gather_cap = 0;       // doubles
  double* h_pad = nullptr;     // pinned host staging of the all-gather send buffer
  size_t h_pad_cap = 0;
  double* d_pad = nullptr;     // (reserved)
  std::string err;
};

#define CK(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                \
      return (e_ == cudaErrorMemoryAllocation) ? SIP_ERR_NOMEM : SIP_ERR_CUDA;      \
    }                                                                               \
  } while (0)
#define CKS(call)                        \
  do {                                   \
    int s_ = (call);                     \
    if (s_ != SIP_OK) {                  \
      if (ctx->err.empty()) ctx->err = #call; \
      return s_;                         \
    }                                    \
  } while (0)
#define CKN(call)                                                           \
  do {                                                                      \
    ncclResult_t r_ = (call);                                               \
    if (r_ != ncclSuccess) {                                                \
      ctx->err = std::string(#call) + ": " + nccl().GetErrorString(r_);     \
      return SIP_ERR_NCCL;                                                  \
    }                                                                       \
  } while (0)


namespace sipb {

int set_device(sip_ctx* ctx);

template <typename P>
int dalloc(sip_ctx* ctx, P** p, size_t bytes) {
  void* v = nullptr;
  CK(cudaMalloc(&v, bytes ? bytes : 16));
  CK(cudaMemset(v, 0, bytes ? bytes : 16));
  *p = static_cast<P*>(v);
  return SIP_OK;
}

inline size_t field3_elems(const BlockDesc& b) {
  return (size_t)(b.nx + 2) * (b.ny + 2) * (b.nz + 2);
}

// Exchange structures of a face-halo plan (sip_api.cu).
int install_plan(sip_ctx* ctx, const std::vector<HaloEntry>& plan);
// One face-halo exchange of phi (device copies + NCCL), on ctx->stream.
template <typename T>
int exchange(sip_ctx* ctx);
// `iters` SIP iterations (K2, K3, halo) on ctx->stream.
template <typename T>
int iterate_t(sip_ctx* ctx, int iters);
// One Field3 array (device) of a local block into the packs (forward pack,
// and the fp64 coefficient pack in single mode).
int scatter_array(sip_ctx* ctx, int local, const double* src, int arr);
// Factors present and stamped with the current system revision.
int check_ready(sip_ctx* ctx);

}  // namespace sipb
