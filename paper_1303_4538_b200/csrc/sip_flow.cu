// sip_flow.cu -- the caller of the SIP hot path:
// assemble_poisson and the pressure-correction outer loop
// pressure_correct with factor reuse -- the factors of the
// constant pressure system are computed once (sip_factor) and every step only
// refreshes the source Q (factorization counter = 1 over 100
// steps).
//
// Flow fields (u, v, w, p) are fp64 Field3 arrays per local block, resident
// in HBM next to the solver's packs (same per-block offsets as the phi
// staging mirror).  Every step is a handful of HBM-bound stencil kernels
// around the SIP iterations: face ghosts of u, v, w (device copies / NCCL,
// the solver's halo plan incl. periodic wraps), divergence + source scatter,
// SIP sweeps from p' = 0, velocity / pressure update from p' in place.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "sip_ctx.h"

using namespace sipb;

namespace {

constexpr int kFlowThreads = 256;

__device__ __forceinline__ long long f3(int nx, int ny, int i, int j, int k) {
  return (long long)i + (long long)(nx + 2) * (j + (long long)(ny + 2) * k);
}

// Field3 index of plane element (a, c) of face `face` of a block, interior
// layer (ghost = false) or ghost layer (ghost = true); kernel face order.
__device__ __forceinline__ long long face_index(const BlockDesc& b, int face, bool ghost, int a,
                                                int c) {
  const int nx = b.nx, ny = b.ny, nz = b.nz;
  switch (face) {
    case G_W: return f3(nx, ny, ghost ? 0 : 1, a + 1, c + 1);
    case G_E: return f3(nx, ny, ghost ? nx + 1 : nx, a + 1, c + 1);
    case G_S: return f3(nx, ny, a + 1, ghost ? 0 : 1, c + 1);
    case G_N: return f3(nx, ny, a + 1, ghost ? ny + 1 : ny, c + 1);
    case G_B: return f3(nx, ny, a + 1, c + 1, ghost ? 0 : 1);
    default: return f3(nx, ny, a + 1, c + 1, ghost ? nz + 1 : nz);
  }
}

// 7-point Poisson coefficients of one block into Field3 arrays
// (AP, AW, AE, AS, AN, AB, AT, Q).  cpl[f]: the block face f is coupled to a
// neighbour (interface or periodic wrap); a domain wall / symmetry face is not.
__global__ void k_poisson_coeffs(int nx, int ny, int nz, int4 cpl_wesn, int2 cpl_bt, double ax,
                                 double ay, double az, int pin, double* const* out8) {
  const long long n = (long long)nx * ny * nz;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(c % nx), j = (int)((c / nx) % ny), k = (int)(c / ((long long)nx * ny));
    const long long x = f3(nx, ny, i + 1, j + 1, k + 1);
    const double w = (i > 0 || cpl_wesn.x) ? ax : 0.0;
    const double e = (i < nx - 1 || cpl_wesn.y) ? ax : 0.0;
    const double s = (j > 0 || cpl_wesn.z) ? ay : 0.0;
    const double nn = (j < ny - 1 || cpl_wesn.w) ? ay : 0.0;
    const double b = (k > 0 || cpl_bt.x) ? az : 0.0;
    const double t = (k < nz - 1 || cpl_bt.y) ? az : 0.0;
    if (pin && c == 0) {  // identity row
      out8[0][x] = 1.0;
      for (int a = 1; a < 8; ++a) out8[a][x] = 0.0;
      continue;
    }
    out8[0][x] = ((((w + e) + s) + nn) + b) + t;
    out8[1][x] = -w;
    out8[2][x] = -e;
    out8[3][x] = -s;
    out8[4][x] = -nn;
    out8[5][x] = -b;
    out8[6][x] = -t;
    out8[7][x] = 0.0;
  }
}

struct FieldSet {
  double* f[3];  // up to three fields with the same block offsets
  int nf;
};

// Face copies of a halo plan applied to Field3 fields: interior plane of the
// source block -> ghost plane of the destination block, or plane -> buffer
// (pack) / buffer -> ghost plane (unpack).  Buffer layout [field][count].
__global__ void k_flow_faces(const FaceCopy* copies, const BlockDesc* blocks, const long long* off,
                             FieldSet fs, const double* buf_in, double* buf_out, long long count) {
  const FaceCopy fc = copies[blockIdx.y];
  const int n = fc.n0 * fc.n1;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
    const int a = x % fc.n0, c = x / fc.n0;
    for (int q = 0; q < fs.nf; ++q) {
      double v;
      if (fc.src_block >= 0)
        v = fs.f[q][off[fc.src_block] + face_index(blocks[fc.src_block], fc.src_face, false, a, c)];
      else
        v = buf_in[q * count + fc.buf + x];
      if (fc.dst_block >= 0)
        fs.f[q][off[fc.dst_block] + face_index(blocks[fc.dst_block], fc.dst_face, true, a, c)] = v;
      else
        buf_out[q * count + fc.buf + x] = v;
    }
  }
}

// Domain-boundary ghosts of one block: ghost = sign * interior on the faces
// with wall[f] != 0 (u_n: -1 -> zero normal velocity at the face; p': +1 ->
// homogeneous Neumann).  sign[q][f] per field.
__global__ void k_flow_walls(BlockDesc b, int nf, double* f0, double* f1, double* f2,
                             int wall_mask, int sign_mask0, int sign_mask1, int sign_mask2) {
  const int face = blockIdx.y;
  if (!((wall_mask >> face) & 1)) return;
  const int n0 = face <= G_E ? b.ny : b.nx;
  const int n1 = face <= G_N ? b.nz : b.ny;
  double* fl[3] = {f0, f1, f2};
  const int sm[3] = {sign_mask0, sign_mask1, sign_mask2};
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n0 * n1; x += gridDim.x * blockDim.x) {
    const int a = x % n0, c = x / n0;
    const long long gi = face_index(b, face, true, a, c), ii = face_index(b, face, false, a, c);
    for (int q = 0; q < nf; ++q) fl[q][gi] = ((sm[q] >> face) & 1) ? -fl[q][ii] : fl[q][ii];
  }
}

// Co-located central divergence of one block; Q = -(V * div) / dt straight
// into the source array of the system's brick-slice pack (pinned cell: 0) and
// the block's L1 partials.  CTA (chunk, c) owns kChunkB consecutive bricks of
// one brick row (up to 32 i x 32 j columns) over planes [kDivKC*c, +kDivKC):
// phase 1 reads u, v, w with 32 consecutive i per warp (256 B rows) and keeps
// Q of the chunk in shared memory; phase 2 writes it brick by brick, slice by
// slice -- a warp writes the kL lanes of one slice (coalesced pack rows).
// The partial of a CTA sums its cells in a fixed order (per thread over j, k;
// fixed shuffle tree, warps in order): deterministic.
constexpr int kChunkB = 4;  // bricks per CTA along i (caller kernels)
constexpr int kDivKC = 4;
__host__ __device__ inline int chunks_i(const BlockDesc& b) { return (b.BX + kChunkB - 1) / kChunkB; }
template <typename T>
__global__ void __launch_bounds__(kFlowThreads) k_divergence(const BlockDesc* blocks, int blk,
                                                             const double* __restrict__ u,
                                                             const double* __restrict__ v,
                                                             const double* __restrict__ w, double c2x, double c2y,
                                                             double c2z, double vol, double dt, int pin,
                                                             T* fw, double* partial) {
  static_assert(kChunkB * kW == 32 && kFlowThreads % 32 == 0, "32 i per warp");
  __shared__ double sq[kDivKC][kL][kChunkB * kW];
  __shared__ double s[kFlowThreads / 32];
  const BlockDesc bd = blocks[blk];
  const int nx = bd.nx, ny = bd.ny, nz = bd.nz;
  const int nci = chunks_i(bd), bq = blockIdx.x % nci, bj = blockIdx.x / nci;
  const int i0 = bq * kChunkB * kW, j0 = bj * kL, k0 = blockIdx.y * kDivKC;
  const int wI = min(kChunkB * kW, nx - i0), wJ = min(kL, ny - j0), wK = min(kDivKC, nz - k0);
  const long long sy = nx + 2, sz = (long long)(nx + 2) * (ny + 2);
  constexpr int kRows = kFlowThreads / 32;
  const int il = threadIdx.x & 31, jq = threadIdx.x >> 5;
  double acc = 0.0;
  if (il < wI) {
    for (int jl = jq; jl < wJ; jl += kRows) {
      for (int kk = 0; kk < wK; ++kk) {
        const long long x = f3(nx, ny, i0 + il + 1, j0 + jl + 1, k0 + kk + 1);
        const double dv = ((u[x + 1] - u[x - 1]) / c2x + (v[x + sy] - v[x - sy]) / c2y) +
                          (w[x + sz] - w[x - sz]) / c2z;
        const bool pinned = pin && i0 + il == 0 && j0 + jl == 0 && k0 + kk == 0;
        sq[kk][jl][il] = pinned ? 0.0 : -(vol * dv) / dt;
        acc += fabs(dv) * vol;
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int x = 0; x < kFlowThreads / 32; ++x) t += s[x];
    partial[(long long)blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
  if (!fw) return;
  // phase 2: per brick, warp q writes slices tau = 8 k0 + q, + 8, ...; lane = jl
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  for (int bb = 0; bb < kChunkB; ++bb) {
    const int bi = bq * kChunkB + bb;
    if (bi >= bd.BX) break;
    const int wIb = min(kW, nx - bi * kW);
    const long long slot = bd.slot0 + (long long)(bi + bd.BX * bj) * bd.ns;
    for (int tau = kW * k0 + q; tau < kW * (k0 + wK) + kL - 1; tau += kRows) {
      const int c = tau - lane, k = c >> 3, ci = c & (kW - 1);
      if (lane < wJ && c >= 0 && k >= k0 && k < k0 + wK && ci < wIb)
        fw[((slot + tau) * F_NA + F_Q) * kL + lane] = static_cast<T>(sq[k - k0][lane][bb * kW + ci]);
    }
  }
}

// Sum of n partials in a fixed order by one CTA: thread t sums t, t+256, ...,
// then the fixed shuffle tree and the warps in order.
__global__ void __launch_bounds__(kFlowThreads) k_sum_partials(const double* partial, int n,
                                                               double* out) {
  __shared__ double s[kFlowThreads / 32];
  double acc = 0.0;
  for (int b = threadIdx.x; b < n; b += kFlowThreads) acc += partial[b];
#pragma unroll
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int r = 0; r < kFlowThreads / 32; ++r) t += s[r];
    *out = t;
  }
}

// u -= dt * dp'/dx (central), v, w likewise; p += p' -- reading p' straight
// from the solver's phi (brick layout): no gather into a Field3 mirror and no
// wall kernel for p'.  CTA (chunk, c) stages p' of kChunkB bricks of one brick
// row (up to 32 i x 32 j columns) over kCorKC planes plus a one-cell halo in
// shared memory: the bricks' own slices incl. the planes below / above as
// coalesced 32-lane rows, the i / j halo cell by cell -- the neighbour brick's
// cell, the phi ghost (interface / periodic face, exchanged after the last
// sweep) or, at a wall / symmetry face, the interior cell (Neumann: what
// k_flow_walls gives a gathered p').  The update then runs with 32
// consecutive i per warp.  Values and operation order are those of the
// Field3 formulation (oracle/flow.py), so u, v, w, p are bitwise the oracle's.
template <typename T>
struct CorCfg {
  static constexpr int KC = sizeof(T) == 8 ? 3 : 4;  // planes per CTA (static smem < 48 KB)
};
constexpr int kCorThreads = kFlowThreads;
template <typename T>
__global__ void __launch_bounds__(kCorThreads) k_correct_b(const BlockDesc* blocks, int blk, int wall,
                                                            const T* __restrict__ phi, double* __restrict__ u,
                                                            double* __restrict__ v, double* __restrict__ w,
                                                            double* __restrict__ p, double c2x, double c2y,
                                                            double c2z, double dt) {
  constexpr int KC = CorCfg<T>::KC, CW = kChunkB * kW;
  __shared__ T sp[KC + 2][kL + 2][CW + 2];
  const BlockDesc bd = blocks[blk];
  const int nx = bd.nx, ny = bd.ny, nz = bd.nz;
  const int nci = chunks_i(bd), bq = blockIdx.x % nci, bj = blockIdx.x / nci;
  const int i0 = bq * CW, j0 = bj * kL, k0 = blockIdx.y * KC;
  const int wI = min(CW, nx - i0), wJ = min(kL, ny - j0), wK = min(KC, nz - k0);
  const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  constexpr int kRows = kCorThreads / 32;
  // own slices incl. planes k0 - 1 and k0 + wK (interior, or the B / T ghost
  // plane in the porch): per brick, warp q loads slices 8 (k0 - 1) + q, + 8, ...
  for (int bb = 0; bb < kChunkB; ++bb) {
    const int bi = bq * kChunkB + bb;
    if (bi >= bd.BX) break;
    const int wIb = min(kW, nx - bi * kW);
    const long long pslot = phi_slot(bd, bi + bd.BX * bj);
    for (int tau = kW * (k0 - 1) + q; tau < kW * (k0 + wK + 1) + kL - 1; tau += kRows) {
      const int c = tau - lane, k = c >> 3, ci = c & (kW - 1);  // arithmetic shift: k = -1 below 0
      if (lane < wJ && k >= k0 - 1 && k <= k0 + wK && ci < wIb)
        sp[k - k0 + 1][lane + 1][bb * kW + ci + 1] = phi[(pslot + tau) * kL + lane];
    }
  }
  // i / j halo faces of the chunk (no edges / corners: 7-point stencil)
  auto pv = [&](int i, int j, int k) {
    if (i < 0 && (wall & (1 << G_W))) i = 0;
    if (i >= nx && (wall & (1 << G_E))) i = nx - 1;
    if (j < 0 && (wall & (1 << G_S))) j = 0;
    if (j >= ny && (wall & (1 << G_N))) j = ny - 1;
    return phi[phi_index(bd, i, j, k)];
  };
  const int hI = 2 * wJ * wK, hJ = 2 * wI * wK;
  for (int t = threadIdx.x; t < hI + hJ; t += kCorThreads) {
    if (t < hI) {
      const int side = t / (wJ * wK), e = t % (wJ * wK), jl = e % wJ, kk = e / wJ;
      const int il = side ? wI : -1;
      sp[kk + 1][jl + 1][il + 1] = pv(i0 + il, j0 + jl, k0 + kk);
    } else {
      const int x = t - hI, side = x / (wI * wK), e = x % (wI * wK), il = e % wI, kk = e / wI;
      const int jl = side ? wJ : -1;
      sp[kk + 1][jl + 1][il + 1] = pv(i0 + il, j0 + jl, k0 + kk);
    }
  }
  __syncthreads();
  // walls below / above: the ghost plane is the interior plane (Neumann)
  const bool wb = k0 == 0 && (wall & (1 << G_B)), wt = k0 + wK == nz && (wall & (1 << G_T));
  if (wb || wt) {
    for (int t = threadIdx.x; t < wI * wJ; t += kCorThreads) {
      const int il = t % wI, jl = t / wI;
      if (wb) sp[0][jl + 1][il + 1] = sp[1][jl + 1][il + 1];
      if (wt) sp[wK + 1][jl + 1][il + 1] = sp[wK][jl + 1][il + 1];
    }
    __syncthreads();
  }
  if (lane >= wI) return;
  const int il = lane;
  for (int jl = q; jl < wJ; jl += kRows) {
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
      if (kk >= wK) break;
      const long long x = f3(nx, ny, i0 + il + 1, j0 + jl + 1, k0 + kk + 1);
      const auto& s0 = sp[kk + 1];
      const double pc = static_cast<double>(s0[jl + 1][il + 1]);
      u[x] = u[x] - dt * ((static_cast<double>(s0[jl + 1][il + 2]) - static_cast<double>(s0[jl + 1][il])) / c2x);
      v[x] = v[x] - dt * ((static_cast<double>(s0[jl + 2][il + 1]) - static_cast<double>(s0[jl][il + 1])) / c2y);
      w[x] = w[x] - dt * ((static_cast<double>(sp[kk + 2][jl + 1][il + 1]) -
                           static_cast<double>(sp[kk][jl + 1][il + 1])) / c2z);
      p[x] = p[x] + pc;
    }
  }
}

int grid_for(long long n) {
  const long long g = (n + kFlowThreads - 1) / kFlowThreads;
  return (int)std::max(1LL, std::min(g, 148LL * 16));
}

}  // namespace

struct sip_flow {
  sip_ctx* ctx = nullptr;
  double* f[4] = {nullptr, nullptr, nullptr, nullptr};  // u, v, w, p
  long long* d_off = nullptr;    // per local block Field3 offset (= phi_stage_off)
  double* partial = nullptr;     // chunk partials
  double* d_blocksum = nullptr;  // per local block L1
  std::vector<int> wall;         // per local block: bit f = domain wall / symmetry face
  std::vector<std::pair<double*, double*>> pbuf;  // per peer: 3-field send / recv buffers
  long long max_cells = 0;
  long long max_parts = 0;  // divergence partial sums of the largest block
  long long plan_gen = 0;   // the context's halo plan this flow's buffers were sized for
  double* d_gather = nullptr;  // multi-rank L1: per-block values, send + all-gather receive
};

namespace {

int flow_err(sip_ctx* ctx, const std::string& e, int code) {
  ctx->err = e;
  return code;
}

// Face ghosts of the fields in `fs` from the context's halo plan (local
// copies + NCCL send / recv of all fields in one message per peer).
int flow_exchange(sip_flow* fl, const FieldSet& fs) {
  sip_ctx* ctx = fl->ctx;
  const cudaStream_t st = ctx->stream;
  if (!ctx->local_copies.empty()) {
    dim3 g((unsigned)std::max(1, std::min(64, (ctx->local_max_plane + kFlowThreads - 1) / kFlowThreads)),
           (unsigned)ctx->local_copies.size());
    k_flow_faces<<<g, kFlowThreads, 0, st>>>(ctx->d_local_copies, ctx->d_blocks, fl->d_off, fs,
                                             nullptr, nullptr, 0);
    CK(cudaGetLastError());
    ++ctx->launches;
  }
  if (!ctx->peers.empty()) {
    for (size_t pi = 0; pi < ctx->peers.size(); ++pi) {
      Peer& p = ctx->peers[pi];
      if (p.pack.empty()) continue;
      dim3 g((unsigned)std::max(1, std::min(64, (p.max_plane + kFlowThreads - 1) / kFlowThreads)),
             (unsigned)p.pack.size());
      k_flow_faces<<<g, kFlowThreads, 0, st>>>(p.d_pack, ctx->d_blocks, fl->d_off, fs, nullptr,
                                               fl->pbuf[pi].first, p.count);
      CK(cudaGetLastError());
      ++ctx->launches;
    }
    CKN(nccl().GroupStart());
    for (size_t pi = 0; pi < ctx->peers.size(); ++pi) {
      Peer& p = ctx->peers[pi];
      const size_t n = (size_t)p.count * fs.nf;
      CKN(nccl().Recv(fl->pbuf[pi].second, n, ncclFloat64, p.rank, ctx->comm, st));
      CKN(nccl().Send(fl->pbuf[pi].first, n, ncclFloat64, p.rank, ctx->comm, st));
    }
    CKN(nccl().GroupEnd());
    for (size_t pi = 0; pi < ctx->peers.size(); ++pi) {
      Peer& p = ctx->peers[pi];
      if (p.unpack.empty()) continue;
      dim3 g((unsigned)std::max(1, std::min(64, (p.max_plane + kFlowThreads - 1) / kFlowThreads)),
             (unsigned)p.unpack.size());
      k_flow_faces<<<g, kFlowThreads, 0, st>>>(p.d_unpack, ctx->d_blocks, fl->d_off, fs,
                                               fl->pbuf[pi].second, nullptr, p.count);
      CK(cudaGetLastError());
      ++ctx->launches;
    }
  }
  return SIP_OK;
}

// Domain-wall ghosts of up to three fields of every local block.
int flow_walls(sip_flow* fl, double* const* fields, int nf, const int* sign_masks) {
  sip_ctx* ctx = fl->ctx;
  for (size_t lb = 0; lb < ctx->local.size(); ++lb) {
    if (!fl->wall[lb]) continue;
    const BlockDesc& b = ctx->hblocks[lb];
    const size_t o = ctx->phi_stage_off[lb];
    const int plane = std::max(b.nx, b.ny) * std::max(b.ny, b.nz);
    dim3 g((unsigned)std::max(1, std::min(64, (plane + kFlowThreads - 1) / kFlowThreads)), 6);
    k_flow_walls<<<g, kFlowThreads, 0, ctx->stream>>>(
        b, nf, fields[0] + o, nf > 1 ? fields[1] + o : nullptr,
        nf > 2 ? fields[2] + o : nullptr, fl->wall[lb], sign_masks[0], nf > 1 ? sign_masks[1] : 0,
        nf > 2 ? sign_masks[2] : 0);
    CK(cudaGetLastError());
    ++ctx->launches;
  }
  return SIP_OK;
}

// Sum of per-block values over all ranks in global block order (the fixed
// order makes the result independent of the block placement).
int allsum_blocks(sip_flow* fl, const std::vector<double>& local_vals, double* out) {
  sip_ctx* ctx = fl->ctx;
  const int nb = (int)ctx->L.blocks.size();
  std::vector<double> all(nb, 0.0);
  if (ctx->nranks == 1) {
    for (size_t lb = 0; lb < ctx->local.size(); ++lb) all[ctx->local[lb]] = local_vals[lb];
  } else {
    std::vector<std::vector<int>> blocks_of(ctx->nranks);
    for (int b = 0; b < nb; ++b) blocks_of[ctx->rank_of[b]].push_back(b);
    int maxl = 1;
    for (auto& v : blocks_of) maxl = std::max<int>(maxl, (int)v.size());
    double* d_send = fl->d_gather;  // [maxl] send, then [nranks * maxl] receive
    double* d_recv = fl->d_gather + maxl;
    std::vector<double> pad(maxl, 0.0);
    for (size_t lb = 0; lb < ctx->local.size(); ++lb) pad[lb] = local_vals[lb];
    CK(cudaMemcpyAsync(d_send, pad.data(), sizeof(double) * maxl, cudaMemcpyHostToDevice, ctx->stream));
    CKN(nccl().AllGather(d_send, d_recv, (size_t)maxl, ncclFloat64, ctx->comm, ctx->stream));
    std::vector<double> got((size_t)maxl * ctx->nranks);
    CK(cudaMemcpyAsync(got.data(), d_recv, got.size() * sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int r = 0; r < ctx->nranks; ++r)
      for (size_t lb = 0; lb < blocks_of[r].size(); ++lb) all[blocks_of[r][lb]] = got[(size_t)maxl * r + lb];
  }
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += all[b];
  *out = s;
  return SIP_OK;
}

// Ghosts of u, v, w, then divergence: Q scattered into the system's source
// (fp64 pack and, in single mode, the fp32 pack) and the L1 norm.
int flow_divergence(sip_flow* fl, double dt, bool write_q, double* l1) {
  sip_ctx* ctx = fl->ctx;
  FieldSet fs{{fl->f[0], fl->f[1], fl->f[2]}, 3};
  CKS(flow_exchange(fl, fs));
  const int signs[3] = {(1 << G_W) | (1 << G_E), (1 << G_S) | (1 << G_N), (1 << G_B) | (1 << G_T)};
  CKS(flow_walls(fl, fl->f, 3, signs));
  const double hx = ctx->h[0], hy = ctx->h[1], hz = ctx->h[2];
  const double vol = (hx * hy) * hz;
  std::vector<double> vals(ctx->local.size(), 0.0);
  for (size_t lb = 0; lb < ctx->local.size(); ++lb) {
    const BlockDesc& b = ctx->hblocks[lb];
    const size_t o = ctx->phi_stage_off[lb];
    const long long n = (long long)b.nx * b.ny * b.nz;
    const dim3 grid((unsigned)(chunks_i(b) * b.BY), (unsigned)((b.nz + kDivKC - 1) / kDivKC));
    const int nch = (int)(grid.x * grid.y);
    (void)n;
    if (ctx->precision == SIP_PREC_SINGLE)
      k_divergence<float><<<grid, kFlowThreads, 0, ctx->stream>>>(
          ctx->d_blocks, (int)lb, fl->f[0] + o, fl->f[1] + o, fl->f[2] + o, 2.0 * hx, 2.0 * hy,
          2.0 * hz, vol, dt, (int)lb == ctx->pin_local, write_q ? static_cast<float*>(ctx->fw) : nullptr,
          fl->partial);
    else
      k_divergence<double><<<grid, kFlowThreads, 0, ctx->stream>>>(
          ctx->d_blocks, (int)lb, fl->f[0] + o, fl->f[1] + o, fl->f[2] + o, 2.0 * hx, 2.0 * hy,
          2.0 * hz, vol, dt, (int)lb == ctx->pin_local, write_q ? static_cast<double*>(ctx->fw) : nullptr,
          fl->partial);
    k_sum_partials<<<1, kFlowThreads, 0, ctx->stream>>>(fl->partial, nch, fl->d_blocksum + lb);
    CK(cudaGetLastError());
    ctx->launches += 2;
  }
  CK(cudaMemcpyAsync(vals.data(), fl->d_blocksum, sizeof(double) * vals.size(), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return allsum_blocks(fl, vals, l1);
}

// p' = 0 (interior and ghosts), then `sweeps` SIP iterations; p' stays in the
// solver's phi (ghosts from the last exchange) for k_correct_b.
template <typename T>
int flow_solve(sip_flow* fl, int sweeps) {
  sip_ctx* ctx = fl->ctx;
  // p' = 0: interior and every ghost cell (one contiguous phi allocation)
  CK(cudaMemsetAsync(ctx->phi, 0, (size_t)ctx->total_phi_slices * kL * sizeof(T), ctx->stream));
  ctx->n_done = 0;
  CK(cudaMemsetAsync(ctx->d_norm_it, 0, sizeof(unsigned), ctx->stream));
  return iterate_t<T>(ctx, sweeps);
}

}  // namespace

extern "C" {

int sip_assemble_poisson(sip_ctx* ctx, const double len[3], const int bc[6]) {
  if (!ctx) return SIP_ERR_MISUSE;
  if (!len || !bc) return flow_err(ctx, "sip_assemble_poisson: null arguments", SIP_ERR_MISUSE);
  for (int a = 0; a < 3; ++a)
    if (!(len[a] > 0.0) || !std::isfinite(len[a]))
      return flow_err(ctx, "assemble_poisson: domain lengths must be positive", SIP_ERR_CONFIG);
  int mask = 0;
  for (int f = 0; f < 6; ++f) {
    if (bc[f] < SIP_BC_WALL || bc[f] > SIP_BC_SYMMETRY)
      return flow_err(ctx, "assemble_poisson: unknown boundary kind", SIP_ERR_CONFIG);
    if ((bc[f] == SIP_BC_PERIODIC) != (bc[f ^ 1] == SIP_BC_PERIODIC))
      return flow_err(ctx, "grid: periodic faces must come in opposing pairs", SIP_ERR_CONFIG);
    if (bc[f] == SIP_BC_PERIODIC) mask |= 1 << (f / 2);
  }
  CKS(set_device(ctx));
  double h[3];
  for (int a = 0; a < 3; ++a) h[a] = len[a] / ctx->L.g[a];
  // halo plan with the periodic wraps of this grid
  std::vector<HaloEntry> plan;
  plan_halo(ctx->L, ctx->rank_of, ctx->rank, plan, mask);
  CK(cudaStreamSynchronize(ctx->stream));
  CKS(install_plan(ctx, plan));
  const double ax = (h[1] * h[2]) / h[0], ay = (h[0] * h[2]) / h[1], az = (h[0] * h[1]) / h[2];
  const int arr[8] = {F_AP, F_AW, F_AE, F_AS, F_AN, F_AB, F_AT, F_Q};
  ctx->pin_local = ctx->local_of.empty() ? -1 : ctx->local_of[0];  // global cell (0,0,0) is in block 0
  double** d_out8 = nullptr;  // device copy of the 8 staging array pointers
  CKS(dalloc(ctx, &d_out8, 8 * sizeof(double*)));
  struct Free {
    void* p;
    ~Free() { cudaFree(p); }
  } free_out8{d_out8};
  for (size_t lb = 0; lb < ctx->local.size(); ++lb) {
    const BlockDesc& hb = ctx->hblocks[lb];
    const BlockInfo& bi = ctx->L.blocks[ctx->local[lb]];
    int cpl[6];
    for (int f = 0; f < 6; ++f) cpl[f] = bi.nbr[f] >= 0 || bc[f] == SIP_BC_PERIODIC;
    const size_t G = field3_elems(hb);
    double* out8[8];
    for (int a = 0; a < 8; ++a) out8[a] = ctx->staging + a * G;
    CK(cudaMemsetAsync(ctx->staging, 0, 8 * G * sizeof(double), ctx->stream));
    CK(cudaMemcpyAsync(d_out8, out8, sizeof(out8), cudaMemcpyHostToDevice, ctx->stream));
    const long long n = (long long)hb.nx * hb.ny * hb.nz;
    k_poisson_coeffs<<<grid_for(n), kFlowThreads, 0, ctx->stream>>>(
        hb.nx, hb.ny, hb.nz, make_int4(cpl[0], cpl[1], cpl[2], cpl[3]), make_int2(cpl[4], cpl[5]),
        ax, ay, az, (int)lb == ctx->pin_local, d_out8);
    CK(cudaGetLastError());
    ++ctx->launches;
    for (int a = 0; a < 8; ++a) CKS(scatter_array(ctx, (int)lb, out8[a], arr[a]));
    CK(cudaStreamSynchronize(ctx->stream));  // out8 (host array) and staging reused next block
  }
  ++ctx->revision;
  // the identity row of the pinned cell breaks ae(i) = aw(i+1) next to it, so
  // the system is not flagged symmetric (the general Listing-1 path runs)
  ctx->symmetric.assign(ctx->local.size(), 0);
  ctx->poisson = true;
  for (int a = 0; a < 3; ++a) ctx->h[a] = h[a];
  for (int f = 0; f < 6; ++f) ctx->bc[f] = bc[f];
  return SIP_OK;
}

int sip_flow_create(sip_ctx* ctx, sip_flow** out) {
  if (!ctx || !out) return SIP_ERR_MISUSE;
  *out = nullptr;
  if (!ctx->poisson)
    return flow_err(ctx, "sip_flow_create: assemble the pressure system first", SIP_ERR_MISUSE);
  CKS(set_device(ctx));
  sip_flow* fl = new sip_flow();
  fl->ctx = ctx;
  fl->plan_gen = ctx->plan_gen;
  size_t total = 0;
  for (const BlockDesc& b : ctx->hblocks) {
    total += field3_elems(b);
    fl->max_cells = std::max(fl->max_cells, (long long)b.nx * b.ny * b.nz);
    fl->max_parts = std::max(fl->max_parts, (long long)b.nbricks * ((b.nz + kDivKC - 1) / kDivKC));
  }
  auto fail = [&](int s) {
    sip_flow_destroy(fl);
    return s;
  };
  int s = SIP_OK;
  for (int q = 0; q < 4 && s == SIP_OK; ++q) s = dalloc(ctx, &fl->f[q], sizeof(double) * std::max<size_t>(1, total));
  if (s == SIP_OK)
    s = dalloc(ctx, &fl->partial, sizeof(double) * std::max(1LL, fl->max_parts));
  if (s == SIP_OK) s = dalloc(ctx, &fl->d_blocksum, sizeof(double) * std::max<size_t>(1, ctx->local.size()));
  if (s == SIP_OK) s = dalloc(ctx, &fl->d_off, sizeof(long long) * std::max<size_t>(1, ctx->local.size()));
  if (s == SIP_OK) {
    std::vector<int> per_rank(std::max(1, ctx->nranks), 0);
    for (int r : ctx->rank_of) ++per_rank[r];
    const int maxl = std::max(1, *std::max_element(per_rank.begin(), per_rank.end()));
    s = dalloc(ctx, &fl->d_gather, sizeof(double) * (size_t)maxl * (1 + std::max(1, ctx->nranks)));
  }
  if (s != SIP_OK) return fail(s);
  std::vector<long long> off(ctx->phi_stage_off.begin(), ctx->phi_stage_off.end());
  if (!off.empty() && cudaMemcpy(fl->d_off, off.data(), sizeof(long long) * off.size(),
                                 cudaMemcpyHostToDevice) != cudaSuccess)
    return fail(flow_err(ctx, "sip_flow_create: offset upload failed", SIP_ERR_CUDA));
  for (const Peer& p : ctx->peers) {
    double *a = nullptr, *b = nullptr;
    s = dalloc(ctx, &a, sizeof(double) * 3 * std::max(1LL, p.count));
    if (s == SIP_OK) s = dalloc(ctx, &b, sizeof(double) * 3 * std::max(1LL, p.count));
    fl->pbuf.emplace_back(a, b);
    if (s != SIP_OK) return fail(s);
  }
  // domain walls: faces whose ghosts the halo plan does not write
  fl->wall.assign(ctx->local.size(), 0);
  for (size_t lb = 0; lb < ctx->local.size(); ++lb)
    for (int f = 0; f < 6; ++f)
      if (ctx->plan_ghosts[lb][f] < 0) fl->wall[lb] |= 1 << f;
  *out = fl;
  return SIP_OK;
}

int sip_flow_destroy(sip_flow* fl) {
  if (!fl) return SIP_OK;
  if (fl->ctx) cudaSetDevice(fl->ctx->device);
  for (double* p : fl->f)
    if (p) cudaFree(p);
  void* ptrs[] = {fl->d_off, fl->partial, fl->d_blocksum, fl->d_gather};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& pb : fl->pbuf) {
    if (pb.first) cudaFree(pb.first);
    if (pb.second) cudaFree(pb.second);
  }
  delete fl;
  return SIP_OK;
}

int sip_flow_set(sip_flow* fl, int field, double* const* per_block) {
  if (!fl || !per_block) return SIP_ERR_MISUSE;
  sip_ctx* ctx = fl->ctx;
  if (field < SIP_FLOW_U || field > SIP_FLOW_P)
    return flow_err(ctx, "sip_flow_set: field must be SIP_FLOW_U .. SIP_FLOW_P", SIP_ERR_MISUSE);
  CKS(set_device(ctx));
  for (size_t lb = 0; lb < ctx->local.size(); ++lb) {
    if (!per_block[lb]) return flow_err(ctx, "sip_flow_set: null block array", SIP_ERR_MISUSE);
    CK(cudaMemcpyAsync(fl->f[field] + ctx->phi_stage_off[lb], per_block[lb],
                       field3_elems(ctx->hblocks[lb]) * sizeof(double), cudaMemcpyHostToDevice,
                       ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return SIP_OK;
}

int sip_flow_get(sip_flow* fl, int field, double* const* per_block) {
  if (!fl || !per_block) return SIP_ERR_MISUSE;
  sip_ctx* ctx = fl->ctx;
  if (field < SIP_FLOW_U || field > SIP_FLOW_P)
    return flow_err(ctx, "sip_flow_get: field must be SIP_FLOW_U .. SIP_FLOW_P", SIP_ERR_MISUSE);
  CKS(set_device(ctx));
  for (size_t lb = 0; lb < ctx->local.size(); ++lb) {
    if (!per_block[lb]) return flow_err(ctx, "sip_flow_get: null block array", SIP_ERR_MISUSE);
    CK(cudaMemcpyAsync(per_block[lb], fl->f[field] + ctx->phi_stage_off[lb],
                       field3_elems(ctx->hblocks[lb]) * sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return SIP_OK;
}

int sip_flow_divergence(sip_flow* fl, double* l1) {
  if (!fl || !l1) return SIP_ERR_MISUSE;
  sip_ctx* ctx = fl->ctx;
  if (fl->plan_gen != ctx->plan_gen)
    return flow_err(ctx, "flow created before the current halo plan: create a new flow", SIP_ERR_MISUSE);
  CKS(set_device(ctx));
  return flow_divergence(fl, 1.0, false, l1);
}

int sip_pressure_correct(sip_flow* fl, double dt, double threshold, int max_outer, int sweeps,
                         int* outer_used, double* div_hist) {
  if (!fl) return SIP_ERR_MISUSE;
  sip_ctx* ctx = fl->ctx;
  if (!(dt > 0.0) || max_outer < 0 || sweeps < 1 || !(threshold >= 0.0))
    return flow_err(ctx, "pressure_correct: need dt > 0, threshold >= 0, max_outer >= 0, sweeps >= 1",
                    SIP_ERR_CONFIG);
  if (fl->plan_gen != ctx->plan_gen)
    return flow_err(ctx, "flow created before the current halo plan: create a new flow", SIP_ERR_MISUSE);
  if (!ctx->poisson)
    return flow_err(ctx, "pressure_correct: the context's system is no longer the assembled pressure "
                         "system (sip_set_system / sip_generate_system since sip_assemble_poisson)",
                    SIP_ERR_MISUSE);
  CKS(check_ready(ctx));  // factors of the assembled system, reused (never refactored here)
  CKS(set_device(ctx));
  if (outer_used) *outer_used = 0;
  double d = 0.0;
  for (int outer = 0;; ++outer) {
    CKS(flow_divergence(fl, dt, true, &d));
    if (div_hist) div_hist[outer] = d;
    if (outer_used) *outer_used = outer;
    if (d <= threshold) return SIP_OK;
    if (outer == max_outer) {
      char buf[160];
      snprintf(buf, sizeof(buf),
               "pressure_correct: %d outer iterations left the divergence L1 at %.6e > %.6e", outer,
               d, threshold);
      return flow_err(ctx, buf, SIP_ERR_NOCONV);
    }
    CKS(ctx->precision == SIP_PREC_SINGLE ? flow_solve<float>(fl, sweeps) : flow_solve<double>(fl, sweeps));
    const double hx = ctx->h[0], hy = ctx->h[1], hz = ctx->h[2];
    for (size_t lb = 0; lb < ctx->local.size(); ++lb) {
      const BlockDesc& b = ctx->hblocks[lb];
      const size_t o = ctx->phi_stage_off[lb];
      const int kc = ctx->precision == SIP_PREC_SINGLE ? CorCfg<float>::KC : CorCfg<double>::KC;
      const dim3 grid((unsigned)(chunks_i(b) * b.BY), (unsigned)((b.nz + kc - 1) / kc));
      if (ctx->precision == SIP_PREC_SINGLE)
        k_correct_b<float><<<grid, kCorThreads, 0, ctx->stream>>>(
            ctx->d_blocks, (int)lb, fl->wall[lb], static_cast<const float*>(ctx->phi), fl->f[0] + o,
            fl->f[1] + o, fl->f[2] + o, fl->f[3] + o, 2.0 * hx, 2.0 * hy, 2.0 * hz, dt);
      else
        k_correct_b<double><<<grid, kCorThreads, 0, ctx->stream>>>(
            ctx->d_blocks, (int)lb, fl->wall[lb], static_cast<const double*>(ctx->phi), fl->f[0] + o,
            fl->f[1] + o, fl->f[2] + o, fl->f[3] + o, 2.0 * hx, 2.0 * hy, 2.0 * hz, dt);
      CK(cudaGetLastError());
      ++ctx->launches;
    }
  }
}

}  // extern "C"
