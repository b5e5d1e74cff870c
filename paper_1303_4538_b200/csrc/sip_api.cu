// sip_api.cu -- host runtime behind the C-ABI (include/sip_c.h): device
// memory for the tile-slice packs, factor/solve orchestration on one CUDA
// stream, face-halo exchange (device copies inside a GPU, NCCL send/recv
// between GPUs), deterministic norm reduction and per-kernel timing.
// Host C++ only calls kernels through the launchers of sip_kernels.cu.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

#include "sip_ctx.h"

using namespace sipb;

namespace {
thread_local std::string g_create_err;
}  // namespace
void sipb::set_thread_error(const std::string& err) { g_create_err = err; }

NcclApi& sipb::nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.err = std::string("dlopen libnccl.so.2: ") + dlerror();
      return a;
    }
#define SIPB_SYM(f) a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, "nccl" #f))
    SIPB_SYM(GetUniqueId); SIPB_SYM(CommInitRank); SIPB_SYM(CommDestroy); SIPB_SYM(Send);
    SIPB_SYM(Recv); SIPB_SYM(GroupStart); SIPB_SYM(GroupEnd); SIPB_SYM(AllGather);
    SIPB_SYM(GetErrorString);
#undef SIPB_SYM
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv &&
           a.GroupStart && a.GroupEnd && a.AllGather && a.GetErrorString;
    if (!a.ok) a.err = "libnccl.so.2 lacks required symbols";
    return a;
  }();
  return api;
}

int sipb::set_device(sip_ctx* ctx) {
  CK(cudaSetDevice(ctx->device));
  return SIP_OK;
}

// -------------------------------------------------------------- construction
// Source plane E / N / T (K3 finishes it first) <=> ghost W / S / B written.
static bool early_src(int kf) { return kf == G_E || kf == G_N || kf == G_T; }
static bool early_dst(int kf) { return kf == G_W || kf == G_S || kf == G_B; }

// The SIP exchange lists of the installed plan (sip_ctx::d_x / d_ux): local
// copies and packs, early entries first; unpacks, early first.  Each peer's
// message is [early | late] in plan order on both sides (a sender's E / N / T
// plane lands in the receiver's W / S / B ghost), so phase 1 sends the first
// s1 elements and phase 2 the rest, and the unsplit exchange sends it whole.
static int install_exchange(sip_ctx* ctx) {
  const size_t es = ctx->esize;
  std::vector<FaceCopy> x[2], ux[2];  // [early, late]
  int mp = 0;
  for (const FaceCopy& f : ctx->local_copies) {
    x[early_src(f.src_face) ? 0 : 1].push_back(f);
    mp = std::max(mp, f.n0 * f.n1);
  }
  long long so = 0, ro = 0;
  for (Peer& p : ctx->peers) {
    p.soff = so;
    p.roff = ro;
    p.s1 = p.r1 = 0;
    for (const FaceCopy& f : p.pack)
      if (early_src(f.src_face)) p.s1 += (long long)f.n0 * f.n1;
    for (const FaceCopy& f : p.unpack)
      if (early_dst(f.dst_face)) p.r1 += (long long)f.n0 * f.n1;
    long long se = so, sl = so + p.s1, re = ro, rl = ro + p.r1;
    for (FaceCopy f : p.pack) {
      long long& o = early_src(f.src_face) ? se : sl;
      f.buf = o;
      o += (long long)f.n0 * f.n1;
      x[early_src(f.src_face) ? 0 : 1].push_back(f);
    }
    for (FaceCopy f : p.unpack) {
      long long& o = early_dst(f.dst_face) ? re : rl;
      f.buf = o;
      o += (long long)f.n0 * f.n1;
      ux[early_dst(f.dst_face) ? 0 : 1].push_back(f);
    }
    mp = std::max(mp, p.max_plane);
    so += p.count;
    ro += p.count;
  }
  // phase 1 work items: each early copy's source plane split by brick, in the
  // order K3 finishes them -- the brick's position in K3's ticket order for
  // a T plane (its top slices are done a few stages after it starts), one
  // resident wave later for an E / N plane (the whole brick)
  std::vector<int> pos(ctx->hbricks.size(), 0);
  for (size_t t = 0; t < ctx->order_b.size(); ++t) pos[ctx->order_b[t]] = (int)t;
  std::vector<std::pair<long long, XItem>> items;
  for (int e = 0; e < (int)x[0].size(); ++e) {
    const FaceCopy& f = x[0][e];
    const BlockDesc& b = ctx->hblocks[f.src_block];
    for (int bj = 0; bj < b.BY; ++bj)
      for (int bi = 0; bi < b.BX; ++bi) {
        XItem it{e, b.brick0 + bi + b.BX * bj, 1, 0, 0, 0, 0};
        const int i0 = bi * kW, i1 = std::min(b.nx, i0 + kW), j0 = bj * kL, j1 = std::min(b.ny, j0 + kL);
        if (f.src_face == G_E) {
          if (bi != b.BX - 1) continue;
          it.x0b = j0, it.x0e = j1, it.x1b = 0, it.x1e = b.nz;
        } else if (f.src_face == G_N) {
          if (bj != b.BY - 1) continue;
          it.x0b = i0, it.x0e = i1, it.x1b = 0, it.x1e = b.nz;
        } else {  // G_T
          it.sel = 0;
          it.x0b = i0, it.x0e = i1, it.x1b = j0, it.x1e = j1;
        }
        items.emplace_back(pos[it.brick] + (it.sel ? (long long)ctx->grid_b : 0), it);
      }
  }
  std::stable_sort(items.begin(), items.end(),
                   [](const auto& a, const auto& b) { return a.first < b.first; });
  std::vector<XItem> hitems;
  for (auto& pr : items) hitems.push_back(pr.second);
  ctx->n_xitems = (int)hitems.size();
  if (!hitems.empty()) {
    CKS(dalloc(ctx, &ctx->d_xitems, sizeof(XItem) * hitems.size()));
    CK(cudaMemcpy(ctx->d_xitems, hitems.data(), sizeof(XItem) * hitems.size(), cudaMemcpyHostToDevice));
  }
  ctx->x_early = (int)x[0].size();
  ctx->x_late = (int)x[1].size();
  ctx->ux_early = (int)ux[0].size();
  ctx->ux_late = (int)ux[1].size();
  ctx->x_max_plane = mp;
  x[0].insert(x[0].end(), x[1].begin(), x[1].end());
  ux[0].insert(ux[0].end(), ux[1].begin(), ux[1].end());
  if (!x[0].empty()) {
    CKS(dalloc(ctx, &ctx->d_x, sizeof(FaceCopy) * x[0].size()));
    CK(cudaMemcpy(ctx->d_x, x[0].data(), sizeof(FaceCopy) * x[0].size(), cudaMemcpyHostToDevice));
  }
  if (!ux[0].empty()) {
    CKS(dalloc(ctx, &ctx->d_ux, sizeof(FaceCopy) * ux[0].size()));
    CK(cudaMemcpy(ctx->d_ux, ux[0].data(), sizeof(FaceCopy) * ux[0].size(), cudaMemcpyHostToDevice));
  }
  if (!ctx->peers.empty()) {
    CKS(dalloc(ctx, &ctx->x_sbuf, (size_t)std::max(1LL, so) * es));
    CKS(dalloc(ctx, &ctx->x_rbuf, (size_t)std::max(1LL, ro) * es));
    for (Peer& p : ctx->peers) {
      p.sbuf = static_cast<char*>(ctx->x_sbuf) + p.soff * es;
      p.rbuf = static_cast<char*>(ctx->x_rbuf) + p.roff * es;
    }
  }
  if (!ctx->xstream) {  // comm stream of the split exchange (highest priority)
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&ctx->xstream, cudaStreamNonBlocking, hi));
    CK(cudaEventCreateWithFlags(&ctx->ev_k2, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_k3, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_x, cudaEventDisableTiming));
  }
  return SIP_OK;
}

// Exchange structures of a face-halo plan (this rank's entries, plan order):
// local entries -> device face copies, send / recv entries -> per-peer NCCL
// pack / unpack lists.  Replaces a previously installed plan.
int sipb::install_plan(sip_ctx* ctx, const std::vector<HaloEntry>& plan) {
  const size_t es = ctx->esize;
  ++ctx->plan_gen;
  if (ctx->d_local_copies) cudaFree(ctx->d_local_copies);
  ctx->d_local_copies = nullptr;
  ctx->local_copies.clear();
  ctx->local_max_plane = 0;
  for (Peer& p : ctx->peers) {
    if (p.d_pack) cudaFree(p.d_pack);
    if (p.d_unpack) cudaFree(p.d_unpack);
  }
  ctx->peers.clear();
  for (void* q : {(void*)ctx->d_x, (void*)ctx->d_ux, ctx->x_sbuf, ctx->x_rbuf, (void*)ctx->d_xitems})
    if (q) cudaFree(q);
  ctx->d_x = ctx->d_ux = nullptr;
  ctx->d_xitems = nullptr;
  ctx->n_xitems = 0;
  ctx->x_sbuf = ctx->x_rbuf = nullptr;
  ctx->plan_ghosts.assign(ctx->local.size(), {-1, -1, -1, -1, -1, -1});
  // bsfv face id (E,W,N,S,T,B) -> kernel face (W,E,S,N,B,T)
  auto kface = [](int f) { static const int m[6] = {G_E, G_W, G_N, G_S, G_T, G_B}; return m[f]; };
  auto plane = [&](int gblock, int kf, int& n0, int& n1) {
    const BlockInfo& bi = ctx->L.blocks[gblock];
    if (kf <= G_E) { n0 = bi.n[1]; n1 = bi.n[2]; }
    else if (kf <= G_N) { n0 = bi.n[0]; n1 = bi.n[2]; }
    else { n0 = bi.n[0]; n1 = bi.n[1]; }
  };
  for (const HaloEntry& e : plan) {
    FaceCopy fc{};
    if (e.dir == 0 && ctx->nccl_self) {
      // debugging / hardware test of the multi-rank path on one GPU: a local
      // transfer becomes a send + recv pair with this rank itself, so the
      // pack kernels, NCCL send / recv and unpack kernels all run
      HaloEntry snd = e, rcv = e;
      snd.dir = 1;
      snd.peer = ctx->rank;
      rcv.dir = 2;
      rcv.peer = ctx->rank;
      rcv.owner = e.neighbor;
      rcv.neighbor = e.owner;
      rcv.face = e.face ^ 1;
      std::vector<HaloEntry> pair = {snd, rcv};
      for (const HaloEntry& x : pair) {
        auto it = std::find_if(ctx->peers.begin(), ctx->peers.end(),
                               [&](const Peer& pp) { return pp.rank == x.peer; });
        if (it == ctx->peers.end()) {
          ctx->peers.emplace_back();
          ctx->peers.back().rank = x.peer;
          it = ctx->peers.end() - 1;
        }
        FaceCopy f{};
        if (x.dir == 1) {
          f.src_block = ctx->local_of[x.owner];
          f.src_face = kface(x.face);
          f.dst_block = -1;
          plane(x.owner, f.src_face, f.n0, f.n1);
          for (auto& q : it->pack) f.buf += (long long)q.n0 * q.n1;
          it->pack.push_back(f);
        } else {
          f.src_block = -1;
          f.dst_block = ctx->local_of[x.owner];
          f.dst_face = kface(x.face);
          ctx->plan_ghosts[f.dst_block][f.dst_face] = x.neighbor;
          plane(x.owner, f.dst_face, f.n0, f.n1);
          for (auto& q : it->unpack) f.buf += (long long)q.n0 * q.n1;
          it->unpack.push_back(f);
        }
        it->max_plane = std::max(it->max_plane, f.n0 * f.n1);
      }
      continue;
    }
    if (e.dir == 0) {  // local: owner = src block, face = src plane; dst ghost = opposite
      fc.src_block = ctx->local_of[e.owner];
      fc.src_face = kface(e.face);
      fc.dst_block = ctx->local_of[e.neighbor];
      fc.dst_face = kface(e.face ^ 1);
      ctx->plan_ghosts[fc.dst_block][fc.dst_face] = e.owner;
      plane(e.owner, fc.src_face, fc.n0, fc.n1);
      ctx->local_copies.push_back(fc);
      ctx->local_max_plane = std::max(ctx->local_max_plane, fc.n0 * fc.n1);
      continue;
    }
    auto it = std::find_if(ctx->peers.begin(), ctx->peers.end(),
                           [&](const Peer& p) { return p.rank == e.peer; });
    if (it == ctx->peers.end()) {
      ctx->peers.emplace_back();
      ctx->peers.back().rank = e.peer;
      it = ctx->peers.end() - 1;
    }
    if (e.dir == 1) {  // send: owner = local src block, plane face
      fc.src_block = ctx->local_of[e.owner];
      fc.src_face = kface(e.face);
      fc.dst_block = -1;
      plane(e.owner, fc.src_face, fc.n0, fc.n1);
      fc.buf = 0;
      for (auto& q : it->pack) fc.buf += (long long)q.n0 * q.n1;
      it->pack.push_back(fc);
    } else {  // recv: owner = local dst block, face = ghost face
      fc.src_block = -1;
      fc.dst_block = ctx->local_of[e.owner];
      fc.dst_face = kface(e.face);
      ctx->plan_ghosts[fc.dst_block][fc.dst_face] = e.neighbor;
      plane(e.owner, fc.dst_face, fc.n0, fc.n1);
      fc.buf = 0;
      for (auto& q : it->unpack) fc.buf += (long long)q.n0 * q.n1;
      it->unpack.push_back(fc);
    }
    it->max_plane = std::max(it->max_plane, fc.n0 * fc.n1);
  }
  if (!ctx->local_copies.empty()) {
    CKS(dalloc(ctx, &ctx->d_local_copies, sizeof(FaceCopy) * ctx->local_copies.size()));
    CK(cudaMemcpy(ctx->d_local_copies, ctx->local_copies.data(),
                  sizeof(FaceCopy) * ctx->local_copies.size(), cudaMemcpyHostToDevice));
  }
  for (Peer& p : ctx->peers) {
    long long ns = 0, nr = 0;
    for (auto& q : p.pack) ns += (long long)q.n0 * q.n1;
    for (auto& q : p.unpack) nr += (long long)q.n0 * q.n1;
    if (ns != nr) {
      ctx->err = "halo plan: send/recv volume mismatch with rank " + std::to_string(p.rank);
      return SIP_ERR_CONFIG;
    }
    p.count = ns;
    CKS(dalloc(ctx, &p.d_pack, sizeof(FaceCopy) * std::max<size_t>(1, p.pack.size())));
    CKS(dalloc(ctx, &p.d_unpack, sizeof(FaceCopy) * std::max<size_t>(1, p.unpack.size())));
    if (!p.pack.empty())
      CK(cudaMemcpy(p.d_pack, p.pack.data(), sizeof(FaceCopy) * p.pack.size(), cudaMemcpyHostToDevice));
    if (!p.unpack.empty())
      CK(cudaMemcpy(p.d_unpack, p.unpack.data(), sizeof(FaceCopy) * p.unpack.size(),
                    cudaMemcpyHostToDevice));
  }
  return install_exchange(ctx);
}

static int build(sip_ctx* ctx) {
  // local blocks and their bricks (sip_internal.h layout)
  const int nb = (int)ctx->L.blocks.size();
  ctx->local_of.assign(nb, -1);
  for (int b = 0; b < nb; ++b)
    if (ctx->rank_of[b] == ctx->rank) {
      ctx->local_of[b] = (int)ctx->local.size();
      ctx->local.push_back(b);
    }
  long long slot = 0, pslot = 0, medge = 0, mrow = 0;
  for (size_t lb = 0; lb < ctx->local.size(); ++lb) {
    const BlockInfo& bi = ctx->L.blocks[ctx->local[lb]];
    BlockDesc bd{};
    bd.id = ctx->local[lb];
    bd.nx = bi.n[0]; bd.ny = bi.n[1]; bd.nz = bi.n[2];
    bd.BX = (bd.nx + kW - 1) / kW;
    bd.BY = (bd.ny + kL - 1) / kL;
    bd.ns = bd.nz * kW + kL;
    bd.brick0 = (int)ctx->hbricks.size();
    bd.nbricks = bd.BX * bd.BY;
    bd.gE = bd.nx % kW == 0;
    bd.gN = bd.ny % kL == 0;
    bd.slot0 = slot;
    bd.pbase = pslot;
    bd.medge0 = medge;
    bd.mrow0 = mrow;
    const long long me = (long long)kL * bd.nz, mr = (long long)kW * bd.nz;
    for (int bj = 0; bj < bd.BY; ++bj)
      for (int bi = 0; bi < bd.BX; ++bi) {
        const int r = bi + bd.BX * bj;
        BrickDesc k{};
        k.slot = slot + (long long)r * bd.ns;
        k.pslot = phi_slot(bd, r);
        k.pW = bi > 0 ? phi_slot(bd, r - 1) : phi_slot(bd, bd.nbricks + bj);
        k.pE = bi + 1 < bd.BX ? phi_slot(bd, r + 1) : bd.gE ? phi_slot(bd, bd.nbricks + bd.BY + bj) : k.pslot;
        k.pS = bj > 0 ? phi_slot(bd, r - bd.BX) : phi_slot(bd, bd.nbricks + bd.BY * (1 + bd.gE) + bi);
        k.pN = bj + 1 < bd.BY ? phi_slot(bd, r + bd.BX)
               : bd.gN ? phi_slot(bd, bd.nbricks + bd.BY * (1 + bd.gE) + bd.BX + bi) : k.pslot;
        k.medge = medge + r * me;
        k.mrow = mrow + r * mr;
        k.mWe = bi > 0 ? medge + (r - 1) * me : -1;
        k.mEe = bi + 1 < bd.BX ? medge + (r + 1) * me : -1;
        k.mSr = bj > 0 ? mrow + (r - bd.BX) * mr : -1;
        k.mNr = bj + 1 < bd.BY ? mrow + (r + bd.BX) * mr : -1;
        k.block = (int)lb;
        k.bi = bi; k.bj = bj;
        k.i0 = bi * kW; k.j0 = bj * kL;
        k.wI = std::min(kW, bd.nx - k.i0);
        k.wJ = std::min(kL, bd.ny - k.j0);
        k.nz = bd.nz;
        k.ns = bd.ns;
        ctx->hbricks.push_back(k);
      }
    slot += (long long)bd.nbricks * bd.ns;
    pslot += (long long)phi_bricks(bd) * phi_stride(bd);
    medge += (long long)bd.nbricks * me;
    mrow += (long long)bd.nbricks * mr;
    ctx->hblocks.push_back(bd);
    ctx->gmax = std::max(ctx->gmax, field3_elems(bd));
  }
  ctx->total_slices = slot;
  ctx->total_phi_slices = pslot;
  ctx->total_edge = medge;
  ctx->total_row = mrow;
  const int nt = (int)ctx->hbricks.size();
  // topological ticket order: a brick lags its W neighbour by about one
  // stage plus the hand-off latency and its S neighbour by about kL steps,
  // so order by bi + 2 bj (ties: block, then bi)
  std::vector<std::tuple<int, int, int, int>> keys;
  for (int t = 0; t < nt; ++t) {
    const BrickDesc& k = ctx->hbricks[t];
    keys.emplace_back(k.bi + 2 * k.bj, k.block, k.bi, t);
  }
  std::sort(keys.begin(), keys.end());
  for (auto& k : keys) ctx->order_f.push_back(std::get<3>(k));
  ctx->order_b.assign(ctx->order_f.rbegin(), ctx->order_f.rend());

  const size_t es = ctx->esize;
  CKS(dalloc(ctx, &ctx->d_blocks, sizeof(BlockDesc) * std::max<size_t>(1, ctx->hblocks.size())));
  CKS(dalloc(ctx, &ctx->d_bricks, sizeof(BrickDesc) * std::max(1, nt)));
  CKS(dalloc(ctx, &ctx->d_order_f, sizeof(int) * std::max(1, nt)));
  CKS(dalloc(ctx, &ctx->d_order_b, sizeof(int) * std::max(1, nt)));
  if (nt) {
    CK(cudaMemcpy(ctx->d_blocks, ctx->hblocks.data(), sizeof(BlockDesc) * ctx->hblocks.size(),
                  cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_bricks, ctx->hbricks.data(), sizeof(BrickDesc) * nt, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_order_f, ctx->order_f.data(), sizeof(int) * nt, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_order_b, ctx->order_b.data(), sizeof(int) * nt, cudaMemcpyHostToDevice));
  }
  const size_t S = (size_t)ctx->total_slices * kL;
  CKS(dalloc(ctx, &ctx->fw, S * F_NA * es));
  CKS(dalloc(ctx, &ctx->bw, S * B_NA * es));
  CKS(dalloc(ctx, &ctx->R, S * es));
  CKS(dalloc(ctx, &ctx->phi, (size_t)ctx->total_phi_slices * kL * es));
  if (ctx->precision == SIP_PREC_SINGLE) {
    CKS(dalloc(ctx, &ctx->coef64, S * C_NA * sizeof(double)));
    ctx->coef_na = C_NA;
  } else {
    ctx->coef64 = static_cast<double*>(ctx->fw);
    ctx->coef_na = F_NA;
  }
  // mailboxes: edge entries (kL * nz per brick) and row entries (kW * nz per
  // brick); words per entry: es / 4 (K2, K3), 6 (K1: three fp64 values)
  const size_t ew = es / 4;
  const size_t words[6] = {ew * ctx->total_edge, ew * ctx->total_row, ew * ctx->total_edge,
                           ew * ctx->total_row, 6 * (size_t)ctx->total_edge, 6 * (size_t)ctx->total_row};
  for (int m = 0; m < 6; ++m) {
    ctx->mbox_bytes[m] = std::max<size_t>(1, words[m]) * sizeof(unsigned long long);
    CKS(dalloc(ctx, &ctx->mbox[m], ctx->mbox_bytes[m]));
    // tag 0xFFFFFFFF never matches a live epoch
    CK(cudaMemset(ctx->mbox[m], 0xff, ctx->mbox_bytes[m]));
  }
  CKS(dalloc(ctx, &ctx->epochs, 4 * sizeof(unsigned)));
  CKS(dalloc(ctx, &ctx->d_norm_it, sizeof(unsigned)));
  CKS(dalloc(ctx, &ctx->d_ctl, 4 * sizeof(unsigned)));
  CKS(dalloc(ctx, &ctx->d_xflag, 2 * sizeof(unsigned) * std::max(1, nt)));
  CKS(dalloc(ctx, &ctx->d_xseq, sizeof(unsigned)));
  if (const char* xs = getenv("SIPB_XSPLIT")) ctx->xsplit = atoi(xs) != 0;
  // CUDA-graph replay of sip_iterate is opt-in (SIPB_GRAPH=1): the two
  // launches per iteration are already enqueued back to back
  if (const char* gr = getenv("SIPB_GRAPH")) ctx->use_graphs = atoi(gr) != 0;
  const size_t st = 32;
  CKS(dalloc(ctx, &ctx->st_f, st * sizeof(unsigned)));
  CKS(dalloc(ctx, &ctx->st_b, st * sizeof(unsigned)));
  CKS(dalloc(ctx, &ctx->st_fac, st * sizeof(unsigned)));
  CKS(dalloc(ctx, &ctx->partial, sizeof(double) * std::max(1, nt)));
  CKS(dalloc(ctx, &ctx->d_bad, sizeof(unsigned long long)));
  CKS(dalloc(ctx, &ctx->staging, sizeof(double) * 8 * std::max<size_t>(1, ctx->gmax)));
  size_t pst = 0;
  for (const BlockDesc& b : ctx->hblocks) {
    ctx->phi_stage_off.push_back(pst);
    pst += field3_elems(b);
  }
  CKS(dalloc(ctx, &ctx->phi_stage, sizeof(double) * std::max<size_t>(1, pst)));

  int cap = 0;
  CKS(max_resident_ctas(1, ctx->precision, &cap));
  ctx->grid_f = std::max(1, std::min(nt, cap));
  CKS(max_resident_ctas(2, ctx->precision, &cap));
  ctx->grid_b = std::max(1, std::min(nt, cap));
  CKS(max_resident_ctas(0, ctx->precision, &cap));
  ctx->grid_fac = std::max(1, std::min(nt, cap));
  if (const char* g = getenv("SIPB_GRID")) {  // debugging: cap the persistent grid
    const int gg = std::max(1, atoi(g));
    ctx->grid_f = std::min(ctx->grid_f, gg);
    ctx->grid_b = std::min(ctx->grid_b, gg);
    ctx->grid_fac = std::min(ctx->grid_fac, gg);
  }

  // halo plan: faces only, canonical order (transfers.cpp:148-165)
  std::vector<HaloEntry> plan;
  plan_halo(ctx->L, ctx->rank_of, ctx->rank, plan);
  CKS(install_plan(ctx, plan));
  CK(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
  ctx->stream = ctx->own_stream;
  return SIP_OK;
}

static int create_common(int device, int gnx, int gny, int gnz, int px, int py, int pz,
                         const int* block_rank, int rank, int nranks, const void* nccl_id,
                         int precision, sip_ctx** out) {
  if (!out) return SIP_ERR_CONFIG;
  *out = nullptr;
  if (precision != SIP_PREC_DOUBLE && precision != SIP_PREC_SINGLE) {
    g_create_err = "precision must be SIP_PREC_DOUBLE or SIP_PREC_SINGLE";
    return SIP_ERR_CONFIG;
  }
  if (nranks < 1 || rank < 0 || rank >= nranks) {
    g_create_err = "rank out of range";
    return SIP_ERR_CONFIG;
  }
  sip_ctx* ctx = new sip_ctx();
  ctx->device = device;
  ctx->precision = precision;
  ctx->esize = precision == SIP_PREC_DOUBLE ? 8 : 4;
  ctx->rank = rank;
  ctx->nranks = nranks;
  std::string err;
  if (!build_lattice(gnx, gny, gnz, px, py, pz, ctx->L, err)) {
    g_create_err = err;
    delete ctx;
    return SIP_ERR_CONFIG;
  }
  const int nb = px * py * pz;
  if (block_rank) {
    ctx->rank_of.assign(block_rank, block_rank + nb);
    for (int r : ctx->rank_of)
      if (r < 0 || r >= nranks) {
        g_create_err = "block_rank entry out of range";
        delete ctx;
        return SIP_ERR_CONFIG;
      }
  } else if (!plan_block_ranks(px, py, pz, nranks, ctx->rank_of)) {
    g_create_err = "cannot place " + std::to_string(nb) + " blocks on " + std::to_string(nranks) +
                   " ranks";
    delete ctx;
    return SIP_ERR_CONFIG;
  }
  if (nranks == 1 && getenv("SIPB_NCCL_SELF")) ctx->nccl_self = atoi(getenv("SIPB_NCCL_SELF")) != 0;
  int s = set_device(ctx);
  if (s == SIP_OK) s = build(ctx);
  if (s == SIP_OK && ctx->nccl_self) {  // 1-rank communicator for the self-exchange test mode
    ncclUniqueId id;
    if (!nccl().ok) {
      ctx->err = nccl().err;
      s = SIP_ERR_NCCL;
    } else if (nccl().GetUniqueId(&id) != ncclSuccess ||
               nccl().CommInitRank(&ctx->comm, 1, id, 0) != ncclSuccess) {
      ctx->err = "ncclCommInitRank (self mode) failed";
      s = SIP_ERR_NCCL;
    }
  }
  if (s == SIP_OK && nranks > 1) {
    if (!nccl_id) {
      ctx->err = "nccl_id required when nranks > 1";
      s = SIP_ERR_CONFIG;
    } else {
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      if (!nccl().ok) {
        ctx->err = nccl().err;
        s = SIP_ERR_NCCL;
      } else {
        ncclResult_t r = nccl().CommInitRank(&ctx->comm, nranks, id, rank);
        if (r != ncclSuccess) {
          ctx->err = std::string("ncclCommInitRank: ") + nccl().GetErrorString(r);
          s = SIP_ERR_NCCL;
        }
      }
    }
  }
  if (s != SIP_OK) {
    g_create_err = ctx->err;
    sip_destroy(ctx);
    return s;
  }
  *out = ctx;
  return SIP_OK;
}

// ------------------------------------------------------------------ helpers
static int ensure_norm_cap(sip_ctx* ctx, int need) {
  if (need <= ctx->norm_cap) return SIP_OK;
  const int cap = std::max(need, std::max(64, 2 * ctx->norm_cap));
  const int nl = std::max<int>(1, (int)ctx->local.size());
  double *n = nullptr, *bn = nullptr;
  CK(cudaStreamSynchronize(ctx->stream));
  CKS(dalloc(ctx, &n, sizeof(double) * cap));
  CKS(dalloc(ctx, &bn, sizeof(double) * cap * nl));
  if (ctx->d_norms) {
    CK(cudaMemcpy(n, ctx->d_norms, sizeof(double) * ctx->norm_cap, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(bn, ctx->d_bnorms, sizeof(double) * ctx->norm_cap * nl, cudaMemcpyDeviceToDevice));
    cudaFree(ctx->d_norms);
    cudaFree(ctx->d_bnorms);
  }
  ctx->d_norms = n;
  ctx->d_bnorms = bn;
  ctx->norm_cap = cap;
  return SIP_OK;
}

// split exchange in use: enabled, and some transfer's source is final before K3 ends
static bool use_xsplit(const sip_ctx* ctx) {
  return ctx->xsplit && (ctx->x_early > 0 || ctx->ux_early > 0);
}

template <typename T>
static SweepParams<T> sweep_params(sip_ctx* ctx, bool forward) {
  SweepParams<T> p{};
  p.bricks = ctx->d_bricks;
  p.blocks = ctx->d_blocks;
  p.order = forward ? ctx->d_order_f : ctx->d_order_b;
  p.nbricks = (int)ctx->hbricks.size();
  p.nblocks = (int)ctx->hblocks.size();
  p.fw = static_cast<T*>(ctx->fw);
  p.bw = static_cast<T*>(ctx->bw);
  p.phi = static_cast<T*>(ctx->phi);
  p.R = static_cast<T*>(ctx->R);
  p.mA = ctx->mbox[forward ? 0 : 2];
  p.mB = ctx->mbox[forward ? 1 : 3];
  p.epoch = ctx->epochs + (forward ? 0 : 1);
  p.state = forward ? ctx->st_f : ctx->st_b;
  p.state_other = forward ? ctx->st_b : ctx->st_f;
  p.partial = ctx->partial;
  // the iteration's norm slot comes from the device counter d_norm_it
  p.norms_base = ctx->d_norms;
  p.bnorms_base = ctx->d_bnorms;
  p.norm_it = ctx->d_norm_it;
  p.target = ctx->solve_target;
  p.ctl = ctx->d_ctl;
  if (use_xsplit(ctx)) {  // K2 bumps the stamp value, K3 stamps
    p.xseq = ctx->d_xseq;
    p.xflag = forward ? nullptr : ctx->d_xflag;
  }
  p.trace = ctx->trace ? ctx->trace + (forward ? 0 : 4 * ctx->hbricks.size()) : nullptr;
  p.trace_brick = ctx->trace_brick;
  return p;
}

static void ev_begin(sip_ctx* ctx, int kind, cudaEvent_t* a) {
  if (!ctx->prof) return;
  cudaEvent_t b;
  cudaEventCreate(a);
  cudaEventCreate(&b);
  cudaEventRecord(*a, ctx->stream);
  ctx->events.emplace_back(kind, *a, b);
}
static void ev_end(sip_ctx* ctx) {
  if (!ctx->prof) return;
  cudaEventRecord(std::get<2>(ctx->events.back()), ctx->stream);
}

// NCCL phase of the exchange: per peer, elements [b, e) of the message
// (0 / s1 / count); all receives and sends posted in one group, matched per
// peer in issue order (non-blocking exchange)
template <typename T>
static int nccl_phase(sip_ctx* ctx, int phase, cudaStream_t st) {
  const ncclDataType_t dt = sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
  const size_t es = sizeof(T);
  CKN(nccl().GroupStart());
  for (Peer& p : ctx->peers) {
    const long long rb = phase == 2 ? p.r1 : 0, re = phase == 1 ? p.r1 : p.count;
    const long long sb = phase == 2 ? p.s1 : 0, se = phase == 1 ? p.s1 : p.count;
    if (re > rb)
      CKN(nccl().Recv(static_cast<char*>(p.rbuf) + rb * es, (size_t)(re - rb), dt, p.rank, ctx->comm, st));
    if (se > sb)
      CKN(nccl().Send(static_cast<char*>(p.sbuf) + sb * es, (size_t)(se - sb), dt, p.rank, ctx->comm, st));
  }
  CKN(nccl().GroupEnd());
  return SIP_OK;
}

// The whole exchange on ctx->stream: local copies + packs, NCCL (phase 0 =
// whole messages), unpacks.
template <typename T>
int sipb::exchange(sip_ctx* ctx) {
  const int nx = ctx->x_early + ctx->x_late, nux = ctx->ux_early + ctx->ux_late;
  if (nx == 0 && nux == 0) return SIP_OK;
  cudaEvent_t e;
  ev_begin(ctx, 2, &e);
  T* phi = static_cast<T*>(ctx->phi);
  if (nx) {
    CKS(launch_face_copies<T>(ctx->d_x, nx, ctx->x_max_plane, ctx->d_blocks, phi, nullptr,
                              static_cast<T*>(ctx->x_sbuf), ctx->stream));
    ++ctx->launches;
  }
  if (!ctx->peers.empty()) {
    CKS(nccl_phase<T>(ctx, 0, ctx->stream));
    if (nux) {
      CKS(launch_face_copies<T>(ctx->d_ux, nux, ctx->x_max_plane, ctx->d_blocks, phi,
                                static_cast<T*>(ctx->x_rbuf), nullptr, ctx->stream));
      ++ctx->launches;
    }
  }
  ev_end(ctx);
  return SIP_OK;
}

// The exchange split around K3, enqueued right after K3 on
// ctx->stream (ev_k2 recorded between K2 and K3).  Comm stream: from the end
// of K2, the early copies / packs (waiting on K3's per-brick stamps), NCCL
// phase 1, early unpacks -- all while K3 runs; then, after K3, the late
// copies / packs, NCCL phase 2, late unpacks.  ctx->stream waits for it
// before the next K2.  The profiled halo time (kind 2) is the exposed part:
// from the end of K3 to the end of the exchange.
template <typename T>
static int exchange_split(sip_ctx* ctx) {
  cudaEvent_t e;
  ev_begin(ctx, 2, &e);
  T* phi = static_cast<T*>(ctx->phi);
  const cudaStream_t xs = ctx->xstream;
  T* sbuf = static_cast<T*>(ctx->x_sbuf);
  T* rbuf = static_cast<T*>(ctx->x_rbuf);
  CK(cudaStreamWaitEvent(xs, ctx->ev_k2, 0));
  if (ctx->x_early) {
    unsigned long long* xt =
        ctx->trace ? ctx->trace + 8 * ctx->hbricks.size() + 5 * kTraceStages * kTraceMarks : nullptr;
    CKS(launch_face_copies_after<T>(ctx->d_x, ctx->d_xitems, ctx->n_xitems, ctx->d_blocks, phi, sbuf,
                                    ctx->d_xflag, ctx->d_xseq, xt, xs));
    ++ctx->launches;
  }
  if (!ctx->peers.empty()) {
    CKS(nccl_phase<T>(ctx, 1, xs));
    if (ctx->ux_early) {
      CKS(launch_face_copies<T>(ctx->d_ux, ctx->ux_early, ctx->x_max_plane, ctx->d_blocks, phi, rbuf,
                                nullptr, xs));
      ++ctx->launches;
    }
  }
  CK(cudaEventRecord(ctx->ev_k3, ctx->stream));
  CK(cudaStreamWaitEvent(xs, ctx->ev_k3, 0));
  if (ctx->x_late) {
    CKS(launch_face_copies<T>(ctx->d_x + ctx->x_early, ctx->x_late, ctx->x_max_plane, ctx->d_blocks, phi,
                              nullptr, sbuf, xs));
    ++ctx->launches;
  }
  if (!ctx->peers.empty()) {
    CKS(nccl_phase<T>(ctx, 2, xs));
    if (ctx->ux_late) {
      CKS(launch_face_copies<T>(ctx->d_ux + ctx->ux_early, ctx->ux_late, ctx->x_max_plane, ctx->d_blocks,
                                phi, rbuf, nullptr, xs));
      ++ctx->launches;
    }
  }
  CK(cudaEventRecord(ctx->ev_x, xs));
  CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_x, 0));
  ev_end(ctx);
  return SIP_OK;
}

template <typename T>
static int launch_iterations_impl(sip_ctx* ctx, int iters);
template <typename T>
static int launch_iterations(sip_ctx* ctx, int iters) {
  const int s = launch_iterations_impl<T>(ctx, iters);
  if (s != SIP_OK) ctx->failed = true;
  return s;
}
template <typename T>
static int launch_iterations_impl(sip_ctx* ctx, int iters) {
  for (int n = 0; n < iters; ++n) {
    (void)n;
    cudaEvent_t e;
    ev_begin(ctx, 0, &e);
    CKS(launch_forward<T>(sweep_params<T>(ctx, true), ctx->grid_f, ctx->stream));
    ++ctx->launches;
    ev_end(ctx);
    const bool split = use_xsplit(ctx);
    if (split) CK(cudaEventRecord(ctx->ev_k2, ctx->stream));
    ev_begin(ctx, 1, &e);
    CKS(launch_backward<T>(sweep_params<T>(ctx, false), ctx->grid_b, ctx->stream));
    ++ctx->launches;
    ev_end(ctx);
    if (split) CKS(exchange_split<T>(ctx));
    else CKS(exchange<T>(ctx));
  }
  return SIP_OK;
}

static void drop_graph(sip_ctx* ctx) {
  if (ctx->graph_exec) cudaGraphExecDestroy(ctx->graph_exec);
  ctx->graph_exec = nullptr;
  ctx->graph_iters = -1;
}

// `iters` iterations.  Single-rank contexts without profiling / tracing replay
// a CUDA graph of the whole call (edge records, K2, K3 and the local halo
// copies of every iteration): captured on the first call with this iteration
// count, re-captured when the halo plan, the norm buffers, the stream or the
// kernel variant change.  Norm slots come from the device counter, so the
// replay needs no new parameters.
template <typename T>
int sipb::iterate_t(sip_ctx* ctx, int iters) {
  if (ctx->failed) {
    ctx->err = "an earlier sweep launch failed part-way: sip_load_phi (or sip_solve) resets the context";
    return SIP_ERR_CUDA;
  }
  CKS(ensure_norm_cap(ctx, ctx->n_done + iters));
  const int sym = 0;  // one forward kernel for general and symmetric systems
  const bool graph = ctx->use_graphs && iters > 0 && !ctx->prof && !ctx->trace && ctx->peers.empty();
  if (!graph) {
    CKS(launch_iterations<T>(ctx, iters));
  } else {
    if (!(ctx->graph_exec && ctx->graph_iters == iters && ctx->graph_plan == ctx->plan_gen &&
          ctx->graph_norms == ctx->d_norms && ctx->graph_stream == ctx->stream &&
          ctx->graph_sym == sym)) {
      drop_graph(ctx);
      const long long l0 = ctx->launches;
      CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
      const int st = launch_iterations<T>(ctx, iters);
      cudaGraph_t g = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(ctx->stream, &g);
      if (st != SIP_OK) {
        if (g) cudaGraphDestroy(g);
        return st;
      }
      CK(ec);
      const cudaError_t ei = cudaGraphInstantiate(&ctx->graph_exec, g, 0);
      cudaGraphDestroy(g);
      CK(ei);
      ctx->graph_launches = ctx->launches - l0;
      ctx->launches = l0;
      ctx->graph_iters = iters;
      ctx->graph_plan = ctx->plan_gen;
      ctx->graph_norms = ctx->d_norms;
      ctx->graph_stream = ctx->stream;
      ctx->graph_sym = sym;
    }
    CK(cudaGraphLaunch(ctx->graph_exec, ctx->stream));
    ctx->launches += ctx->graph_launches;
  }
  ctx->n_done += iters;
  return SIP_OK;
}

int sipb::check_ready(sip_ctx* ctx) {
  if (!ctx->factored) {
    ctx->err = "solve before sip_factor (no factors for this system)";
    return SIP_ERR_MISUSE;
  }
  if (ctx->factor_stamp != ctx->revision) {
    ctx->err = "factors stamped with revision " + std::to_string(ctx->factor_stamp) +
               " used against system revision " + std::to_string(ctx->revision);
    return SIP_ERR_STALE;
  }
  return SIP_OK;
}

// One Field3 array (device staging) of a local block into the packs: the
// forward pack in the context precision and, in single mode, the fp64
// coefficient pack the factorisation reads (AP..AT; Q is not needed there).
int sipb::scatter_array(sip_ctx* ctx, int local, const double* src, int arr) {
  const BlockDesc& hb = ctx->hblocks[local];
  if (ctx->precision == SIP_PREC_SINGLE) {
    CKS(launch_scatter<float>(src, ctx->d_blocks, local, hb, static_cast<float*>(ctx->fw), F_NA, arr,
                              ctx->stream));
    if (arr < C_NA) CKS(launch_scatter<double>(src, ctx->d_blocks, local, hb, ctx->coef64, C_NA, arr, ctx->stream));
  } else {
    CKS(launch_scatter<double>(src, ctx->d_blocks, local, hb, static_cast<double*>(ctx->fw), F_NA, arr,
                               ctx->stream));
  }
  return SIP_OK;
}

template <typename T>
static FactorParams<T> factor_params(sip_ctx* ctx, double alpha) {
  FactorParams<T> fp{};
  fp.bricks = ctx->d_bricks;
  fp.blocks = ctx->d_blocks;
  fp.order = ctx->d_order_f;
  fp.nbricks = (int)ctx->hbricks.size();
  fp.alpha = alpha;
  fp.coef = ctx->coef64;
  fp.coef_na = ctx->coef_na;
  fp.fw = static_cast<T*>(ctx->fw);
  fp.bw = static_cast<T*>(ctx->bw);
  fp.mA = ctx->mbox[4];
  fp.mB = ctx->mbox[5];
  fp.epoch = ctx->epochs + 2;
  fp.state = ctx->st_fac;
  fp.bad = ctx->d_bad;
  return fp;
}

template int sipb::exchange<float>(sip_ctx*);
template int sipb::exchange<double>(sip_ctx*);
template int sipb::iterate_t<float>(sip_ctx*, int);
template int sipb::iterate_t<double>(sip_ctx*, int);

// =================================================================== C-ABI
extern "C" {

const char* sip_version(void) {
  return "b200-sip 0.3 (sm_100a, 8x32-column brick wavefront K1/K2/K3: warp-specialised TMA-fed rings, tagged cross-brick mailboxes, NCCL face halos, pressure-correction caller)";
}

const char* sip_status_string(int s) {
  switch (s) {
    case SIP_OK: return "ok";
    case SIP_ERR_SINGULAR: return "singular factorization";
    case SIP_ERR_STALE: return "stale factors";
    case SIP_ERR_MISUSE: return "misuse";
    case SIP_ERR_CONFIG: return "invalid configuration";
    case SIP_ERR_CUDA: return "CUDA error";
    case SIP_ERR_NCCL: return "NCCL error";
    case SIP_ERR_NOMEM: return "device out of memory";
    case SIP_ERR_FORMAT: return "malformed transfer table";
    case SIP_ERR_PROTOCOL: return "transfer table protocol violation";
    case SIP_ERR_NOCONV: return "pressure correction did not converge";
    default: return "unknown status";
  }
}

const char* sip_last_error(const sip_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_err.c_str();
}

int sip_create(int device, int nx, int ny, int nz, int precision, sip_ctx** out) {
  return create_common(device, nx, ny, nz, 1, 1, 1, nullptr, 0, 1, nullptr, precision, out);
}

int sip_create_lattice(int device, int gnx, int gny, int gnz, int px, int py, int pz,
                       const int* block_rank, int rank, int nranks, const void* nccl_id,
                       int precision, sip_ctx** out) {
  return create_common(device, gnx, gny, gnz, px, py, pz, block_rank, rank, nranks, nccl_id,
                       precision, out);
}

int sip_destroy(sip_ctx* ctx) {
  if (!ctx) return SIP_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->comm) nccl().CommDestroy(ctx->comm);
  for (auto& e : ctx->events) {
    cudaEventDestroy(std::get<1>(e));
    cudaEventDestroy(std::get<2>(e));
  }
  void* ptrs[] = {ctx->d_blocks, ctx->d_bricks, ctx->d_order_f, ctx->d_order_b, ctx->fw, ctx->bw,
                  ctx->phi, ctx->R, ctx->st_f, ctx->st_b, ctx->st_fac, ctx->partial, ctx->d_norms,
                  ctx->d_bnorms, ctx->d_bad, ctx->staging, ctx->d_local_copies, ctx->phi_stage,
                  ctx->trace, ctx->epochs, ctx->d_gather, ctx->d_norm_it, ctx->d_pad, ctx->d_ctl};
  if (ctx->graph_exec) cudaGraphExecDestroy(ctx->graph_exec);
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto* m : ctx->mbox)
    if (m) cudaFree(m);
  if (ctx->precision == SIP_PREC_SINGLE && ctx->coef64) cudaFree(ctx->coef64);
  if (ctx->h_pad) cudaFreeHost(ctx->h_pad);
  for (Peer& p : ctx->peers) {
    if (p.d_pack) cudaFree(p.d_pack);
    if (p.d_unpack) cudaFree(p.d_unpack);
  }
  for (void* q : {(void*)ctx->d_x, (void*)ctx->d_ux, ctx->x_sbuf, ctx->x_rbuf, (void*)ctx->d_xflag,
                  (void*)ctx->d_xseq, (void*)ctx->d_xitems})
    if (q) cudaFree(q);
  if (ctx->cstream) {
    cudaStreamSynchronize(ctx->cstream);
    cudaStreamDestroy(ctx->cstream);
  }
  for (auto& a : ctx->ev_qcopy)
    for (auto e : a) cudaEventDestroy(e);
  for (auto& a : ctx->ev_qscat)
    for (auto e : a) cudaEventDestroy(e);
  if (ctx->q_stage) cudaFree(ctx->q_stage);
  if (ctx->phi_stage2) cudaFree(ctx->phi_stage2);
  for (AsyncSolve& a : ctx->async) {
    if (a.h_norms) cudaFreeHost(a.h_norms);
    if (a.done) cudaEventDestroy(a.done);
    if (a.h2d) cudaEventDestroy(a.h2d);
    for (auto e : a.chunk_ev) cudaEventDestroy(e);
  }
  if (ctx->xstream) {
    cudaStreamSynchronize(ctx->xstream);
    cudaStreamDestroy(ctx->xstream);
    cudaEventDestroy(ctx->ev_k2);
    cudaEventDestroy(ctx->ev_k3);
    cudaEventDestroy(ctx->ev_x);
  }
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
  return SIP_OK;
}

int sip_num_local_blocks(const sip_ctx* ctx, int* n) {
  if (!ctx || !n) return SIP_ERR_MISUSE;
  *n = (int)ctx->local.size();
  return SIP_OK;
}

int sip_local_block(const sip_ctx* ctx, int local, int* block_id, int dims[3], int origin[3]) {
  if (!ctx || local < 0 || local >= (int)ctx->local.size()) return SIP_ERR_MISUSE;
  const BlockInfo& bi = ctx->L.blocks[ctx->local[local]];
  if (block_id) *block_id = ctx->local[local];
  for (int a = 0; a < 3; ++a) {
    if (dims) dims[a] = bi.n[a];
    if (origin) origin[a] = bi.lo[a];
  }
  return SIP_OK;
}

int sip_set_system(sip_ctx* ctx, int local, const double* ap, const double* aw, const double* ae,
                   const double* as, const double* an, const double* ab, const double* at,
                   const double* q) {
  if (!ctx) return SIP_ERR_MISUSE;
  if (local < 0 || local >= (int)ctx->local.size()) {
    ctx->err = "sip_set_system: local block index out of range";
    return SIP_ERR_MISUSE;
  }
  const double* src[8] = {ap, aw, ae, as, an, ab, at, q};
  const int arr[8] = {F_AP, F_AW, F_AE, F_AS, F_AN, F_AB, F_AT, F_Q};
  for (const double* s : src)
    if (!s) {
      ctx->err = "sip_set_system: null array";
      return SIP_ERR_MISUSE;
    }
  CKS(set_device(ctx));
  const BlockDesc& hb = ctx->hblocks[local];
  const size_t G = field3_elems(hb);
  for (int a = 0; a < 8; ++a) {
    CK(cudaMemcpyAsync(ctx->staging, src[a], G * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CKS(scatter_array(ctx, local, ctx->staging, arr[a]));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  ++ctx->revision;
  if (ctx->symmetric.size() != ctx->local.size()) ctx->symmetric.assign(ctx->local.size(), 0);
  ctx->symmetric[local] = 0;  // a new system is not flagged until sip_set_symmetric
  ctx->poisson = false;       // no longer the assembled pressure system
  return SIP_OK;
}

int sip_set_symmetric(sip_ctx* ctx, int local, int symmetric) {
  if (!ctx) return SIP_ERR_MISUSE;
  if (local < 0 || local >= (int)ctx->local.size()) {
    ctx->err = "sip_set_symmetric: local block index out of range";
    return SIP_ERR_MISUSE;
  }
  if (ctx->symmetric.size() != ctx->local.size()) ctx->symmetric.assign(ctx->local.size(), 0);
  if (!symmetric) {
    ctx->symmetric[local] = 0;
    return SIP_OK;
  }
  CKS(set_device(ctx));
  const BlockDesc& hb = ctx->hblocks[local];
  unsigned long long* bad = reinterpret_cast<unsigned long long*>(ctx->staging);
  CK(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), ctx->stream));
  CKS(launch_check_symmetric(ctx->d_blocks, local, hb, ctx->coef64, ctx->coef_na, bad, ctx->stream));
  ++ctx->launches;
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, bad, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (h) {
    ctx->err = "sip_set_symmetric: " + std::to_string(h) +
               " coefficient pairs violate ae(i)=aw(i+1), an(j)=as(j+1), at(k)=ab(k+1)";
    return SIP_ERR_CONFIG;
  }
  ctx->symmetric[local] = 1;
  return SIP_OK;
}

int sip_set_source(sip_ctx* ctx, int local, const double* q) {
  if (!ctx) return SIP_ERR_MISUSE;
  if (local < 0 || local >= (int)ctx->local.size() || !q) {
    ctx->err = "sip_set_source: bad arguments";
    return SIP_ERR_MISUSE;
  }
  CKS(set_device(ctx));
  const BlockDesc& hb = ctx->hblocks[local];
  CK(cudaMemcpyAsync(ctx->staging, q, field3_elems(hb) * sizeof(double), cudaMemcpyHostToDevice,
                     ctx->stream));
  CKS(scatter_array(ctx, local, ctx->staging, F_Q));
  return SIP_OK;
}

int sip_generate_system(sip_ctx* ctx, int kind, uint64_t seed) {
  if (!ctx) return SIP_ERR_MISUSE;
  if (kind != 0 && kind != 2 && kind != 3) {
    ctx->err = "generator kind must be 0, 2 or 3 (symmetric)";
    return SIP_ERR_CONFIG;
  }
  CKS(set_device(ctx));
  const int arr[8] = {F_AP, F_AW, F_AE, F_AS, F_AN, F_AB, F_AT, F_Q};
  for (size_t lb = 0; lb < ctx->local.size(); ++lb) {
    const BlockDesc& hb = ctx->hblocks[lb];
    const BlockInfo& bi = ctx->L.blocks[ctx->local[lb]];
    const size_t G = field3_elems(hb);
    double* out8[8];
    for (int a = 0; a < 8; ++a) out8[a] = ctx->staging + a * G;
    CK(cudaMemsetAsync(ctx->staging, 0, 8 * G * sizeof(double), ctx->stream));
    const int g[3] = {ctx->L.g[0], ctx->L.g[1], ctx->L.g[2]};
    CKS(launch_generate(kind, seed + (uint64_t)ctx->local[lb], g, bi.lo.data(), hb.nx, hb.ny, hb.nz, out8,
                        ctx->stream));
    for (int a = 0; a < 8; ++a) CKS(scatter_array(ctx, (int)lb, out8[a], arr[a]));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  ++ctx->revision;
  ctx->symmetric.assign(ctx->local.size(), 0);  // generated systems are not flagged
  ctx->poisson = false;
  return SIP_OK;
}

int sip_factor(sip_ctx* ctx, double alpha, long long* bad_block, long long* bad_cell) {
  if (!ctx) return SIP_ERR_MISUSE;
  if (!(alpha >= 0.0 && alpha < 1.0)) {
    ctx->err = "alpha must be in [0, 1) (SPEC.md:124-127)";
    return SIP_ERR_CONFIG;
  }
  CKS(set_device(ctx));
  const int nt = (int)ctx->hbricks.size();
  CK(cudaMemsetAsync(ctx->st_fac, 0, 32 * sizeof(unsigned), ctx->stream));
  CK(cudaMemsetAsync(ctx->d_bad, 0xff, sizeof(unsigned long long), ctx->stream));
  if (nt) {
    if (ctx->precision == SIP_PREC_SINGLE)
      CKS(launch_factor<float>(factor_params<float>(ctx, alpha), ctx->grid_fac, ctx->stream));
    else
      CKS(launch_factor<double>(factor_params<double>(ctx, alpha), ctx->grid_fac, ctx->stream));
    ++ctx->launches;
    ++ctx->factor_count;
  }
  unsigned long long bad = ~0ULL;
  CK(cudaMemcpyAsync(&bad, ctx->d_bad, sizeof(bad), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (bad != ~0ULL) {
    const long long blk = (long long)(bad >> 40), cell = (long long)(bad & ((1ULL << 40) - 1));
    if (bad_block) *bad_block = blk;
    if (bad_cell) *bad_cell = cell;
    ctx->factored = false;
    ctx->err = "singular factorization: |pivot| < 1e-30 at block " + std::to_string(blk) +
               ", Field3 index " + std::to_string(cell);
    return SIP_ERR_SINGULAR;
  }
  if (bad_block) *bad_block = -1;
  if (bad_cell) *bad_cell = -1;
  ctx->factored = true;
  ctx->factor_stamp = ctx->revision;
  ctx->alpha = alpha;
  return SIP_OK;
}

// phi0 into the device mirror `stage` (copy == false: already there) and the
// brick layout; resets the iteration state.
static int load_phi_into(sip_ctx* ctx, double* const* phi, double* stage, bool copy) {
  if (!ctx || !phi) return SIP_ERR_MISUSE;
  CKS(set_device(ctx));
  for (size_t lb = 0; lb < ctx->local.size(); ++lb) {
    if (!phi[lb]) {
      ctx->err = "sip_load_phi: null phi";
      return SIP_ERR_MISUSE;
    }
    const BlockDesc& hb = ctx->hblocks[lb];
    double* st = stage + ctx->phi_stage_off[lb];
    // Field3 -> device mirror (keeps the caller's ghost layer for the store)
    if (copy)
      CK(cudaMemcpyAsync(st, phi[lb], field3_elems(hb) * sizeof(double), cudaMemcpyHostToDevice,
                         ctx->stream));
    if (ctx->precision == SIP_PREC_SINGLE)
      CKS(launch_phi_in<float>(st, ctx->d_blocks, (int)lb, hb, static_cast<float*>(ctx->phi), ctx->stream));
    else
      CKS(launch_phi_in<double>(st, ctx->d_blocks, (int)lb, hb, static_cast<double*>(ctx->phi), ctx->stream));
    ++ctx->launches;
  }
  // interface ghosts <- neighbours' phi0 (the exchange that precedes sweep 1)
  int s = ctx->precision == SIP_PREC_SINGLE ? exchange<float>(ctx) : exchange<double>(ctx);
  ctx->n_done = 0;
  CK(cudaMemsetAsync(ctx->d_norm_it, 0, sizeof(unsigned), ctx->stream));
  CK(cudaMemsetAsync(ctx->d_ctl, 0, 4 * sizeof(unsigned), ctx->stream));
  if (ctx->failed) {  // device sweep state back to "no sweep in flight"
    CK(cudaMemsetAsync(ctx->st_f, 0, 32 * sizeof(unsigned), ctx->stream));
    CK(cudaMemsetAsync(ctx->st_b, 0, 32 * sizeof(unsigned), ctx->stream));
    ctx->failed = false;
  }
  return s;
}

int sip_load_phi(sip_ctx* ctx, double* const* phi) {
  return ctx ? load_phi_into(ctx, phi, ctx->phi_stage, true) : SIP_ERR_MISUSE;
}

int sip_store_phi(sip_ctx* ctx, double* const* phi) {
  if (!ctx || !phi) return SIP_ERR_MISUSE;
  CKS(set_device(ctx));
  for (size_t lb = 0; lb < ctx->local.size(); ++lb) {
    const BlockDesc& hb = ctx->hblocks[lb];
    double* st = ctx->phi_stage + ctx->phi_stage_off[lb];
    // interior + the ghost faces the halo plan writes (interfaces, periodic
    // wraps) are overwritten; other ghosts, edges and corners keep the values
    // loaded by sip_load_phi
    const int* written = ctx->plan_ghosts[lb].data();
    if (ctx->precision == SIP_PREC_SINGLE)
      CKS(launch_gather<float>(static_cast<float*>(ctx->phi), ctx->d_blocks, (int)lb, hb, written, st,
                               ctx->stream));
    else
      CKS(launch_gather<double>(static_cast<double*>(ctx->phi), ctx->d_blocks, (int)lb, hb, written, st,
                                ctx->stream));
    ++ctx->launches;
    CK(cudaMemcpyAsync(phi[lb], st, field3_elems(hb) * sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return SIP_OK;
}

int sip_iterate(sip_ctx* ctx, int iters) {
  if (!ctx) return SIP_ERR_MISUSE;
  if (iters < 0) {
    ctx->err = "iters must be >= 0";
    return SIP_ERR_CONFIG;
  }
  CKS(check_ready(ctx));
  CKS(set_device(ctx));
  return ctx->precision == SIP_PREC_SINGLE ? iterate_t<float>(ctx, iters)
                                           : iterate_t<double>(ctx, iters);
}

int sip_read_norms(sip_ctx* ctx, int first, int count, double* norms, double* block_norms) {
  if (!ctx || first < 0 || count < 0 || first + count > ctx->n_done) {
    if (ctx) ctx->err = "sip_read_norms: range outside the iterations run";
    return SIP_ERR_MISUSE;
  }
  CKS(set_device(ctx));
  const int nl = std::max<int>(1, (int)ctx->local.size());
  std::vector<double> bn((size_t)count * nl);
  if (count) {
    CK(cudaMemcpyAsync(bn.data(), ctx->d_bnorms + (size_t)first * nl, bn.size() * sizeof(double),
                       cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  const int nb = (int)ctx->L.blocks.size();
  std::vector<double> all((size_t)count * nb, 0.0);
  if (ctx->nranks == 1) {
    for (int it = 0; it < count; ++it)
      for (int lb = 0; lb < (int)ctx->local.size(); ++lb)
        all[(size_t)it * nb + ctx->local[lb]] = bn[(size_t)it * nl + lb];
  } else {
    // all-gather every rank's block norms (Endpoint::all_reduce, net.hpp:131:
    // fixed block order makes the sum independent of the placement)
    int maxl = 0;
    std::vector<std::vector<int>> blocks_of(ctx->nranks);
    for (int b = 0; b < nb; ++b) blocks_of[ctx->rank_of[b]].push_back(b);
    for (auto& v : blocks_of) maxl = std::max<int>(maxl, (int)v.size());
    const size_t per = (size_t)count * maxl;
    // persistent gather buffers (sip_solve with a target reads one norm per
    // iteration: no allocation on that path)
    const size_t need = std::max<size_t>(1, per) * (1 + ctx->nranks);
    if (need > ctx->gather_cap) {
      if (ctx->d_gather) cudaFree(ctx->d_gather);
      ctx->d_gather = nullptr;
      ctx->gather_cap = 0;
      CKS(dalloc(ctx, &ctx->d_gather, sizeof(double) * need));
      ctx->gather_cap = need;
    }
    double* d_send = ctx->d_gather;
    double* d_recv = ctx->d_gather + std::max<size_t>(1, per);
    if (per > ctx->h_pad_cap) {
      if (ctx->h_pad) cudaFreeHost(ctx->h_pad);
      ctx->h_pad = nullptr;
      ctx->h_pad_cap = 0;
      CK(cudaMallocHost(&ctx->h_pad, per * sizeof(double)));
      ctx->h_pad_cap = per;
    }
    double* pad = ctx->h_pad;
    std::fill(pad, pad + per, 0.0);
    for (int it = 0; it < count; ++it)
      for (int lb = 0; lb < (int)ctx->local.size(); ++lb) pad[(size_t)it * maxl + lb] = bn[(size_t)it * nl + lb];
    // stream-ordered with the all-gather (the context stream is non-blocking)
    CK(cudaMemcpyAsync(d_send, pad, per * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    CKN(nccl().AllGather(d_send, d_recv, per, ncclFloat64, ctx->comm, ctx->stream));
    std::vector<double> got(per * ctx->nranks);
    CK(cudaMemcpyAsync(got.data(), d_recv, got.size() * sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (int r = 0; r < ctx->nranks; ++r)
      for (int it = 0; it < count; ++it)
        for (size_t lb = 0; lb < blocks_of[r].size(); ++lb)
          all[(size_t)it * nb + blocks_of[r][lb]] = got[per * r + (size_t)it * maxl + lb];
  }
  for (int it = 0; it < count; ++it) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += all[(size_t)it * nb + b];
    if (norms) norms[it] = s;
    if (block_norms)
      for (int b = 0; b < nb; ++b) block_norms[(size_t)it * nb + b] = all[(size_t)it * nb + b];
  }
  return SIP_OK;
}

// the oldest pending sip_solve_async: wait for it, deliver its norms
static int finish_async(sip_ctx* ctx) {
  if (ctx->async_count == 0) return SIP_OK;
  AsyncSolve& a = ctx->async[ctx->async_head];
  CK(cudaEventSynchronize(a.done));
  if (a.out) std::memcpy(a.out, a.h_norms, sizeof(double) * a.iters);
  a.out = nullptr;
  ctx->async_head ^= 1;
  --ctx->async_count;
  return SIP_OK;
}

int sip_synchronize(sip_ctx* ctx) {
  if (!ctx) return SIP_ERR_MISUSE;
  CKS(set_device(ctx));
  CK(cudaStreamSynchronize(ctx->stream));
  while (ctx->async_count) CKS(finish_async(ctx));
  return SIP_OK;
}

int sip_wait_async(sip_ctx* ctx) {
  if (!ctx) return SIP_ERR_MISUSE;
  CKS(set_device(ctx));
  return finish_async(ctx);
}

static int ensure_cstream(sip_ctx* ctx) {
  if (ctx->cstream) return SIP_OK;
  CK(cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking));
  return SIP_OK;
}

int sip_set_source_async(sip_ctx* ctx, int local, const double* q) {
  if (!ctx) return SIP_ERR_MISUSE;
  if (local < 0 || local >= (int)ctx->local.size() || !q) {
    ctx->err = "sip_set_source_async: bad arguments";
    return SIP_ERR_MISUSE;
  }
  CKS(set_device(ctx));
  CKS(ensure_cstream(ctx));
  const size_t nl = ctx->local.size();
  if (!ctx->q_stage) {
    size_t tot = 0;
    for (const BlockDesc& b : ctx->hblocks) tot += field3_elems(b);
    CKS(dalloc(ctx, &ctx->q_stage, sizeof(double) * 2 * std::max<size_t>(1, tot)));
    ctx->q_slot.assign(nl, 0);
    ctx->ev_qcopy.resize(nl);
    ctx->ev_qscat.resize(nl);
    for (size_t b = 0; b < nl; ++b)
      for (int k = 0; k < 2; ++k) {
        CK(cudaEventCreateWithFlags(&ctx->ev_qcopy[b][k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ctx->ev_qscat[b][k], cudaEventDisableTiming));
        CK(cudaEventRecord(ctx->ev_qscat[b][k], ctx->stream));  // slot free
      }
  }
  const BlockDesc& hb = ctx->hblocks[local];
  const size_t G = field3_elems(hb);
  const int k = ctx->q_slot[local];
  ctx->q_slot[local] ^= 1;
  double* st = ctx->q_stage + 2 * ctx->phi_stage_off[local] + k * G;
  // the copy may start at once (copy stream), once the scatter that last
  // read this slot is done; the scatter waits for the copy and follows the
  // work already on the context's stream
  CK(cudaStreamWaitEvent(ctx->cstream, ctx->ev_qscat[local][k], 0));
  CK(cudaMemcpyAsync(st, q, G * sizeof(double), cudaMemcpyHostToDevice, ctx->cstream));
  CK(cudaEventRecord(ctx->ev_qcopy[local][k], ctx->cstream));
  CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_qcopy[local][k], 0));
  CKS(scatter_array(ctx, local, st, F_Q));
  CK(cudaEventRecord(ctx->ev_qscat[local][k], ctx->stream));
  return SIP_OK;
}

// Up to two solves in flight, each with its own device phi mirror.  When a
// solve's phi0 buffer is the one the previous pending solve writes its result
// into, the upload goes chunk by chunk on the copy stream, each chunk as soon
// as that chunk of the previous result has arrived in host memory (the two
// directions of the link overlap).
int sip_solve_async(sip_ctx* ctx, double* const* phi, int iters, double* norms_out) {
  if (!ctx || !phi) return SIP_ERR_MISUSE;
  if (ctx->nranks != 1 || iters < 1 || ctx->async_count == 2) {
    ctx->err = ctx->async_count == 2 ? "sip_solve_async: two solves pending (sip_wait_async first)"
                                     : "sip_solve_async: single rank, iters >= 1";
    return SIP_ERR_MISUSE;
  }
  CKS(check_ready(ctx));
  CKS(set_device(ctx));
  CKS(ensure_cstream(ctx));
  const size_t nl = ctx->local.size();
  const int si = (ctx->async_head + ctx->async_count) & 1;
  AsyncSolve& a = ctx->async[si];
  if (!a.done) {
    CK(cudaEventCreateWithFlags(&a.done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&a.h2d, cudaEventDisableTiming));
    a.chunk_ev.resize(nl * kAsyncChunks);
    for (auto& e : a.chunk_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if (si == 1 && !ctx->phi_stage2) {
    size_t tot = 0;
    for (const BlockDesc& b : ctx->hblocks) tot += field3_elems(b);
    CKS(dalloc(ctx, &ctx->phi_stage2, sizeof(double) * std::max<size_t>(1, tot)));
  }
  double* const stage = si == 0 ? ctx->phi_stage : ctx->phi_stage2;
  const AsyncSolve* prev = ctx->async_count ? &ctx->async[si ^ 1] : nullptr;
  // phi0 upload: chunked after the previous result where the buffers coincide
  bool chunked = false;
  for (size_t lb = 0; lb < nl; ++lb) {
    if (!phi[lb]) {
      ctx->err = "sip_solve_async: null phi";
      return SIP_ERR_MISUSE;
    }
    const size_t G = field3_elems(ctx->hblocks[lb]);
    double* st = stage + ctx->phi_stage_off[lb];
    if (prev && prev->phi[lb] == phi[lb]) {
      const size_t per = (G + kAsyncChunks - 1) / kAsyncChunks;
      for (int c = 0; c < kAsyncChunks; ++c) {
        const size_t b = c * per, e = std::min(G, b + per);
        if (b >= e) break;
        CK(cudaStreamWaitEvent(ctx->cstream, prev->chunk_ev[lb * kAsyncChunks + c], 0));
        CK(cudaMemcpyAsync(st + b, phi[lb] + b, (e - b) * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->cstream));
      }
      chunked = true;
    } else {
      CK(cudaMemcpyAsync(st, phi[lb], G * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    }
  }
  if (chunked) {
    CK(cudaEventRecord(a.h2d, ctx->cstream));
    CK(cudaStreamWaitEvent(ctx->stream, a.h2d, 0));
  }
  CKS(load_phi_into(ctx, phi, stage, false));
  CKS(sip_iterate(ctx, iters));
  a.iters = iters;
  a.out = norms_out;
  if (norms_out) {
    if (iters > a.h_cap) {
      if (a.h_norms) cudaFreeHost(a.h_norms);
      a.h_norms = nullptr;
      CK(cudaMallocHost(&a.h_norms, sizeof(double) * iters));
      a.h_cap = iters;
    }
    CK(cudaMemcpyAsync(a.h_norms, ctx->d_norms, sizeof(double) * iters, cudaMemcpyDeviceToHost,
                       ctx->stream));
  }
  // sip_store_phi into this solve's mirror, the download in chunks
  a.phi.assign(phi, phi + nl);
  for (size_t lb = 0; lb < nl; ++lb) {
    const BlockDesc& hb = ctx->hblocks[lb];
    double* st = stage + ctx->phi_stage_off[lb];
    const int* written = ctx->plan_ghosts[lb].data();
    if (ctx->precision == SIP_PREC_SINGLE)
      CKS(launch_gather<float>(static_cast<float*>(ctx->phi), ctx->d_blocks, (int)lb, hb, written, st,
                               ctx->stream));
    else
      CKS(launch_gather<double>(static_cast<double*>(ctx->phi), ctx->d_blocks, (int)lb, hb, written, st,
                                ctx->stream));
    ++ctx->launches;
    const size_t G = field3_elems(hb), per = (G + kAsyncChunks - 1) / kAsyncChunks;
    for (int c = 0; c < kAsyncChunks; ++c) {
      const size_t b = std::min(G, c * per), e = std::min(G, b + per);
      if (e > b)
        CK(cudaMemcpyAsync(phi[lb] + b, st + b, (e - b) * sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
      CK(cudaEventRecord(a.chunk_ev[lb * kAsyncChunks + c], ctx->stream));
    }
  }
  CK(cudaEventRecord(a.done, ctx->stream));
  ++ctx->async_count;
  return SIP_OK;
}

int sip_solve_ex(sip_ctx* ctx, double* const* phi, int max_iters, double target, int check_every,
                 double* norms_out, int* iters_used) {
  if (!ctx) return SIP_ERR_MISUSE;
  if (max_iters < 1) {
    ctx->err = "max_iters must be >= 1 (SPEC.md:124-127)";
    return SIP_ERR_CONFIG;
  }
  CKS(check_ready(ctx));
  if (iters_used) *iters_used = 0;
  if (target >= 1.0) return SIP_OK;  // no-op: fi0 returned, 0 iterations
  CKS(sip_load_phi(ctx, phi));
  int used = 0;
  if (target <= 0.0) {
    CKS(sip_iterate(ctx, max_iters));
    used = max_iters;
  } else if (ctx->nranks == 1) {
    // the K2 finaliser evaluates the reduction and stops the remaining
    // sweeps on the device: no host synchronisation per sweep; the host only
    // polls the stop flag between chunks of check_every sweeps (<= 0: all
    // sweeps enqueued at once) to avoid enqueueing no-op launches
    const int chunk = check_every > 0 ? check_every : max_iters;
    ctx->solve_target = target;
    int queued = 0, st = SIP_OK;
    unsigned stop = 0;
    while (queued < max_iters && st == SIP_OK) {
      const int n = std::min(chunk, max_iters - queued);
      st = sip_iterate(ctx, n);
      queued += n;
      if (st == SIP_OK && queued < max_iters) {
        cudaError_t e = cudaMemcpyAsync(&stop, ctx->d_ctl, sizeof(stop), cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) {
          ctx->err = std::string("solve: stop flag read: ") + cudaGetErrorString(e);
          st = SIP_ERR_CUDA;
        }
        if (stop) break;
      }
    }
    ctx->solve_target = 0.0;
    CKS(st);
    unsigned done = 0;
    CK(cudaMemcpyAsync(&done, ctx->d_norm_it, sizeof(done), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    used = (int)done;
    ctx->n_done = used;  // the sweeps that ran (no-op launches do not count)
  } else {
    // several ranks: the reduction needs the global norm (all-gather of the
    // block norms), evaluated every check_every-th sweep (SPEC.md DESIGN
    // DECISIONS: norm evaluation frequency configurable)
    const int every = check_every > 0 ? check_every : 1;
    double n0 = 0.0;
    while (used < max_iters) {
      const int n = std::min(every, max_iters - used);
      CKS(sip_iterate(ctx, n));
      used += n;
      std::vector<double> nr(n);
      CKS(sip_read_norms(ctx, used - n, n, nr.data(), nullptr));
      if (used == n) n0 = nr[0];
      if (n0 == 0.0 || nr[n - 1] / n0 <= target) break;
    }
  }
  if (norms_out) CKS(sip_read_norms(ctx, 0, used, norms_out, nullptr));
  CKS(sip_store_phi(ctx, phi));
  if (iters_used) *iters_used = used;
  return SIP_OK;
}

int sip_solve(sip_ctx* ctx, double* const* phi, int max_iters, double target, double* norms_out,
              int* iters_used) {
  // single rank: exact device-side stop, stop flag polled every 8 sweeps;
  // several ranks: global norm tested after every sweep (exact stop)
  return sip_solve_ex(ctx, phi, max_iters, target, ctx && ctx->nranks > 1 ? 1 : 8, norms_out,
                      iters_used);
}

int sip_set_halo_tables(sip_ctx* ctx, int nranks, const int* counts, const int* entries) {
  if (!ctx) return SIP_ERR_MISUSE;
  if (nranks != ctx->nranks || (nranks > 0 && (!counts || !entries))) {
    ctx->err = "sip_set_halo_tables: the table set has " + std::to_string(nranks) +
               " ranks, the context " + std::to_string(ctx->nranks);
    return SIP_ERR_CONFIG;
  }
  std::vector<std::vector<std::array<int, 12>>> t(nranks);
  long long at = 0;
  for (int r = 0; r < nranks; ++r)
    for (int k = 0; k < counts[r]; ++k, ++at) {
      std::array<int, 12> row;
      for (int f = 0; f < 12; ++f) row[f] = entries[at * 12 + f];
      t[r].push_back(row);
    }
  std::string err;
  if (!ftt1_validate(t, err)) {
    ctx->err = err;
    return SIP_ERR_PROTOCOL;
  }
  CKS(set_device(ctx));
  const int nb = (int)ctx->L.blocks.size();
  std::vector<HaloEntry> plan;
  for (const auto& row : t[ctx->rank]) {
    if (row[1] != 0) continue;  // edge / corner patches: not read by the 7-point stencil
    HaloEntry e{};
    e.dir = row[0];
    e.face = row[2];
    e.peer = row[3];
    e.owner = row[4];
    e.neighbor = row[5];
    for (int a = 0; a < 3; ++a) {
      e.lo[a] = row[6 + 2 * a];
      e.hi[a] = row[7 + 2 * a];
    }
    auto bad = [&](const std::string& why) {
      ctx->err = "sip_set_halo_tables: face entry (owner " + std::to_string(e.owner) +
                 ", neighbor " + std::to_string(e.neighbor) + ", face " + std::to_string(e.face) +
                 "): " + why;
      return SIP_ERR_CONFIG;
    };
    if (e.owner < 0 || e.owner >= nb || e.neighbor < 0 || e.neighbor >= nb)
      return bad("block id outside the lattice");
    if (ctx->rank_of[e.owner] != ctx->rank) return bad("owner block is not on this rank");
    if (e.dir == 0 && ctx->rank_of[e.neighbor] != ctx->rank)
      return bad("local entry with a remote neighbor block");
    if (e.dir != 0 && ctx->rank_of[e.neighbor] != e.peer)
      return bad("peer rank does not own the neighbor block");
    // the whole face: the plane of the owner block normal to the face axis
    const BlockInfo& bi = ctx->L.blocks[e.owner];
    const int axis = e.face / 2;
    long long plane = 1;
    for (int a = 0; a < 3; ++a)
      if (a != axis) plane *= bi.n[a];
    long long cells = 1;
    for (int a = 0; a < 3; ++a) cells *= std::max(0, e.hi[a] - e.lo[a] + 1);
    if (cells != plane) return bad("partial face patches are not supported");
    const BlockInfo& bn = ctx->L.blocks[e.neighbor];
    for (int a = 0; a < 3; ++a)
      if (a != axis && bn.n[a] != bi.n[a]) return bad("non-conforming neighbor face");
    plan.push_back(e);
  }
  CK(cudaStreamSynchronize(ctx->stream));
  CKS(install_plan(ctx, plan));
  return SIP_OK;
}

int sip_residual(sip_ctx* ctx, int symmetric, double* const* res) {
  if (!ctx || !res) return SIP_ERR_MISUSE;
  if (symmetric)
    for (size_t lb = 0; lb < ctx->local.size(); ++lb)
      if (lb >= ctx->symmetric.size() || !ctx->symmetric[lb]) {
        ctx->err = "residual_symmetric: system of local block " + std::to_string(lb) +
                   " is not flagged symmetric (sip_set_symmetric)";
        return SIP_ERR_MISUSE;
      }
  CKS(set_device(ctx));
  for (size_t lb = 0; lb < ctx->local.size(); ++lb) {
    const BlockDesc& hb = ctx->hblocks[lb];
    const size_t G = field3_elems(hb);
    CK(cudaMemsetAsync(ctx->staging, 0, G * sizeof(double), ctx->stream));
    if (ctx->precision == SIP_PREC_SINGLE)
      CKS(launch_residual<float>(ctx->d_blocks, (int)lb, hb, static_cast<float*>(ctx->fw),
                                 static_cast<float*>(ctx->phi), symmetric, ctx->staging, ctx->stream));
    else
      CKS(launch_residual<double>(ctx->d_blocks, (int)lb, hb, static_cast<double*>(ctx->fw),
                                  static_cast<double*>(ctx->phi), symmetric, ctx->staging, ctx->stream));
    ++ctx->launches;
    CK(cudaMemcpyAsync(res[lb], ctx->staging, G * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return SIP_OK;
}

int sip_set_stream(sip_ctx* ctx, void* stream) {
  if (!ctx) return SIP_ERR_MISUSE;
  const cudaStream_t ns = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
  if (ns != ctx->stream) {
    // work already enqueued (sweeps, async solves, pending source scatters)
    // stays ordered before anything enqueued on the new stream
    CKS(set_device(ctx));
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaEventRecord(e, ctx->stream));
    CK(cudaStreamWaitEvent(ns, e, 0));
    cudaEventDestroy(e);  // released once the recorded work completes
    ctx->stream = ns;
  }
  return SIP_OK;
}

void* sip_get_stream(const sip_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int sip_set_profiling(sip_ctx* ctx, int on) {
  if (!ctx) return SIP_ERR_MISUSE;
  CKS(set_device(ctx));
  CK(cudaStreamSynchronize(ctx->stream));
  for (auto& e : ctx->events) {
    cudaEventDestroy(std::get<1>(e));
    cudaEventDestroy(std::get<2>(e));
  }
  ctx->events.clear();
  ctx->t_fwd = ctx->t_bwd = ctx->t_halo = 0;
  ctx->prof = on != 0;
  ctx->prof_launches = ctx->launches;
  return SIP_OK;
}

int sip_get_profile(sip_ctx* ctx, double* fwd_ms, double* bwd_ms, double* halo_ms,
                    long long* launches) {
  if (!ctx) return SIP_ERR_MISUSE;
  CKS(set_device(ctx));
  CK(cudaStreamSynchronize(ctx->stream));
  for (auto& e : ctx->events) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, std::get<1>(e), std::get<2>(e)));
    (std::get<0>(e) == 0 ? ctx->t_fwd : std::get<0>(e) == 1 ? ctx->t_bwd : ctx->t_halo) += ms;
    cudaEventDestroy(std::get<1>(e));
    cudaEventDestroy(std::get<2>(e));
  }
  ctx->events.clear();
  if (fwd_ms) *fwd_ms = ctx->t_fwd;
  if (bwd_ms) *bwd_ms = ctx->t_bwd;
  if (halo_ms) *halo_ms = ctx->t_halo;
  if (launches) *launches = ctx->launches - ctx->prof_launches;
  return SIP_OK;
}

long long sip_launch_count(const sip_ctx* ctx) { return ctx ? ctx->launches : 0; }

int sip_geometry(const sip_ctx* ctx, int* ti, int* tj, long long* tiles, long long* slices) {
  if (!ctx) return SIP_ERR_MISUSE;
  if (ti) *ti = kW;
  if (tj) *tj = kL;
  if (tiles) *tiles = (long long)ctx->hbricks.size();
  if (slices) *slices = ctx->total_slices;
  return SIP_OK;
}

long long sip_factor_count(const sip_ctx* ctx) { return ctx ? ctx->factor_count : 0; }

int sip_num_global_blocks(const sip_ctx* ctx, int* n) {
  if (!ctx || !n) return SIP_ERR_MISUSE;
  *n = (int)ctx->L.blocks.size();
  return SIP_OK;
}

// ---- debugging / test helpers (not part of the reference interface) ----
// Runs one forward sweep (K2) only, on the current device phi.
int sip_debug_forward(sip_ctx* ctx) {
  if (!ctx) return SIP_ERR_MISUSE;
  CKS(check_ready(ctx));
  CKS(set_device(ctx));
  CKS(ensure_norm_cap(ctx, ctx->n_done + 1));
  const size_t st = 32 * sizeof(unsigned);
  CK(cudaMemsetAsync(ctx->st_f, 0, st, ctx->stream));
  CK(cudaMemsetAsync(ctx->d_ctl, 0, 4 * sizeof(unsigned), ctx->stream));
  if (ctx->precision == SIP_PREC_SINGLE)
    CKS(launch_forward<float>(sweep_params<float>(ctx, true), ctx->grid_f, ctx->stream));
  else
    CKS(launch_forward<double>(sweep_params<double>(ctx, true), ctx->grid_f, ctx->stream));
  CK(cudaMemsetAsync(ctx->st_f, 0, st, ctx->stream));
  CK(cudaMemsetAsync(ctx->st_b, 0, st, ctx->stream));
  CK(cudaMemsetAsync(ctx->d_ctl, 0, 4 * sizeof(unsigned), ctx->stream));
  // the debug sweep does not count as an iteration: put the norm slot back
  const unsigned it = (unsigned)ctx->n_done;
  CK(cudaMemcpyAsync(ctx->d_norm_it, &it, sizeof(it), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SIP_OK;
}

// Gathers a device pack (0 = phi, 1 = R, 2..13 = forward pack arrays
// AP..LP, 14..16 = UN/UE/UT) of one local block into a Field3 array.
int sip_debug_field(sip_ctx* ctx, int local, int which, double* out) {
  if (!ctx || !out || local < 0 || local >= (int)ctx->local.size() || which < 0 || which > 16)
    return SIP_ERR_MISUSE;
  CKS(set_device(ctx));
  const BlockDesc& hb = ctx->hblocks[local];
  const size_t G = field3_elems(hb);
  CK(cudaMemsetAsync(ctx->staging, 0, G * sizeof(double), ctx->stream));
  auto run = [&](auto* phi, auto* R, auto* fw, auto* bw) -> int {
    using T = std::remove_pointer_t<decltype(phi)>;
    if (which == 0) return launch_gather_any<T>(phi, 0, 0, ctx->d_blocks, local, hb, ctx->staging, ctx->stream);
    if (which == 1) return launch_gather_any<T>(R, 1, 0, ctx->d_blocks, local, hb, ctx->staging, ctx->stream);
    if (which < 14)
      return launch_gather_any<T>(fw, F_NA, which - 2, ctx->d_blocks, local, hb, ctx->staging, ctx->stream);
    return launch_gather_any<T>(bw, B_NA, which - 14, ctx->d_blocks, local, hb, ctx->staging, ctx->stream);
  };
  const int rc = ctx->precision == SIP_PREC_SINGLE
                     ? run(static_cast<float*>(ctx->phi), static_cast<float*>(ctx->R),
                           static_cast<float*>(ctx->fw), static_cast<float*>(ctx->bw))
                     : run(static_cast<double*>(ctx->phi), static_cast<double*>(ctx->R),
                           static_cast<double*>(ctx->fw), static_cast<double*>(ctx->bw));
  CKS(rc);
  CK(cudaMemcpyAsync(out, ctx->staging, G * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SIP_OK;
}

// Per-brick timestamps (ns) of the most recent forward and backward sweep:
// out[2][nbricks][4] = {start, end, smid, 0}.  Enabled by the first call.
int sip_debug_trace(sip_ctx* ctx, unsigned long long* out, long long* ntiles) {
  if (!ctx || !ntiles) return SIP_ERR_MISUSE;
  CKS(set_device(ctx));
  const size_t nt = ctx->hbricks.size();
  *ntiles = (long long)nt;
  if (!ctx->trace) {
    CKS(dalloc(ctx, &ctx->trace, sizeof(unsigned long long) *
                                     (8 * std::max<size_t>(1, nt) + 5 * kTraceStages * kTraceMarks + 2 * kXTraceCtas)));
    if (const char* tb = getenv("SIPB_TRACE_BRICK")) ctx->trace_brick = atoi(tb);
    if (const char* tu = getenv("SIPB_TRACE_UP")) ctx->trace_brick |= atoi(tu) << 20;  // hop_trace: upstream offset
    return SIP_OK;
  }
  if (out) {
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(out, ctx->trace,
                  sizeof(unsigned long long) * (8 * nt + 5 * kTraceStages * kTraceMarks + 2 * kXTraceCtas),
                  cudaMemcpyDeviceToHost));
  }
  return SIP_OK;
}

int sip_nccl_unique_id(void* out128) {
  if (!out128) return SIP_ERR_MISUSE;
  ncclUniqueId id;
  if (!nccl().ok || nccl().GetUniqueId(&id) != ncclSuccess) return SIP_ERR_NCCL;
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, sizeof(id));
  return SIP_OK;
}

}  // extern "C"
