// sip_internal.h -- shared declarations of the B200 SIP library (host + device).
//
// Device data layout: every block is cut into
// bricks of kW (i) x kL (j) columns that run through all nz planes.  One warp
// owns a brick: lane jl holds row j0 + jl and walks its cells
// c = k * kW + il (il = i - i0) in order, one cell per step, skewed by jl
// steps behind lane 0, so at step ("slice") tau = c + jl every lane sits on
// its own cell and
//   * the W neighbour (il - 1) is the lane's own previous step,
//   * the S neighbour (jl - 1) is lane jl - 1's previous step (one shfl),
//   * the B neighbour (k - 1) is the lane's own step tau - kW.
// A slice is one contiguous row of kL values per array, so the packs are
//   pack[((slot + tau) * NA + array) * kL + jl]
// (slice-major, array, lane), and a run of slices is one contiguous range --
// the sweep kernels stream it with TMA bulk copies.  A brick has
// ns = nz * kW + kL slices (kL - 1 of skew, rounded up to whole stages).
//
// phi carries its ghost cells in the same layout: the B / T ghost planes are
// the skew padding of the brick's own slices (cells c < 0 and c >= nz * kW,
// inside a porch of kPorch slices on either side), the W / E / S / N ghost
// faces live in ghost bricks (or in the padding column / lane of a ragged last
// brick), so every phi value the 7-point residual touches has one address
// (phi_index) and the halo exchange writes straight into it.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#ifndef __CUDACC__
#define __host__
#define __device__
#endif

#include "../../include/sip_c.h"

namespace sipb {

constexpr int kW = 8;       // brick extent along i (cells per lane per plane)
constexpr int kL = 32;      // brick extent along j (one warp lane per row)
constexpr int kStage = kW;  // slices per pipeline stage (one plane of a lane's cells)
constexpr int kPorch = 32;  // phi slices kept before tau = 0 and after ns

// forward pack: coefficients, source and lower factors (12 arrays)
enum FwArray { F_AP = 0, F_AW, F_AE, F_AS, F_AN, F_AB, F_AT, F_Q, F_LB, F_LW, F_LS, F_LP, F_NA };
// backward pack: upper factors
enum BwArray { B_UN = 0, B_UE, B_UT, B_NA };
// fp64 coefficient pack of single-precision contexts (factor input): AP..AT
constexpr int C_NA = 7;

// Ghost-face order (kernel order).
enum GhostFace { G_W = 0, G_E, G_S, G_N, G_B, G_T };

struct BlockDesc {
  int id;              // global block id
  int nx, ny, nz;
  int BX, BY;          // bricks along i / j
  int ns;              // slices per brick = nz * kW + kL
  int brick0, nbricks; // range in the brick array (brick r = bi + BX * bj)
  int gE, gN;          // ghost brick columns on E (nx % kW == 0) / rows on N (ny % kL == 0)
  long long slot0;     // fw / bw / R: slice tau = 0 of brick 0 (brick r at slot0 + r * ns)
  long long pbase;     // phi: first slice of the block's phi region
  long long medge0;    // mailbox: first edge entry of brick 0 (kL * nz per brick)
  long long mrow0;     // mailbox: first row entry of brick 0 (kW * nz per brick)
};

// phi bricks of a block: real bricks, then ghost W (BY), E (BY if gE), S (BX), N (BX if gN)
__host__ __device__ inline long long phi_stride(const BlockDesc& b) { return (long long)b.ns + 2 * kPorch; }
__host__ __device__ inline int phi_bricks(const BlockDesc& b) {
  return b.nbricks + b.BY * (1 + b.gE) + b.BX * (1 + b.gN);
}
// slice tau = 0 of phi brick pb (0-based within the block)
__host__ __device__ inline long long phi_slot(const BlockDesc& b, int pb) {
  return b.pbase + (long long)pb * phi_stride(b) + kPorch;
}

struct BrickDesc {
  long long slot;            // fw / bw / R slice tau = 0
  long long pslot;           // phi slice tau = 0
  long long pW, pE, pS, pN;  // phi slice tau = 0 of the W / E / S / N neighbour (real or ghost)
  long long medge, mrow;     // own mailbox entries (published: K2 E col / N row, K3 W col / S row)
  long long mWe, mEe;        // W / E neighbour's edge mailbox (-1: block boundary, value 0)
  long long mSr, mNr;        // S / N neighbour's row mailbox (-1: block boundary)
  int block, bi, bj;
  int i0, j0, wI, wJ;
  int nz, ns;
};

// Slice of interior cell (i, j, k) in its brick (0-based, within the block).
__host__ __device__ inline long long pack_slice(const BlockDesc& b, int i, int j, int k) {
  const int bi = i / kW, il = i - bi * kW, bj = j / kL, jl = j - bj * kL;
  return b.slot0 + (long long)(bi + b.BX * bj) * b.ns + (long long)k * kW + il + jl;
}
// Pack element index of interior cell (i, j, k).
__host__ __device__ inline long long pack_index(const BlockDesc& b, int na, int arr, int i, int j,
                                                int k) {
  return (pack_slice(b, i, j, k) * na + arr) * kL + (j % kL);
}
// phi element index of cell (i, j, k) with i in [-1, nx], j in [-1, ny],
// k in [-1, nz] (interior or face ghost; edges / corners are not stored).
__host__ __device__ inline long long phi_index(const BlockDesc& b, int i, int j, int k) {
  int pb, il, jl;
  if (i < 0) {
    pb = b.nbricks + j / kL;
    il = kW - 1;
    jl = j % kL;
  } else if (j < 0) {
    pb = b.nbricks + b.BY * (1 + b.gE) + i / kW;
    il = i % kW;
    jl = kL - 1;
  } else if (i == b.nx && b.gE) {
    pb = b.nbricks + b.BY + j / kL;
    il = 0;
    jl = j % kL;
  } else if (j == b.ny && b.gN) {
    pb = b.nbricks + b.BY * (1 + b.gE) + b.BX + i / kW;
    il = i % kW;
    jl = 0;
  } else {  // interior, B / T ghosts (porch) and ragged E / N ghosts (padding)
    pb = i / kW + b.BX * (j / kL);
    il = i % kW;
    jl = j % kL;
  }
  return (phi_slot(b, pb) + (long long)k * kW + il + jl) * kL + jl;
}

// ---------------------------------------------------------------- planning
struct BlockInfo {
  std::array<int, 3> coord{0, 0, 0};
  std::array<int, 3> lo{0, 0, 0};  // global 0-based first interior cell
  std::array<int, 3> n{0, 0, 0};   // extents
  std::array<int, 6> nbr{-1, -1, -1, -1, -1, -1};  // W,E,S,N,B,T block ids
};
struct Lattice {
  std::vector<int> g{0, 0, 0}, p{1, 1, 1};
  std::vector<BlockInfo> blocks;
};
struct HaloEntry {
  int dir, face, owner, neighbor, peer;
  int lo[3], hi[3];
};

// Thread-local error text returned by sip_last_error(NULL) (free functions).
void set_thread_error(const std::string& err);
bool ftt1_validate(const std::vector<std::vector<std::array<int, 12>>>& t, std::string& err);

bool build_lattice(int gnx, int gny, int gnz, int px, int py, int pz, Lattice& L, std::string& err);
bool plan_block_ranks(int px, int py, int pz, int nranks, std::vector<int>& out);
// face transfers of this rank; bit a of periodic_mask: axis a wraps
void plan_halo(const Lattice& L, const std::vector<int>& rank_of, int rank,
               std::vector<HaloEntry>& out, int periodic_mask = 0);

// ---------------------------------------------------------------- kernels
// One face copy: interior plane of src block -> ghost face of dst block, or
// plane -> linear buffer (pack) / buffer -> ghost face (unpack).
struct FaceCopy {
  int src_block;   // local block index (or -1 when reading a buffer)
  int src_face;    // kernel face order: which interior plane (W = i=0 plane ...)
  int dst_block;   // local block index (or -1 when writing a buffer)
  int dst_face;    // ghost face written
  long long buf;   // element offset into the linear buffer
  int n0, n1;      // plane extents (fast, slow)
};

// Cross-brick edge values travel as self-validating tagged words: value bits
// + the 32-bit launch epoch of the producing sweep, one 64-bit word per fp32
// value, two per fp64 value (each carrying 32 value bits).  A mailbox entry is
// written exactly once per launch, so a matching epoch means "this launch's
// value": no flag, fence or counter.
template <typename T>
struct SweepParams {
  const BrickDesc* bricks;
  const BlockDesc* blocks;
  const int* order;  // ticket -> brick (topological order of this sweep)
  int nbricks;
  int nblocks;
  const T* fw;
  const T* bw;
  T* phi;
  T* R;
  //   K2: mA = R of each brick's E column (edge entries), mB = R of its N row (row entries)
  //   K3: mA = delta of each brick's W column,            mB = delta of its S row
  unsigned long long* mA;
  unsigned long long* mB;
  unsigned* epoch;        // launch counter of this sweep kind (bumped by the finaliser)
  unsigned* state;        // this sweep: [0] ticket, [1] done
  unsigned* state_other;  // the other sweep's state, reset by our finaliser
  double* partial;        // [nbricks] brick norm partials
  // forward only: norms of iteration it = *norm_it go to norms_base[it] and
  // bnorms_base[it * nblocks + b]; the finaliser then bumps *norm_it, so a
  // captured CUDA graph of several iterations replays without new parameters
  double* norms_base;
  double* bnorms_base;
  unsigned* norm_it;
  // device-side stop of a target-reduction solve (single rank): the K2
  // finaliser of the first sweep with norm / norm[0] <= target sets ctl[0];
  // a K2 launch that finds ctl[0] set returns at once.  ctl[1]: a K2 ran and
  // its K3 is pending (K3 returns at once when it is 0).  target <= 0: never stop.
  double target;
  unsigned* ctl;
  // split exchange: K2's finaliser bumps *xseq; K3 stamps
  // xflag[2 * brick] (its top slices, k = nz - 1, stored) and xflag[2 * brick + 1]
  // (all stored) with that value, so the E / N / T face copies on the comm
  // stream can start while K3 still runs.  nullptr: no split exchange.
  unsigned* xseq;
  unsigned* xflag;
  unsigned long long* trace;  // optional [nbricks][4]: start ns, end ns, smid, stalls (debug)
  // debug: per-stage clock64 marks of brick trace_brick (first kTraceStages stages,
  // kTraceMarks each) after the per-brick table
  int trace_brick;
};
constexpr int kTraceStages = 64, kTraceMarks = 6;

template <typename T>
struct FactorParams {
  const BrickDesc* bricks;
  const BlockDesc* blocks;
  const int* order;
  int nbricks;
  double alpha;
  const double* coef;  // fp64 AP..AT: the fp64 forward pack (coef_na = F_NA) or the
  int coef_na;         // fp64 coefficient pack of single-precision contexts (C_NA)
  T* fw;               // out: LB LW LS LP (forward pack)
  T* bw;               // out: UN UE UT
  unsigned long long* mA;  // (UN, UE, UT) of each brick's E column, fp64 tagged
  unsigned long long* mB;  // (UN, UE, UT) of each brick's N row
  unsigned* epoch;
  unsigned* state;
  unsigned long long* bad;  // (block << 40) | Field3 index of the first singular cell
};

// launchers (sip_kernels.cu); all asynchronous on `stream`
template <typename T>
int launch_factor(const FactorParams<T>& p, int grid, void* stream);
template <typename T>
int launch_forward(const SweepParams<T>& p, int grid, void* stream);
template <typename T>
int launch_backward(const SweepParams<T>& p, int grid, void* stream);
int launch_check_symmetric(const BlockDesc* d_blocks, int block, const BlockDesc& hb,
                           const double* coef, int coef_na, unsigned long long* bad, void* stream);
template <typename T>
int launch_scatter(const double* src, const BlockDesc* d_blocks, int block, const BlockDesc& hb,
                   T* pack, int na, int arr, void* stream);
template <typename T>
int launch_phi_in(const double* src, const BlockDesc* d_blocks, int block, const BlockDesc& hb,
                  T* phi, void* stream);
template <typename T>
int launch_gather(const T* phi, const BlockDesc* d_blocks, int block, const BlockDesc& hb,
                  const int* nbr6, double* dst, void* stream);
template <typename T>
int launch_face_copies(const FaceCopy* d_copies, int ncopies, int max_plane,
                       const BlockDesc* d_blocks, T* phi, const T* buf_in, T* buf_out,
                       void* stream);
// Split exchange phase 1 work item: the part of early copy `entry`'s source
// plane held by one brick -- plane rectangle [x0b, x0e) x [x1b, x1e) in the
// copy's (x0, x1) coordinates -- ready once K3 stamped xflag[2 * brick + sel]
// (sel 0: the brick's top slices, T planes; 1: the whole brick, E / N planes).
struct XItem {
  int entry, brick, sel;
  int x0b, x0e, x1b, x1e;
};
// split exchange phase 1 (comm stream, during K3): waits on K3's per-brick stamps
template <typename T>
int launch_face_copies_after(const FaceCopy* d_copies, const XItem* d_items, int nitems,
                             const BlockDesc* d_blocks, T* phi, T* buf_out, const unsigned* xflag,
                             const unsigned* xseq, unsigned long long* xtrace, void* stream);
// debug trace layout (sip_debug_trace): [4 nbricks] K2, [4 nbricks] K3, stage
// marks, then kXTraceCtas x 2 of the split exchange's copy kernel
constexpr int kXTraceCtas = 256;
template <typename T>
int launch_residual(const BlockDesc* d_blocks, int block, const BlockDesc& hb, const T* fw,
                    const T* phi, int symmetric, double* out, void* stream);
template <typename T>
int launch_gather_any(const T* pack, int na, int arr, const BlockDesc* d_blocks, int block,
                      const BlockDesc& hb, double* dst, void* stream);
int launch_generate(int kind, uint64_t seed, const int g[3], const int o[3], int nx, int ny, int nz,
                    double* const* out8, void* stream);
// persistent grid of a sweep kind (0 factor, 1 forward, 2 backward)
int max_resident_ctas(int kind, int precision, int* grid);

}  // namespace sipb
