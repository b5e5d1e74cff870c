// sip_internal.h -- shared declarations of the B200 SIP library (host + device).
//
// Device data layout: every block is cut into
// (TI x TJ)-column tiles of the (i, j) plane; a tile streams along k.  Cell
// (ti, tj, k) of a tile is processed at wavefront step t = k + ti + tj (the
// hyperplane index inside the tile), so each step of a tile touches one
// "slice" of TI*TJ cells.  Packs store slices contiguously:
//     pack[((slot + t) * NA + array) * TT + pos(ti, tj)]
// where slot is the tile's first slice, NA the arrays in the pack and pos()
// numbers the tile's cells by anti-diagonal (d = ti + tj ascending, then ti),
// so a slice's valid cells are always one contiguous range -- fill/drain
// slices are fetched with range-limited bulk copies (no padding traffic).
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

constexpr int kTI = 16;  // tile extent along i (columns)
constexpr int kTJ = 16;  // tile extent along j
constexpr int kTT = kTI * kTJ;
constexpr int kD = kTI + kTJ - 1;  // diagonals per tile = skew + 1

// forward pack: coefficients, source and lower factors (12 arrays)
enum FwArray { F_AP = 0, F_AW, F_AE, F_AS, F_AN, F_AB, F_AT, F_Q, F_LB, F_LW, F_LS, F_LP, F_NA };
// backward pack: upper factors
enum BwArray { B_UN = 0, B_UE, B_UT, B_NA };

// Ghost-face order inside a block's ghost record (kernel order).
enum GhostFace { G_W = 0, G_E, G_S, G_N, G_B, G_T };

struct TileDesc {
  long long slot;  // first slice of this tile in the packs
  long long edge;  // element offset of this tile's delta edge records
  int block;       // local block index
  int i0, j0;      // first column, 0-based within the block
  int wI, wJ;      // valid extents (ragged last tiles)
  int nW, nE, nS, nN;  // neighbour tile (index into the tile array) or -1
  int ns;          // slices = nz + kD - 1
  int nz;
};

struct BlockDesc {
  int id;            // global block id
  int nx, ny, nz;
  int TX, TY;        // tiles per axis
  int ns;            // slices per tile
  long long slot0;   // first slice of the block's first tile
  long long ghost;   // element offset of the block's 6 ghost faces
  int tile0, ntiles; // range in the tile array (block-major, row-major tiles)
};

__host__ __device__ inline long long ghost_face_offset(const BlockDesc& b, int face) {
  const long long yz = (long long)b.ny * b.nz, xz = (long long)b.nx * b.nz;
  switch (face) {
    case G_W: return b.ghost;
    case G_E: return b.ghost + yz;
    case G_S: return b.ghost + 2 * yz;
    case G_N: return b.ghost + 2 * yz + xz;
    case G_B: return b.ghost + 2 * yz + 2 * xz;
    default: return b.ghost + 2 * yz + 2 * xz + (long long)b.nx * b.ny;
  }
}
__host__ __device__ inline long long ghost_count(int nx, int ny, int nz) {
  return 2LL * ny * nz + 2LL * nx * nz + 2LL * nx * ny;
}

// first cell index of diagonal d (0 <= d <= kD) in a square S x S tile:
// d(d+1)/2 below the main anti-diagonal, S^2 - (2S-1-d)(2S-d)/2 above it.
static_assert(kTI == kTJ, "closed-form diagonal offsets assume square tiles");
__host__ __device__ constexpr int diag_off(int d) {
  return d <= kTI ? d * (d + 1) / 2 : kTT - (2 * kTI - 1 - d) * (2 * kTI - d) / 2;
}
__host__ __device__ inline int tile_pos(int ti, int tj) {
  const int d = ti + tj;
  const int lo = d - (kTJ - 1) > 0 ? d - (kTJ - 1) : 0;
  return diag_off(d) + (ti - lo);
}

// Pack element index of interior cell (i, j, k), 0-based within the block.
__host__ __device__ inline long long pack_index(const BlockDesc& b, int na, int arr, int i, int j,
                                                int k) {
  const int a = i / kTI, ti = i - a * kTI;
  const int c = j / kTJ, tj = j - c * kTJ;
  const long long slot = b.slot0 + (long long)(a + b.TX * c) * b.ns + (k + ti + tj);
  return (slot * na + arr) * kTT + tile_pos(ti, tj);
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

template <typename T>
struct SweepParams {
  const TileDesc* tiles;
  const BlockDesc* blocks;
  const int* order;  // ticket -> tile (topological order of this sweep)
  int ntiles;
  int nblocks;
  T* fw;
  T* bw;
  T* phi;
  T* R;
  T* ghost;
  T* edgeW;  // (factor kernel only) unused by K2/K3
  T* edgeS;
  // K2: the static (old-phi / ghost) part of each step's edge record,
  // [slot + s][64] = phiW, phiE, phiS, phiN (16 each); built by k_edge_phi
  // after every halo exchange and bulk-copied with the step's phi slice
  T* rec_phi;
  int symmetric;  // K2: every block's system flagged symmetric -> Listing-1 fast path
  // Cross-tile edge values as self-validating tagged words (DESIGN.md
  // "Cross-tile hand-off"): value bits + 32-bit tag (epoch << 16 | k), one
  // 64-bit word per fp32 value, two per fp64 value; index (edge + k*16 + c).
  //   K2: tagA = R of each tile's E column, tagB = R of its N row
  //   K3: tagA = delta of each tile's W column, tagB = delta of its S row
  unsigned long long* tagA;
  unsigned long long* tagB;
  unsigned* epoch;        // launch counter of this sweep kind (bumped by the finaliser)
  unsigned* state;        // this sweep: [0] ticket, [1] done, prog at state + 32
  unsigned* state_other;  // the other sweep's state, reset by our finaliser
  double* partial;        // [ntiles] tile norm partials
  // forward only: norms of iteration it = *norm_it go to norms_base[it] and
  // bnorms_base[it * nblocks + b]; the finaliser then bumps *norm_it, so a
  // captured CUDA graph of several iterations replays without new parameters
  double* norms_base;
  double* bnorms_base;
  unsigned* norm_it;
  unsigned long long* trace;  // optional [ntiles][4]: start ns, end ns, smid, cta (debug)
  int trace_tile;             // debug: tile whose per-step times are recorded after the table
};

struct FactorParams {
  const TileDesc* tiles;
  const BlockDesc* blocks;
  const int* order;
  int ntiles;
  double alpha;
  double* fw;
  double* bw;
  unsigned* state;
  unsigned long long* bad;  // (block << 40) | Field3 index of the first singular cell
};

// launchers (sip_kernels.cu); all asynchronous on `stream`
int launch_factor(const FactorParams& p, int grid, void* stream);
template <typename T>
int launch_forward(const SweepParams<T>& p, int grid, void* stream);
template <typename T>
int launch_backward(const SweepParams<T>& p, int grid, void* stream);
template <typename T>
int launch_edge_phi(const SweepParams<T>& p, void* stream);
int launch_check_symmetric(const BlockDesc* d_blocks, int block, const BlockDesc& hb,
                           const double* fw, unsigned long long* bad, void* stream);
template <typename T>
int launch_scatter(const double* src, const BlockDesc* d_blocks, int block, const BlockDesc& hb,
                   T* pack, int na, int arr, void* stream);
template <typename T>
int launch_ghost_in(const double* src, const BlockDesc* d_blocks, int block, const BlockDesc& hb,
                    T* ghost, void* stream);
template <typename T>
int launch_gather(const T* pack, const T* ghost, const BlockDesc* d_blocks, int block,
                  const BlockDesc& hb, const int* nbr6, double* dst, void* stream);
template <typename T>
int launch_face_copies(const FaceCopy* d_copies, int ncopies, int max_plane,
                       const BlockDesc* d_blocks, const T* phi, T* ghost, T* buf_in, T* buf_out,
                       void* stream);
template <typename T>
int launch_residual(const BlockDesc* d_blocks, int block, const BlockDesc& hb, const T* fw,
                    const T* phi, const T* ghost, int symmetric, double* out, void* stream);
template <typename T>
int launch_gather_any(const T* pack, int na, int arr, const BlockDesc* d_blocks, int block,
                      const BlockDesc& hb, double* dst, void* stream);
int launch_convert(const double* src, float* dst, long long n, void* stream);
int launch_generate(int kind, uint64_t seed, const int g[3], const int o[3], int nx, int ny, int nz,
                    double* const* out8, void* stream);
int max_resident_ctas(int kind, int precision, int* grid);

}  // namespace sipb
