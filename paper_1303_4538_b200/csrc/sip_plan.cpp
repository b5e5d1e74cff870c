// sip_plan.cpp -- host-side planning for the block-structured SIP path:
// block lattice (mirrors bsfv::decompose, proj/src/grid.cpp:50-89), compact
// block -> rank placement (replaces with_ranks' contiguous slabs,
// grid.cpp:91-102, which SURVEY.md 0.4(e) shows cannot give a 2x2x2 lattice
// per GPU), and the face-halo plan (the face subset of build_transfers,
// proj/src/transfers.cpp:45-167, in its canonical order transfers.cpp:148-165).
// Pure C++, no device code: exercised by the CPU test-suite.
#include <algorithm>
#include <array>
#include <cstring>
#include <tuple>
#include <vector>

#include "sip_internal.h"

namespace sipb {

bool build_lattice(int gnx, int gny, int gnz, int px, int py, int pz, Lattice& L, std::string& err) {
  const int g[3] = {gnx, gny, gnz};
  const int p[3] = {px, py, pz};
  const char* names[3] = {"x", "y", "z"};
  for (int a = 0; a < 3; ++a) {
    if (g[a] < 1) {
      err = std::string("grid: axis ") + names[a] + " needs at least 1 cell";
      return false;
    }
    if (p[a] < 1) {
      err = "decompose: block counts must be positive";
      return false;
    }
    if (p[a] > g[a]) {
      err = std::string("decompose: axis ") + names[a] + " has more blocks (" +
            std::to_string(p[a]) + ") than cells (" + std::to_string(g[a]) + ")";
      return false;
    }
  }
  L.g = {gnx, gny, gnz};
  L.p = {px, py, pz};
  L.blocks.clear();
  L.blocks.resize(static_cast<size_t>(px) * py * pz);
  for (int bz = 0; bz < pz; ++bz)
    for (int by = 0; by < py; ++by)
      for (int bx = 0; bx < px; ++bx) {
        const int bc[3] = {bx, by, bz};
        BlockInfo bi;
        bi.coord = {bx, by, bz};
        for (int a = 0; a < 3; ++a) {
          const int base = g[a] / p[a];
          bi.lo[a] = bc[a] * base;
          // remainder cells go to the last block on the axis (grid.cpp:76-78)
          const int hi = (bc[a] == p[a] - 1) ? g[a] - 1 : bi.lo[a] + base - 1;
          bi.n[a] = hi - bi.lo[a] + 1;
        }
        // face neighbours in our kernel order W,E,S,N,B,T (non-periodic: SIP
        // systems carry their boundary conditions in the coefficients)
        for (int f = 0; f < 6; ++f) {
          const int a = f / 2, s = (f % 2) ? +1 : -1;
          std::array<int, 3> c = bi.coord;
          c[a] += s;
          bi.nbr[f] = (c[a] < 0 || c[a] >= p[a]) ? -1 : c[0] + px * (c[1] + py * c[2]);
        }
        // device kernels index a block's cells with 32-bit arithmetic
        if ((long long)bi.n[0] * bi.n[1] >= (1LL << 31) ||
            (long long)bi.n[0] * bi.n[1] * bi.n[2] >= (1LL << 32)) {
          err = "decompose: a block must have fewer than 2^32 cells (2^31 per k-plane)";
          return false;
        }
        L.blocks[bx + px * (by + py * bz)] = bi;
      }
  return true;
}

// Near-cubic factorisation of nranks into (rx, ry, rz) dividing (px, py, pz),
// preferring to split the longest block axis first; falls back to contiguous
// chunks (with_ranks semantics) when no such factorisation exists.
bool plan_block_ranks(int px, int py, int pz, int nranks, std::vector<int>& out) {
  const int nb = px * py * pz;
  out.assign(nb, 0);
  if (nranks < 1 || nranks > nb) return false;
  int best[3] = {0, 0, 0};
  long best_cost = -1;
  for (int rx = 1; rx <= nranks; ++rx) {
    if (nranks % rx || px % rx) continue;
    for (int ry = 1; ry <= nranks / rx; ++ry) {
      if ((nranks / rx) % ry || py % ry) continue;
      const int rz = nranks / rx / ry;
      if (pz % rz) continue;
      // cost: surface of one rank's sub-lattice (in blocks), smaller is better
      const long sx = px / rx, sy = py / ry, sz = pz / rz;
      const long cost = sx * sy + sy * sz + sx * sz;
      // tie-break: split z first, then y (keeps x-contiguous slabs longest)
      if (best_cost < 0 || cost < best_cost ||
          (cost == best_cost && std::make_tuple(rz, ry) > std::make_tuple(best[2], best[1]))) {
        best_cost = cost;
        best[0] = rx; best[1] = ry; best[2] = rz;
      }
    }
  }
  if (best_cost < 0) {
    for (int b = 0; b < nb; ++b)
      out[b] = static_cast<int>((static_cast<long long>(b) * nranks) / nb);
    return true;
  }
  const int sx = px / best[0], sy = py / best[1], sz = pz / best[2];
  for (int bz = 0; bz < pz; ++bz)
    for (int by = 0; by < py; ++by)
      for (int bx = 0; bx < px; ++bx) {
        const int rx = bx / sx, ry = by / sy, rz = bz / sz;
        out[bx + px * (by + py * bz)] = rx + best[0] * (ry + best[1] * rz);
      }
  return true;
}

// Face transfers of the whole decomposition in the reference's canonical
// order (transfers.cpp:153-165 key restricted to PatchKind::Face), then the
// per-rank entries in table order (tables.cpp:25-40).
void plan_halo(const Lattice& L, const std::vector<int>& rank_of, int rank,
               std::vector<HaloEntry>& out, int periodic_mask) {
  struct T {
    int src, dst, face_dst, off[3];
    int src_lo[3], src_hi[3], dst_lo[3], dst_hi[3];
  };
  std::vector<T> all;
  const int nb = static_cast<int>(L.blocks.size());
  for (int dst = 0; dst < nb; ++dst) {
    const BlockInfo& X = L.blocks[dst];
    for (int a = 0; a < 3; ++a)
      for (int sign : {+1, -1}) {
        // our nbr order is W,E,S,N,B,T = (a, -1), (a, +1)
        int src = X.nbr[2 * a + (sign > 0 ? 1 : 0)];
        if (src < 0 && ((periodic_mask >> a) & 1)) {  // wrap (transfers.cpp:15-25)
          std::array<int, 3> c = X.coord;
          c[a] = (c[a] + sign + L.p[a]) % L.p[a];
          src = c[0] + L.p[0] * (c[1] + L.p[1] * c[2]);
        }
        if (src < 0) continue;
        const BlockInfo& N = L.blocks[src];
        T t{};
        t.src = src;
        t.dst = dst;
        t.off[0] = t.off[1] = t.off[2] = 0;
        t.off[a] = sign;
        t.face_dst = 2 * a + (sign > 0 ? 0 : 1);  // bsfv Face id: E,W,N,S,T,B
        for (int b = 0; b < 3; ++b) {
          if (b == a) {
            t.dst_lo[b] = t.dst_hi[b] = (sign > 0) ? X.n[b] + 1 : 0;
            t.src_lo[b] = t.src_hi[b] = (sign > 0) ? 1 : N.n[b];
          } else {
            t.dst_lo[b] = 1; t.dst_hi[b] = X.n[b];
            t.src_lo[b] = 1; t.src_hi[b] = N.n[b];
          }
        }
        all.push_back(t);
      }
  }
  auto key = [&](const T& t) {
    const int ra = rank_of[t.src], rb = rank_of[t.dst];
    return std::make_tuple(std::min(ra, rb), std::max(ra, rb), t.src, t.dst, t.off[0], t.off[1],
                           t.off[2], t.src_lo[2], t.src_lo[1], t.src_lo[0]);
  };
  std::stable_sort(all.begin(), all.end(), [&](const T& x, const T& y) { return key(x) < key(y); });
  out.clear();
  for (const T& t : all) {
    const int rs = rank_of[t.src], rd = rank_of[t.dst];
    auto mk = [&](int dir, int face, int owner, int nbrb, int peer, const int* lo, const int* hi) {
      HaloEntry e{};
      e.dir = dir;
      e.face = face;
      e.owner = owner;
      e.neighbor = nbrb;
      e.peer = peer;
      for (int b = 0; b < 3; ++b) {
        e.lo[b] = lo[b];
        e.hi[b] = hi[b];
      }
      return e;
    };
    const int src_face = t.face_dst ^ 1;  // opposite(dst_face)
    if (rs == rd) {
      if (rs == rank) out.push_back(mk(0, src_face, t.src, t.dst, rs, t.src_lo, t.src_hi));
    } else {
      if (rs == rank) out.push_back(mk(1, src_face, t.src, t.dst, rd, t.src_lo, t.src_hi));
      if (rd == rank) out.push_back(mk(2, t.face_dst, t.dst, t.src, rs, t.dst_lo, t.dst_hi));
    }
  }
}

}  // namespace sipb

extern "C" int sip_plan_block_ranks(int px, int py, int pz, int nranks, int* block_rank) {
  if (!block_rank || px < 1 || py < 1 || pz < 1) return SIP_ERR_CONFIG;
  std::vector<int> v;
  if (!sipb::plan_block_ranks(px, py, pz, nranks, v)) return SIP_ERR_CONFIG;
  std::memcpy(block_rank, v.data(), v.size() * sizeof(int));
  return SIP_OK;
}

extern "C" int sip_plan_halo_periodic(int gnx, int gny, int gnz, int px, int py, int pz,
                                      const int* block_rank, int rank, int periodic_mask,
                                      int* n_entries, int* entries) {
  sipb::Lattice L;
  std::string err;
  if (!n_entries || !sipb::build_lattice(gnx, gny, gnz, px, py, pz, L, err)) return SIP_ERR_CONFIG;
  const int nb = px * py * pz;
  std::vector<int> rank_of(nb);
  if (block_rank) {
    for (int b = 0; b < nb; ++b) rank_of[b] = block_rank[b];
  } else {
    for (int b = 0; b < nb; ++b) rank_of[b] = b;  // decompose(): one block per rank
  }
  std::vector<sipb::HaloEntry> v;
  sipb::plan_halo(L, rank_of, rank, v, periodic_mask);
  if (entries) {
    if (*n_entries < static_cast<int>(v.size())) return SIP_ERR_CONFIG;
    for (size_t n = 0; n < v.size(); ++n) {
      int* e = entries + 12 * n;
      e[0] = v[n].dir; e[1] = 0; e[2] = v[n].face; e[3] = v[n].peer;
      e[4] = v[n].owner; e[5] = v[n].neighbor;
      e[6] = v[n].lo[0]; e[7] = v[n].hi[0]; e[8] = v[n].lo[1];
      e[9] = v[n].hi[1]; e[10] = v[n].lo[2]; e[11] = v[n].hi[2];
    }
  }
  *n_entries = static_cast<int>(v.size());
  return SIP_OK;
}

extern "C" int sip_plan_halo(int gnx, int gny, int gnz, int px, int py, int pz,
                             const int* block_rank, int rank, int* n_entries, int* entries) {
  return sip_plan_halo_periodic(gnx, gny, gnz, px, py, pz, block_rank, rank, 0, n_entries, entries);
}
