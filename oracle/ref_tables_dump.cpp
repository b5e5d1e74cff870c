// ref_tables_dump.cpp -- TEST INFRASTRUCTURE: links the reference's own
// grid.cpp / transfers.cpp / tables.cpp (compiled in place from
// /root/reference/proj, see oracle/Makefile target `ref`) and prints the
// face entries of bsfv::build_transfer_tables plus bsfv::decompose extents as
// JSON, for the golden fixtures under tests/golden/ (oracle/make_golden.py).
//
// usage: ref_tables_dump gnx gny gnz px py pz ranks
//   ranks == 0: one block per rank (decompose()); otherwise with_ranks(ranks)
// All faces use Bc::Wall (the SIP systems carry boundary conditions in their
// coefficients, so the lattice is non-periodic).
#include <cstdio>
#include <cstdlib>

#include "bsfv/grid.hpp"
#include "bsfv/tables.hpp"

int main(int argc, char** argv) {
  if (argc < 8) {
    std::fprintf(stderr, "usage: %s gnx gny gnz px py pz ranks\n", argv[0]);
    return 2;
  }
  bsfv::GridSpec g;
  g.nx = std::atoi(argv[1]);
  g.ny = std::atoi(argv[2]);
  g.nz = std::atoi(argv[3]);
  for (auto& b : g.bc) b = bsfv::Bc::Wall;
  const int px = std::atoi(argv[4]), py = std::atoi(argv[5]), pz = std::atoi(argv[6]);
  const int ranks = std::atoi(argv[7]);
  bsfv::BlockDecomposition dec = bsfv::decompose(g, px, py, pz);
  if (ranks > 0) dec = bsfv::with_ranks(dec, ranks);
  const bsfv::TableSet ts = bsfv::build_transfer_tables(dec, g);
  std::printf("{\"blocks\": [");
  for (int b = 0; b < dec.num_blocks(); ++b) {
    const auto& e = dec.blocks[b];
    std::printf("%s[%d,%d,%d,%d,%d,%d,%d]", b ? "," : "", e.lo[0], e.lo[1], e.lo[2], e.hi[0],
                e.hi[1], e.hi[2], dec.rank_of_block[b]);
  }
  std::printf("], \"ranks\": [");
  for (int r = 0; r < ts.ranks(); ++r) {
    std::printf("%s[", r ? "," : "");
    bool first = true;
    for (const auto& e : ts.per_rank[r]) {
      if (e.kind != bsfv::PatchKind::Face) continue;
      std::printf("%s[%d,%d,%d,%u,%u,%u,%d,%d,%d,%d,%d,%d]", first ? "" : ",",
                  static_cast<int>(e.dir), static_cast<int>(e.kind), static_cast<int>(e.face),
                  e.peer_rank, e.owner_block, e.neighbor_block, e.bounds.lo[0], e.bounds.hi[0],
                  e.bounds.lo[1], e.bounds.hi[1], e.bounds.lo[2], e.bounds.hi[2]);
      first = false;
    }
    std::printf("]");
  }
  std::printf("]}\n");
  return 0;
}
