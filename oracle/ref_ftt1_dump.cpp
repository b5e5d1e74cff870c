// ref_ftt1_dump.cpp -- TEST INFRASTRUCTURE: the reference's own FTT1 writer,
// reader and send/recv validator (proj/src/tables.cpp, with grid.cpp and
// transfers.cpp; compiled in place, oracle/Makefile target `ref`).
//
//   ref_ftt1_dump make gnx gny gnz px py pz ranks periodic_mask out.ftt1
//       build_transfer_tables (bit a of periodic_mask: axis a periodic,
//       other faces Wall) -> write_tables(out.ftt1); prints the read-back
//       entries as JSON
//   ref_ftt1_dump read file      read_tables -> JSON entries, or "error: ..."
//   ref_ftt1_dump validate file  read_tables + validate_matching -> "ok" / "error: ..."
// Output goes to oracle/make_golden.py, which commits tests/golden/ftt1/.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>

#include "bsfv/error.hpp"
#include "bsfv/grid.hpp"
#include "bsfv/tables.hpp"

static void print_json(const bsfv::TableSet& ts) {
  std::printf("{\"ranks\": [");
  for (int r = 0; r < ts.ranks(); ++r) {
    std::printf("%s[", r ? "," : "");
    for (std::size_t k = 0; k < ts.per_rank[r].size(); ++k) {
      const auto& e = ts.per_rank[r][k];
      std::printf("%s[%d,%d,%d,%u,%u,%u,%d,%d,%d,%d,%d,%d]", k ? "," : "", static_cast<int>(e.dir),
                  static_cast<int>(e.kind), static_cast<int>(e.face), e.peer_rank, e.owner_block,
                  e.neighbor_block, e.bounds.lo[0], e.bounds.hi[0], e.bounds.lo[1],
                  e.bounds.hi[1], e.bounds.lo[2], e.bounds.hi[2]);
    }
    std::printf("]");
  }
  std::printf("]}\n");
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  const std::string mode = argv[1];
  try {
    if (mode == "make" && argc >= 11) {
      bsfv::GridSpec g;
      g.nx = std::atoi(argv[2]);
      g.ny = std::atoi(argv[3]);
      g.nz = std::atoi(argv[4]);
      const int mask = std::atoi(argv[9]);
      for (int a = 0; a < 3; ++a) {
        const bsfv::Bc bc = (mask >> a) & 1 ? bsfv::Bc::Periodic : bsfv::Bc::Wall;
        g.bc[2 * a] = g.bc[2 * a + 1] = bc;
      }
      bsfv::BlockDecomposition dec =
          bsfv::decompose(g, std::atoi(argv[5]), std::atoi(argv[6]), std::atoi(argv[7]));
      const int ranks = std::atoi(argv[8]);
      if (ranks > 0) dec = bsfv::with_ranks(dec, ranks);
      const bsfv::TableSet ts = bsfv::build_transfer_tables(dec, g);
      bsfv::write_tables(ts, std::string(argv[10]));
      print_json(bsfv::read_tables(std::string(argv[10])));
    } else if (mode == "read") {
      print_json(bsfv::read_tables(std::string(argv[2])));
    } else if (mode == "validate") {
      bsfv::validate_matching(bsfv::read_tables(std::string(argv[2])));
      std::printf("ok\n");
    } else {
      return 2;
    }
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
  }
  return 0;
}
