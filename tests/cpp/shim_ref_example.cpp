// The drop-in as the reference code base would use it: the reference's own
// Field3 (bsfv::FieldD, proj/include/bsfv/field.hpp) and exception classes
// (proj/include/bsfv/error.hpp) through include/bsfv_sip.hpp.  Built by
// tests/test_cpp_shim.py with -I /root/reference/proj/include (build
// container only).  Prints the norms, the report's times and the factor
// counter; exits 3 on a bsfv::Error (e.g. no CUDA device).
#include <cstdio>
#include <cstdlib>

#include "bsfv/error.hpp"
#include "bsfv/field.hpp"
#define BSFV_SIP_USE_REFERENCE_ERRORS 1
#include "bsfv_sip.hpp"

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 10;
  using bsfv::FieldD;
  bsfv::b200::StencilSystemT<FieldD> A{FieldD(n, n, n), FieldD(n, n, n), FieldD(n, n, n),
                                       FieldD(n, n, n), FieldD(n, n, n), FieldD(n, n, n),
                                       FieldD(n, n, n), FieldD(n, n, n)};
  const int g[3] = {n, n, n}, o[3] = {0, 0, 0};
  sip_generate_host(0, 1303, g, o, n, n, n, A.ap.data(), A.aw.data(), A.ae.data(), A.as.data(),
                    A.an.data(), A.ab.data(), A.at.data(), A.q.data());
  bsfv::b200::SipConfig cfg;
  cfg.max_iters = 6;
  try {
    auto F = bsfv::b200::sip_factor(A, cfg);
    FieldD fi0(n, n, n);
    for (int rep = 0; rep < 3; ++rep) {  // reuse path: no new factorisation
      auto res = bsfv::b200::solve(A, fi0, cfg, &F);
      if (rep == 0)
        for (double v : res.second.norms) std::printf("%.17g\n", v);
      if (res.second.factor_seconds != 0.0 || !(res.second.relax_seconds > 0.0)) {
        std::printf("ERROR: report times\n");
        return 1;
      }
    }
    std::printf("factorizations %lld\n", F.factorizations());
    try {
      A.revision += 1;
      bsfv::b200::solve(A, fi0, cfg, &F);
      std::printf("ERROR: stale factors accepted\n");
      return 1;
    } catch (const bsfv::StaleFactorsError&) {  // the reference's own class
      std::printf("stale ok\n");
    }
  } catch (const bsfv::Error& e) {
    std::printf("bsfv::Error: %s\n", e.what());
    return 3;
  }
  return 0;
}
