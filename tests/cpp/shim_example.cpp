// Drop-in example: the reference's solve() flow through include/bsfv_sip.hpp.
// Field type: a minimal stand-in with the Field3 interface
// (proj/include/bsfv/field.hpp:21-44); bsfv::FieldD works the same way.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bsfv_sip.hpp"

struct Field3 {
  int nx_ = 0, ny_ = 0, nz_ = 0;
  std::vector<double> d;
  Field3() = default;
  Field3(int nx, int ny, int nz) : nx_(nx), ny_(ny), nz_(nz), d((size_t)(nx + 2) * (ny + 2) * (nz + 2)) {}
  int nx() const { return nx_; }
  int ny() const { return ny_; }
  int nz() const { return nz_; }
  double* data() { return d.data(); }
  const double* data() const { return d.data(); }
};

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 12;
  const bool single = argc > 2 && argv[2][0] == 's';
  bsfv::b200::StencilSystemT<Field3> A{Field3(n, n, n), Field3(n, n, n), Field3(n, n, n),
                                       Field3(n, n, n), Field3(n, n, n), Field3(n, n, n),
                                       Field3(n, n, n), Field3(n, n, n)};
  const int g[3] = {n, n, n}, o[3] = {0, 0, 0};
  sip_generate_host(0, 1303, g, o, n, n, n, A.ap.data(), A.aw.data(), A.ae.data(), A.as.data(),
                    A.an.data(), A.ab.data(), A.at.data(), A.q.data());
  bsfv::b200::SipConfig cfg;
  cfg.max_iters = 5;
  cfg.single_precision = single;
  try {
    auto F = bsfv::b200::sip_factor(A, cfg);
    Field3 fi0(n, n, n);
    auto res = bsfv::b200::solve(A, fi0, cfg, &F);
    for (double v : res.second.norms) std::printf("%.17g\n", v);
    // reuse path: a stale system revision must be refused
    A.revision += 1;
    try {
      bsfv::b200::solve(A, fi0, cfg, &F);
      std::printf("ERROR: stale factors accepted\n");
      return 1;
    } catch (const bsfv::b200::StaleFactorsError&) {
      std::printf("stale ok\n");
    }
    // residual_general on the device; residual_symmetric needs A.symmetric
    Field3 r = bsfv::b200::residual_general(A, fi0);
    double l1 = 0.0;
    for (double v : r.d) l1 += v < 0 ? -v : v;
    std::printf("residual_general l1 %.17g\n", l1);
    try {
      bsfv::b200::residual_symmetric(A, fi0);
      std::printf("ERROR: unflagged system accepted\n");
      return 1;
    } catch (const bsfv::b200::MisuseError&) {
      std::printf("misuse ok\n");
    }
  } catch (const bsfv::b200::Error& e) {
    std::printf("error: %s\n", e.what());
    return 3;
  }
  return 0;
}
