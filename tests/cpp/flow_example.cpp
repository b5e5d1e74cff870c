// flow_example.cpp -- the C++ shim's pressure-correction caller
// (bsfv::b200::PressureSolver): a periodic box with a smooth divergent
// velocity field, 100 pressure_correct steps on one factorisation.
// Prints the factorisation count, the outer iterations of each corrected step
// and the divergence before / after; exit 3 on a device error.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "bsfv_sip.hpp"

using namespace bsfv::b200;

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 16;
  try {
    PressureSolver ps({n, n, n}, {2, 1, 1}, {1.0, 1.0, 1.0},
                      {Bc::Periodic, Bc::Periodic, Bc::Periodic, Bc::Periodic, Bc::Wall, Bc::Wall});
    const double tp = 2.0 * std::acos(-1.0);
    int origin_x = 0;
    for (int step = 0; step < 100; ++step) {
      if (step % 25 == 0) {  // a fresh smooth divergent field
        std::vector<std::vector<double>> u(ps.num_blocks()), zero(ps.num_blocks());
        std::vector<const double*> pu, pz;
        origin_x = 0;
        for (int b = 0; b < ps.num_blocks(); ++b) {
          const auto d = ps.block_dims(b);
          const std::size_t G = (std::size_t)(d[0] + 2) * (d[1] + 2) * (d[2] + 2);
          u[b].assign(G, 0.0);
          zero[b].assign(G, 0.0);
          for (int k = 1; k <= d[2]; ++k)
            for (int j = 1; j <= d[1]; ++j)
              for (int i = 1; i <= d[0]; ++i) {
                const double x = (origin_x + i - 0.5) / n, y = (j - 0.5) / n;
                u[b][i + (d[0] + 2) * (j + (d[1] + 2) * (std::size_t)k)] =
                    (1.0 + 0.1 * step / 25) * std::sin(tp * x) * std::cos(tp * y);
              }
          origin_x += d[0];
          pu.push_back(u[b].data());
          pz.push_back(zero[b].data());
        }
        ps.set(SIP_FLOW_U, pu);
        ps.set(SIP_FLOW_V, pz);
        ps.set(SIP_FLOW_W, pz);
        ps.set(SIP_FLOW_P, pz);
        const double d0 = ps.divergence();
        const CorrectionReport r = ps.pressure_correct(0.01, 0.1 * d0, 50, 5);
        std::printf("step %d outer %d div %.6e -> %.6e\n", step, r.outer, r.divergence.front(),
                    r.divergence.back());
      } else {
        ps.pressure_correct(0.01, 1e300, 50, 5);  // mass check only
      }
    }
    bool caught = false;
    try {
      ps.pressure_correct(0.01, 0.0, 0, 5);
    } catch (const NonConvergenceError& e) {
      caught = e.defect() > 0.0;
    }
    std::printf("noconv %s\n", caught ? "ok" : "missing");
    std::printf("factorizations %lld\n", ps.factorizations());
  } catch (const Error& e) {
    std::printf("%s\n", e.what());
    return 3;
  }
  return 0;
}
