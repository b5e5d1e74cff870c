// sip_gen.cpp -- seeded synthetic systems of BASELINE.json's configs
// (DESIGN.md "Synthetic inputs").  Counter-based splitmix64 keyed on
// (seed, array id, global cell id), so values do not depend on the block
// decomposition or GPU placement.  The device kernel k_generate
// (sip_kernels.cu) evaluates the same expressions.
#include <cmath>
#include <cstdint>
#include <cstring>

#include "sip_internal.h"

namespace {
inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
inline double u01(uint64_t seed, uint32_t aid, uint64_t cell) {
  uint64_t h = mix64(seed ^ 0x5851F42D4C957F2DULL);
  h = mix64(h ^ ((uint64_t)(aid + 1) * 0x9E3779B97F4A7C15ULL));
  h = mix64(h ^ cell);
  return (double)(h >> 11) * 0x1.0p-53;
}
}  // namespace

extern "C" int sip_generate_host(int kind, uint64_t seed, const int g[3], const int o[3], int nx,
                                 int ny, int nz, double* AP, double* AW, double* AE, double* AS,
                                 double* AN, double* AB, double* AT, double* Q) {
  if (nx < 1 || ny < 1 || nz < 1 || !g || !o) return SIP_ERR_CONFIG;
  if (kind != 0 && kind != 2 && kind != 3) return SIP_ERR_CONFIG;
  const size_t G = (size_t)(nx + 2) * (ny + 2) * (nz + 2);
  double* arr[8] = {AP, AW, AE, AS, AN, AB, AT, Q};
  for (double* a : arr) {
    if (!a) return SIP_ERR_CONFIG;
    std::memset(a, 0, G * sizeof(double));
  }
#pragma omp parallel for schedule(static)
  for (int k = 1; k <= nz; ++k)
    for (int j = 1; j <= ny; ++j)
      for (int i = 1; i <= nx; ++i) {
        const long gi = o[0] + i - 1, gj = o[1] + j - 1, gk = o[2] + k - 1;
        const uint64_t cell =
            (uint64_t)gi + (uint64_t)g[0] * ((uint64_t)gj + (uint64_t)g[1] * (uint64_t)gk);
        double aw, ae, as, an, ab, at;
        if (kind == 2) {
          const double m = 2.0 * u01(seed, 7, cell);
          ae = -1.0; aw = -1.0 - 1.0 * m;
          an = -10.0; as = -10.0 - 0.5 * m;
          at = -100.0; ab = -100.0 - 0.25 * m;
        } else if (kind == 3) {
          // symmetric system: one coefficient per face, keyed by the face's
          // lower cell, so AW(i) = AE(i-1), AS(j) = AN(j-1), AB(k) = AT(k-1)
          const uint64_t sx = 1, sy = (uint64_t)g[0], sz = (uint64_t)g[0] * (uint64_t)g[1];
          ae = -(1.0 + 0.5 * u01(seed, 1, cell));
          an = -(1.0 + 0.5 * u01(seed, 3, cell));
          at = -(1.0 + 0.5 * u01(seed, 5, cell));
          aw = gi > 0 ? -(1.0 + 0.5 * u01(seed, 1, cell - sx)) : 0.0;
          as = gj > 0 ? -(1.0 + 0.5 * u01(seed, 3, cell - sy)) : 0.0;
          ab = gk > 0 ? -(1.0 + 0.5 * u01(seed, 5, cell - sz)) : 0.0;
        } else {
          aw = -(1.0 + 0.5 * u01(seed, 0, cell));
          ae = -(1.0 + 0.5 * u01(seed, 1, cell));
          as = -(1.0 + 0.5 * u01(seed, 2, cell));
          an = -(1.0 + 0.5 * u01(seed, 3, cell));
          ab = -(1.0 + 0.5 * u01(seed, 4, cell));
          at = -(1.0 + 0.5 * u01(seed, 5, cell));
        }
        if (gi == 0) aw = 0.0;
        if (gi == g[0] - 1) ae = 0.0;
        if (gj == 0) as = 0.0;
        if (gj == g[1] - 1) an = 0.0;
        if (gk == 0) ab = 0.0;
        if (gk == g[2] - 1) at = 0.0;
        const double s = std::fabs(aw) + std::fabs(ae) + std::fabs(as) + std::fabs(an) +
                         std::fabs(ab) + std::fabs(at);
        const size_t c = (size_t)i + (size_t)(nx + 2) * ((size_t)j + (size_t)(ny + 2) * (size_t)k);
        AP[c] = (kind == 2) ? s + 1e-3 : 1.01 * s;
        AW[c] = aw; AE[c] = ae; AS[c] = as; AN[c] = an; AB[c] = ab; AT[c] = at;
        Q[c] = 2.0 * u01(seed, 6, cell) - 1.0;
      }
  return SIP_OK;
}
