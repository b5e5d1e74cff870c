/*
 * sip_oracle.c -- CPU restatement of Stone's strongly implicit procedure (SIP)
 * for the 7-point finite-volume system, as specified by the reference.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path in paper_1303_4538_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path never links or calls it.
 *
 * Parity status: the reference (arXiv 1303.4538 artifact "bsfv") contains NO
 * SIP code -- SIP exists only as normative text.  This restatement follows:
 *   SPEC.md:116-119   StencilSystem (ap*phi_P - sum a_nb*phi_nb = su)
 *   SPEC.md:146       sip_factor recurrences (m_nb = -a_nb)
 *   SPEC.md:155       residual_general
 *   SPEC.md:164       residual_symmetric (Listing 1)
 *   SPEC.md:173       sip_sweep (forward / backward / fi += delta, L1 norm)
 *   SPEC.md:182       solve (convert once at entry / exit)
 *   SPEC.md:197-201   alpha default, L1 norm, fp32 coefficient conversion
 *   PAPER.md:479-482  single-precision relaxation variant
 *   proj/include/bsfv/field.hpp:25-44   Field3 storage (i fastest, 1 ghost)
 * It is pinned by the SPEC's known-answer properties (tests/test_oracle.py),
 * by an independent numpy restatement (oracle/oracle_np.py) and by committed
 * golden vectors (tests/golden/).  "Parity unpinned" at the reference-code
 * level: there is no reference SIP to run ("Oracle").
 *
 * Sign convention: the API takes the matrix entries
 * A_nb (negative for an M-matrix, FASTEST / Ferziger-Peric style), so
 *   AP*phi_P + sum A_nb*phi_nb = Q,  a_nb(SPEC) = -A_nb,  m_nb(SPEC) = A_nb.
 *
 * Fixed per-cell operation order (identical in the CUDA kernels):
 *   factor:   LB = AB/(1+a*(UN_B+UE_B)); LW = AW/(1+a*(UN_W+UT_W));
 *             LS = AS/(1+a*(UE_S+UT_S));
 *             P1 = a*(LB*UN_B+LW*UN_W); P2 = a*(LB*UE_B+LS*UE_S);
 *             P3 = a*(LW*UT_W+LS*UT_S);
 *             den = AP+P1+P2+P3-LB*UT_B-LW*UE_W-LS*UN_S  (left to right)
 *             LP = 1/den; UN=(AN-P1)*LP; UE=(AE-P2)*LP; UT=(AT-P3)*LP
 *   residual: r = -(AE*fE); r -= AW*fW; r -= AN*fN; r -= AS*fS;
 *             r -= AT*fT; r -= AB*fB; r += Q; r -= AP*fP   (Listing 1 order)
 *   forward:  R = (((r - LB*R_B) - LW*R_W) - LS*R_S) * LP
 *   backward: d = ((R - UN*d_N) - UE*d_E) - UT*d_T;  phi += d
 * Out-of-block factor, R and d values are zero.
 * Build with -ffp-contract=off (no FMA contraction), no fast-math.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdatomic.h>
#include <omp.h>

#define IDX(i, j, k) ((size_t)(i) + (size_t)(nx + 2) * ((size_t)(j) + (size_t)(ny + 2) * (size_t)(k)))

/* ------------------------------------------------------------------------ */
/* Seeded counter-based generator.            */
/* ------------------------------------------------------------------------ */
static uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

double orc_u01(uint64_t seed, uint32_t aid, uint64_t cell) {
  uint64_t h = mix64(seed ^ 0x5851F42D4C957F2DULL);
  h = mix64(h ^ ((uint64_t)(aid + 1) * 0x9E3779B97F4A7C15ULL));
  h = mix64(h ^ cell);
  return (double)(h >> 11) * 0x1.0p-53;
}

enum { AID_AW = 0, AID_AE, AID_AS, AID_AN, AID_AB, AID_AT, AID_Q, AID_M };

/*
 * Fill one block's system (Field3 layout, ghosts left at 0).
 *  kind 0: configs 0/1/3/4  A_nb = -(1+0.5U), AP = 1.01*sum|A_nb|, Q ~ U[-1,1]
 *  kind 2: config 2 anisotropic convection-diffusion (weights 1/10/100,
 *          upwind velocity (1,0.5,0.25)*m, m ~ U[0,2); AP = sum|A_nb| + 1e-3)
 * Block interior cell (i,j,k), 1-based, sits at global 0-based coordinates
 * (o[0]+i-1, ...) of a global domain g[0..2].  Coefficients pointing out of
 * the GLOBAL domain are zero (zeroed before AP is formed).  The generator key
 * is (seed, array, global cell id) so values do not depend on placement.
 */
void orc_generate(int kind, uint64_t seed, const int g[3], const int o[3], int nx, int ny, int nz,
                  double* AP, double* AW, double* AE, double* AS, double* AN, double* AB, double* AT,
                  double* Q) {
  size_t G = (size_t)(nx + 2) * (ny + 2) * (nz + 2);
  memset(AP, 0, G * 8); memset(AW, 0, G * 8); memset(AE, 0, G * 8); memset(AS, 0, G * 8);
  memset(AN, 0, G * 8); memset(AB, 0, G * 8); memset(AT, 0, G * 8); memset(Q, 0, G * 8);
  for (int k = 1; k <= nz; ++k)
    for (int j = 1; j <= ny; ++j)
      for (int i = 1; i <= nx; ++i) {
        long gi = o[0] + i - 1, gj = o[1] + j - 1, gk = o[2] + k - 1;
        uint64_t cell = (uint64_t)gi + (uint64_t)g[0] * ((uint64_t)gj + (uint64_t)g[1] * (uint64_t)gk);
        double aw, ae, as, an, ab, at;
        if (kind == 2) {
          double m = 2.0 * orc_u01(seed, AID_M, cell);
          ae = -1.0; aw = -1.0 - 1.0 * m;
          an = -10.0; as = -10.0 - 0.5 * m;
          at = -100.0; ab = -100.0 - 0.25 * m;
        } else if (kind == 3) {
          /* symmetric: one coefficient per face, keyed by its lower cell */
          uint64_t sy = (uint64_t)g[0], sz = (uint64_t)g[0] * (uint64_t)g[1];
          ae = -(1.0 + 0.5 * orc_u01(seed, AID_AE, cell));
          an = -(1.0 + 0.5 * orc_u01(seed, AID_AN, cell));
          at = -(1.0 + 0.5 * orc_u01(seed, AID_AT, cell));
          aw = gi > 0 ? -(1.0 + 0.5 * orc_u01(seed, AID_AE, cell - 1)) : 0.0;
          as = gj > 0 ? -(1.0 + 0.5 * orc_u01(seed, AID_AN, cell - sy)) : 0.0;
          ab = gk > 0 ? -(1.0 + 0.5 * orc_u01(seed, AID_AT, cell - sz)) : 0.0;
        } else {
          aw = -(1.0 + 0.5 * orc_u01(seed, AID_AW, cell));
          ae = -(1.0 + 0.5 * orc_u01(seed, AID_AE, cell));
          as = -(1.0 + 0.5 * orc_u01(seed, AID_AS, cell));
          an = -(1.0 + 0.5 * orc_u01(seed, AID_AN, cell));
          ab = -(1.0 + 0.5 * orc_u01(seed, AID_AB, cell));
          at = -(1.0 + 0.5 * orc_u01(seed, AID_AT, cell));
        }
        if (gi == 0) aw = 0.0;
        if (gi == g[0] - 1) ae = 0.0;
        if (gj == 0) as = 0.0;
        if (gj == g[1] - 1) an = 0.0;
        if (gk == 0) ab = 0.0;
        if (gk == g[2] - 1) at = 0.0;
        double s = fabs(aw) + fabs(ae) + fabs(as) + fabs(an) + fabs(ab) + fabs(at);
        size_t c = IDX(i, j, k);
        AW[c] = aw; AE[c] = ae; AS[c] = as; AN[c] = an; AB[c] = ab; AT[c] = at;
        AP[c] = (kind == 2) ? s + 1e-3 : 1.01 * s;
        Q[c] = 2.0 * orc_u01(seed, AID_Q, cell) - 1.0;
      }
}

/* ------------------------------------------------------------------------ */
/* sip_factor, fp64, lexicographic order.                  */
/* Returns 0, or 1 with *bad = Field3 index of the first singular cell.      */
/* ------------------------------------------------------------------------ */
int orc_factor(int nx, int ny, int nz, double alpha, const double* AP, const double* AW,
               const double* AE, const double* AS, const double* AN, const double* AB,
               const double* AT, double* LB, double* LW, double* LS, double* LP, double* UN,
               double* UE, double* UT, long long* bad) {
  size_t G = (size_t)(nx + 2) * (ny + 2) * (nz + 2);
  memset(LB, 0, G * 8); memset(LW, 0, G * 8); memset(LS, 0, G * 8); memset(LP, 0, G * 8);
  memset(UN, 0, G * 8); memset(UE, 0, G * 8); memset(UT, 0, G * 8);
  const size_t sj = nx + 2, sk = (size_t)(nx + 2) * (ny + 2);
  if (bad) *bad = -1;
  for (int k = 1; k <= nz; ++k)
    for (int j = 1; j <= ny; ++j)
      for (int i = 1; i <= nx; ++i) {
        size_t c = IDX(i, j, k), w = c - 1, s = c - sj, b = c - sk;
        double lb = AB[c] / (1.0 + alpha * (UN[b] + UE[b]));
        double lw = AW[c] / (1.0 + alpha * (UN[w] + UT[w]));
        double ls = AS[c] / (1.0 + alpha * (UE[s] + UT[s]));
        double p1 = alpha * (lb * UN[b] + lw * UN[w]);
        double p2 = alpha * (lb * UE[b] + ls * UE[s]);
        double p3 = alpha * (lw * UT[w] + ls * UT[s]);
        double den = AP[c] + p1 + p2 + p3 - lb * UT[b] - lw * UE[w] - ls * UN[s];
        if (!(fabs(den) >= 1e-30)) {
          if (bad) *bad = (long long)c;
          return 1;
        }
        double lp = 1.0 / den;
        LB[c] = lb; LW[c] = lw; LS[c] = ls; LP[c] = lp;
        UN[c] = (AN[c] - p1) * lp;
        UE[c] = (AE[c] - p2) * lp;
        UT[c] = (AT[c] - p3) * lp;
      }
  return 0;
}

/* residual_general -- res at interior cells, Listing-1 order */
void orc_residual(int nx, int ny, int nz, const double* AP, const double* AW, const double* AE,
                  const double* AS, const double* AN, const double* AB, const double* AT,
                  const double* Q, const double* phi, double* res) {
  const size_t sj = nx + 2, sk = (size_t)(nx + 2) * (ny + 2);
  for (int k = 1; k <= nz; ++k)
    for (int j = 1; j <= ny; ++j)
      for (int i = 1; i <= nx; ++i) {
        size_t c = IDX(i, j, k);
        double r = -(AE[c] * phi[c + 1]);
        r -= AW[c] * phi[c - 1];
        r -= AN[c] * phi[c + sj];
        r -= AS[c] * phi[c - sj];
        r -= AT[c] * phi[c + sk];
        r -= AB[c] * phi[c - sk];
        r += Q[c];
        r -= AP[c] * phi[c];
        res[c] = r;
      }
}

/*
 * residual_symmetric (Listing 1): reads only
 * AE/AN/AT (own and shifted) -- A_W(i) = A_E(i-1) etc. for symmetric systems.
 * Term order equals residual_general, so results are bitwise identical when
 * the system is exactly symmetric.
 */
void orc_residual_symmetric(int nx, int ny, int nz, const double* AP, const double* AE,
                            const double* AN, const double* AT, const double* Q,
                            const double* phi, double* res) {
  const size_t sj = nx + 2, sk = (size_t)(nx + 2) * (ny + 2);
  for (int k = 1; k <= nz; ++k)
    for (int j = 1; j <= ny; ++j)
      for (int i = 1; i <= nx; ++i) {
        size_t c = IDX(i, j, k);
        /* shifted coefficients; at i=1 (j=1, k=1) this reads the ghost layer
         * of AE (AN, AT), which carries the coupling to the W (S, B) side */
        double aw = AE[c - 1];
        double as = AN[c - sj];
        double ab = AT[c - sk];
        double r = -(AE[c] * phi[c + 1]);
        r -= aw * phi[c - 1];
        r -= AN[c] * phi[c + sj];
        r -= as * phi[c - sj];
        r -= AT[c] * phi[c + sk];
        r -= ab * phi[c - sk];
        r += Q[c];
        r -= AP[c] * phi[c];
        res[c] = r;
      }
}

/*
 * One SIP inner iteration, fp64.  work: G doubles (R, then
 * delta in place).  Returns the L1 norm of the pre-update residual.
 */
double orc_sweep_d(int nx, int ny, int nz, const double* AP, const double* AW, const double* AE,
                   const double* AS, const double* AN, const double* AB, const double* AT,
                   const double* Q, const double* LB, const double* LW, const double* LS,
                   const double* LP, const double* UN, const double* UE, const double* UT,
                   double* phi, double* work) {
  const size_t sj = nx + 2, sk = (size_t)(nx + 2) * (ny + 2);
  size_t G = (size_t)(nx + 2) * (ny + 2) * (nz + 2);
  memset(work, 0, G * 8);
  double norm = 0.0;
  for (int k = 1; k <= nz; ++k)
    for (int j = 1; j <= ny; ++j)
      for (int i = 1; i <= nx; ++i) {
        size_t c = IDX(i, j, k);
        double r = -(AE[c] * phi[c + 1]);
        r -= AW[c] * phi[c - 1];
        r -= AN[c] * phi[c + sj];
        r -= AS[c] * phi[c - sj];
        r -= AT[c] * phi[c + sk];
        r -= AB[c] * phi[c - sk];
        r += Q[c];
        r -= AP[c] * phi[c];
        norm += fabs(r);
        work[c] = (((r - LB[c] * work[c - sk]) - LW[c] * work[c - 1]) - LS[c] * work[c - sj]) * LP[c];
      }
  for (int k = nz; k >= 1; --k)
    for (int j = ny; j >= 1; --j)
      for (int i = nx; i >= 1; --i) {
        size_t c = IDX(i, j, k);
        double d = ((work[c] - UN[c] * work[c + sj]) - UE[c] * work[c + 1]) - UT[c] * work[c + sk];
        work[c] = d;
        phi[c] += d;
      }
  return norm;
}

/* Residual + forward substitution only (R left in work); returns the norm. */
double orc_forward_d(int nx, int ny, int nz, const double* AP, const double* AW, const double* AE,
                     const double* AS, const double* AN, const double* AB, const double* AT,
                     const double* Q, const double* LB, const double* LW, const double* LS,
                     const double* LP, const double* phi, double* work) {
  const size_t sj = nx + 2, sk = (size_t)(nx + 2) * (ny + 2);
  size_t G = (size_t)(nx + 2) * (ny + 2) * (nz + 2);
  memset(work, 0, G * 8);
  double norm = 0.0;
  for (int k = 1; k <= nz; ++k)
    for (int j = 1; j <= ny; ++j)
      for (int i = 1; i <= nx; ++i) {
        size_t c = IDX(i, j, k);
        double r = -(AE[c] * phi[c + 1]);
        r -= AW[c] * phi[c - 1];
        r -= AN[c] * phi[c + sj];
        r -= AS[c] * phi[c - sj];
        r -= AT[c] * phi[c + sk];
        r -= AB[c] * phi[c - sk];
        r += Q[c];
        r -= AP[c] * phi[c];
        norm += fabs(r);
        work[c] = (((r - LB[c] * work[c - sk]) - LW[c] * work[c - 1]) - LS[c] * work[c - sj]) * LP[c];
      }
  return norm;
}

/* Same iteration with every relaxation array in fp32. */
double orc_sweep_f(int nx, int ny, int nz, const float* AP, const float* AW, const float* AE,
                   const float* AS, const float* AN, const float* AB, const float* AT,
                   const float* Q, const float* LB, const float* LW, const float* LS,
                   const float* LP, const float* UN, const float* UE, const float* UT, float* phi,
                   float* work) {
  const size_t sj = nx + 2, sk = (size_t)(nx + 2) * (ny + 2);
  size_t G = (size_t)(nx + 2) * (ny + 2) * (nz + 2);
  memset(work, 0, G * 4);
  double norm = 0.0;
  for (int k = 1; k <= nz; ++k)
    for (int j = 1; j <= ny; ++j)
      for (int i = 1; i <= nx; ++i) {
        size_t c = IDX(i, j, k);
        float r = -(AE[c] * phi[c + 1]);
        r -= AW[c] * phi[c - 1];
        r -= AN[c] * phi[c + sj];
        r -= AS[c] * phi[c - sj];
        r -= AT[c] * phi[c + sk];
        r -= AB[c] * phi[c - sk];
        r += Q[c];
        r -= AP[c] * phi[c];
        norm += fabs((double)r);
        work[c] = (((r - LB[c] * work[c - sk]) - LW[c] * work[c - 1]) - LS[c] * work[c - sj]) * LP[c];
      }
  for (int k = nz; k >= 1; --k)
    for (int j = ny; j >= 1; --j)
      for (int i = nx; i >= 1; --i) {
        size_t c = IDX(i, j, k);
        float d = ((work[c] - UN[c] * work[c + sj]) - UE[c] * work[c + 1]) - UT[c] * work[c + sk];
        work[c] = d;
        phi[c] += d;
      }
  return norm;
}

/* ------------------------------------------------------------------------ */
/* The same iteration on `nthreads` host threads (the CPU reference arm of   */
/* bench.py: "the reference's algorithm with all the host threads it can     */
/* use").  Pipelined over j-slabs: thread t owns rows [j0_t, j1_t); in the   */
/* forward pass it processes plane k after thread t-1 finished plane k (the  */
/* S neighbour row), in the backward pass after thread t+1 finished it.      */
/* Every cell does the serial sweep's operations on the same operands, so    */
/* phi is bitwise equal to orc_sweep_d/_f; the norm is summed per thread and */
/* the partials in thread order (a different summation order).  work must    */
/* be zero on its ghost layer (it is never written there).                   */
/* ------------------------------------------------------------------------ */
#define SWEEP_PIPE(NAME, T)                                                                       \
  double NAME(int nx, int ny, int nz, const T* AP, const T* AW, const T* AE, const T* AS,          \
              const T* AN, const T* AB, const T* AT, const T* Q, const T* LB, const T* LW,         \
              const T* LS, const T* LP, const T* UN, const T* UE, const T* UT, T* phi, T* work,    \
              int nthreads) {                                                                     \
    const size_t sj = nx + 2, sk = (size_t)(nx + 2) * (ny + 2);                                   \
    int nt = nthreads < 1 ? 1 : nthreads;                                                         \
    if (nt > ny) nt = ny;                                                                         \
    /* per-thread progress, one cache line each: planes done (forward, backward) */               \
    _Atomic int* prog = (_Atomic int*)calloc((size_t)nt * 32, sizeof(int));                       \
    double* part = (double*)calloc((size_t)nt, sizeof(double));                                   \
    _Pragma("omp parallel num_threads(nt)")                                                       \
    {                                                                                             \
      const int t = omp_get_thread_num();                                                         \
      const int j0 = 1 + (int)((long long)ny * t / nt), j1 = 1 + (int)((long long)ny * (t + 1) / nt); \
      _Atomic int* fwd = prog + 32 * t;                                                           \
      _Atomic int* bwd = prog + 32 * t + 16;                                                      \
      double norm = 0.0;                                                                          \
      for (int k = 1; k <= nz; ++k) {                                                             \
        if (t > 0)                                                                                \
          while (atomic_load_explicit(prog + 32 * (t - 1), memory_order_acquire) < k) {           \
          }                                                                                       \
        for (int j = j0; j < j1; ++j)                                                             \
          for (int i = 1; i <= nx; ++i) {                                                         \
            size_t c = IDX(i, j, k);                                                              \
            T r = -(AE[c] * phi[c + 1]);                                                          \
            r -= AW[c] * phi[c - 1];                                                              \
            r -= AN[c] * phi[c + sj];                                                             \
            r -= AS[c] * phi[c - sj];                                                             \
            r -= AT[c] * phi[c + sk];                                                             \
            r -= AB[c] * phi[c - sk];                                                             \
            r += Q[c];                                                                            \
            r -= AP[c] * phi[c];                                                                  \
            norm += fabs((double)r);                                                              \
            work[c] = (((r - LB[c] * work[c - sk]) - LW[c] * work[c - 1]) - LS[c] * work[c - sj]) * LP[c]; \
          }                                                                                       \
        atomic_store_explicit(fwd, k, memory_order_release);                                      \
      }                                                                                           \
      /* all residuals are read from the old phi: no thread may update phi  */                    \
      /* before every thread finished its forward pass                       */                   \
      _Pragma("omp barrier")                                                                      \
      for (int k = nz; k >= 1; --k) {                                                             \
        if (t < nt - 1)                                                                           \
          while (atomic_load_explicit(prog + 32 * (t + 1) + 16, memory_order_acquire) <           \
                 nz - k + 1) {                                                                    \
          }                                                                                       \
        for (int j = j1 - 1; j >= j0; --j)                                                        \
          for (int i = nx; i >= 1; --i) {                                                         \
            size_t c = IDX(i, j, k);                                                              \
            T d = ((work[c] - UN[c] * work[c + sj]) - UE[c] * work[c + 1]) - UT[c] * work[c + sk]; \
            work[c] = d;                                                                          \
            phi[c] += d;                                                                          \
          }                                                                                       \
        atomic_store_explicit(bwd, nz - k + 1, memory_order_release);                             \
      }                                                                                           \
      part[t] = norm;                                                                             \
    }                                                                                             \
    double norm = 0.0;                                                                            \
    for (int t = 0; t < nt; ++t) norm += part[t];                                                 \
    free(prog);                                                                                   \
    free(part);                                                                                   \
    return norm;                                                                                  \
  }
SWEEP_PIPE(orc_sweep_pipe_d, double)
SWEEP_PIPE(orc_sweep_pipe_f, float)

/* ------------------------------------------------------------------------ */
/* Single-block solve with a fixed iteration count.        */
/* precision 0 = fp64, 1 = fp32 relaxation (convert su/fi/coefficients/      */
/* factors once at entry, phi back once at exit).  A = 8 arrays in order     */
/* AP,AW,AE,AS,AN,AB,AT,Q.  Returns 0, 1 (singular; *bad set) or 2 (alloc).  */
/* ------------------------------------------------------------------------ */
static void* xalloc(size_t n) { return malloc(n ? n : 1); }

int orc_solve(int nx, int ny, int nz, int precision, double alpha, int iters,
              const double* const A[8], double* phi, double* norms, long long* bad) {
  size_t G = (size_t)(nx + 2) * (ny + 2) * (nz + 2);
  double* F = (double*)xalloc(7 * G * 8);
  if (!F) return 2;
  double *LB = F, *LW = F + G, *LS = F + 2 * G, *LP = F + 3 * G, *UN = F + 4 * G, *UE = F + 5 * G,
         *UT = F + 6 * G;
  int rc = orc_factor(nx, ny, nz, alpha, A[0], A[1], A[2], A[3], A[4], A[5], A[6], LB, LW, LS, LP,
                      UN, UE, UT, bad);
  if (rc) { free(F); return rc; }
  if (precision == 0) {
    double* work = (double*)xalloc(G * 8);
    for (int it = 0; it < iters; ++it)
      norms[it] = orc_sweep_d(nx, ny, nz, A[0], A[1], A[2], A[3], A[4], A[5], A[6], A[7], LB, LW,
                              LS, LP, UN, UE, UT, phi, work);
    free(work);
  } else {
    float* S = (float*)xalloc(17 * G * 4);
    for (int a = 0; a < 8; ++a)
      for (size_t n = 0; n < G; ++n) S[a * G + n] = (float)A[a][n];
    for (int a = 0; a < 7; ++a)
      for (size_t n = 0; n < G; ++n) S[(8 + a) * G + n] = (float)F[a * G + n];
    float* ph = S + 15 * G;
    float* work = S + 16 * G;
    for (size_t n = 0; n < G; ++n) ph[n] = (float)phi[n];
    for (int it = 0; it < iters; ++it)
      norms[it] = orc_sweep_f(nx, ny, nz, S, S + G, S + 2 * G, S + 3 * G, S + 4 * G, S + 5 * G,
                              S + 6 * G, S + 7 * G, S + 8 * G, S + 9 * G, S + 10 * G, S + 11 * G,
                              S + 12 * G, S + 13 * G, S + 14 * G, ph, work);
    /* back-conversion of the interior only; ghost inputs stay untouched */
    for (int k = 1; k <= nz; ++k)
      for (int j = 1; j <= ny; ++j)
        for (int i = 1; i <= nx; ++i) phi[IDX(i, j, k)] = (double)ph[IDX(i, j, k)];
    free(S);
  }
  free(F);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Multi-block block-Jacobi SIP (SPEC.md:152-155 ghosts, SPEC.md:263-271     */
/* exchange after every inner iteration, SPEC.md:272-276 fixed-order sum).   */
/* Block b has dims[b*3..], origin org[b*3..] (0-based global), neighbour    */
/* block ids nbr[b*6 + face] (face order W,E,S,N,B,T; -1 = domain boundary). */
/* A[b*8 + a] = array a of block b, phi[b] = block b's Field3 phi (ghosts on  */
/* domain-boundary faces are honoured; interface ghosts are overwritten by    */
/* the exchange).  Factorisation is block-local.  norms[it] = sum over b in   */
/* ascending block order of the block's L1 norm; block_norms[it*nb + b] if    */
/* non-NULL.  nthreads > 1 relaxes blocks concurrently (same results).        */
/* ------------------------------------------------------------------------ */
static void exchange_faces(int nb, const int* dims, const int* nbr, double* const* phi) {
  for (int b = 0; b < nb; ++b) {
    int nx = dims[3 * b], ny = dims[3 * b + 1], nz = dims[3 * b + 2];
    for (int f = 0; f < 6; ++f) {
      int q = nbr[6 * b + f];
      if (q < 0) continue;
      int mx = dims[3 * q], my = dims[3 * q + 1];
      const double* src = phi[q];
      double* dst = phi[b];
#define QIDX(i, j, k) ((size_t)(i) + (size_t)(mx + 2) * ((size_t)(j) + (size_t)(my + 2) * (size_t)(k)))
      if (f == 0 || f == 1) { /* W: ghost i=0 <- q's i=mx ; E: ghost i=nx+1 <- q's i=1 */
        int gi = (f == 0) ? 0 : nx + 1, si = (f == 0) ? mx : 1;
        for (int k = 1; k <= nz; ++k)
          for (int j = 1; j <= ny; ++j) dst[IDX(gi, j, k)] = src[QIDX(si, j, k)];
      } else if (f == 2 || f == 3) {
        int gj = (f == 2) ? 0 : ny + 1, sj = (f == 2) ? my : 1;
        for (int k = 1; k <= nz; ++k)
          for (int i = 1; i <= nx; ++i) dst[IDX(i, gj, k)] = src[QIDX(i, sj, k)];
      } else {
        int mz = dims[3 * q + 2];
        int gk = (f == 4) ? 0 : nz + 1, sk = (f == 4) ? mz : 1;
        for (int j = 1; j <= ny; ++j)
          for (int i = 1; i <= nx; ++i) dst[IDX(i, j, gk)] = src[QIDX(i, j, sk)];
      }
#undef QIDX
    }
  }
}

static void exchange_faces_f(int nb, const int* dims, const int* nbr, float* const* phi) {
  for (int b = 0; b < nb; ++b) {
    int nx = dims[3 * b], ny = dims[3 * b + 1], nz = dims[3 * b + 2];
    for (int f = 0; f < 6; ++f) {
      int q = nbr[6 * b + f];
      if (q < 0) continue;
      int mx = dims[3 * q], my = dims[3 * q + 1];
      const float* src = phi[q];
      float* dst = phi[b];
#define QIDX(i, j, k) ((size_t)(i) + (size_t)(mx + 2) * ((size_t)(j) + (size_t)(my + 2) * (size_t)(k)))
      if (f == 0 || f == 1) {
        int gi = (f == 0) ? 0 : nx + 1, si = (f == 0) ? mx : 1;
        for (int k = 1; k <= nz; ++k)
          for (int j = 1; j <= ny; ++j) dst[IDX(gi, j, k)] = src[QIDX(si, j, k)];
      } else if (f == 2 || f == 3) {
        int gj = (f == 2) ? 0 : ny + 1, sj = (f == 2) ? my : 1;
        for (int k = 1; k <= nz; ++k)
          for (int i = 1; i <= nx; ++i) dst[IDX(i, gj, k)] = src[QIDX(i, sj, k)];
      } else {
        int mz = dims[3 * q + 2];
        int gk = (f == 4) ? 0 : nz + 1, sk = (f == 4) ? mz : 1;
        for (int j = 1; j <= ny; ++j)
          for (int i = 1; i <= nx; ++i) dst[IDX(i, j, gk)] = src[QIDX(i, j, sk)];
      }
#undef QIDX
    }
  }
}

int orc_solve_multi(int nb, const int* dims, const int* nbr, int precision, double alpha, int iters,
                    const double* const* A, double* const* phi, double* norms, double* block_norms,
                    int nthreads, long long* bad) {
  double** F = (double**)calloc(nb, sizeof(double*));
  int rc = 0;
  for (int b = 0; b < nb && !rc; ++b) {
    int nx = dims[3 * b], ny = dims[3 * b + 1], nz = dims[3 * b + 2];
    size_t G = (size_t)(nx + 2) * (ny + 2) * (nz + 2);
    F[b] = (double*)xalloc(7 * G * 8);
    const double* const* a = A + 8 * b;
    rc = orc_factor(nx, ny, nz, alpha, a[0], a[1], a[2], a[3], a[4], a[5], a[6], F[b], F[b] + G,
                    F[b] + 2 * G, F[b] + 3 * G, F[b] + 4 * G, F[b] + 5 * G, F[b] + 6 * G, bad);
  }
  if (rc) goto done;
  double* bn = (double*)xalloc((size_t)nb * 8);
  if (precision == 0) {
    double** work = (double**)calloc(nb, sizeof(double*));
    for (int b = 0; b < nb; ++b) {
      size_t G = (size_t)(dims[3 * b] + 2) * (dims[3 * b + 1] + 2) * (dims[3 * b + 2] + 2);
      work[b] = (double*)xalloc(G * 8);
    }
    exchange_faces(nb, dims, nbr, phi);
    for (int it = 0; it < iters; ++it) {
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1) if (nthreads > 1)
      for (int b = 0; b < nb; ++b) {
        int nx = dims[3 * b], ny = dims[3 * b + 1], nz = dims[3 * b + 2];
        size_t G = (size_t)(nx + 2) * (ny + 2) * (nz + 2);
        const double* const* a = A + 8 * b;
        double* f = F[b];
        bn[b] = orc_sweep_d(nx, ny, nz, a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], f, f + G,
                            f + 2 * G, f + 3 * G, f + 4 * G, f + 5 * G, f + 6 * G, phi[b], work[b]);
      }
      double s = 0.0;
      for (int b = 0; b < nb; ++b) {
        s += bn[b];
        if (block_norms) block_norms[(size_t)it * nb + b] = bn[b];
      }
      norms[it] = s;
      exchange_faces(nb, dims, nbr, phi);
    }
    for (int b = 0; b < nb; ++b) free(work[b]);
    free(work);
  } else {
    float** S = (float**)calloc(nb, sizeof(float*));
    float** ph = (float**)calloc(nb, sizeof(float*));
    for (int b = 0; b < nb; ++b) {
      size_t G = (size_t)(dims[3 * b] + 2) * (dims[3 * b + 1] + 2) * (dims[3 * b + 2] + 2);
      S[b] = (float*)xalloc(17 * G * 4);
      for (int a = 0; a < 8; ++a)
        for (size_t n = 0; n < G; ++n) S[b][a * G + n] = (float)A[8 * b + a][n];
      for (int a = 0; a < 7; ++a)
        for (size_t n = 0; n < G; ++n) S[b][(8 + a) * G + n] = (float)F[b][a * G + n];
      ph[b] = S[b] + 15 * G;
      for (size_t n = 0; n < G; ++n) ph[b][n] = (float)phi[b][n];
    }
    exchange_faces_f(nb, dims, nbr, ph);
    for (int it = 0; it < iters; ++it) {
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1) if (nthreads > 1)
      for (int b = 0; b < nb; ++b) {
        int nx = dims[3 * b], ny = dims[3 * b + 1], nz = dims[3 * b + 2];
        size_t G = (size_t)(nx + 2) * (ny + 2) * (nz + 2);
        float* s = S[b];
        bn[b] = orc_sweep_f(nx, ny, nz, s, s + G, s + 2 * G, s + 3 * G, s + 4 * G, s + 5 * G,
                            s + 6 * G, s + 7 * G, s + 8 * G, s + 9 * G, s + 10 * G, s + 11 * G,
                            s + 12 * G, s + 13 * G, s + 14 * G, ph[b], s + 16 * G);
      }
      double s = 0.0;
      for (int b = 0; b < nb; ++b) {
        s += bn[b];
        if (block_norms) block_norms[(size_t)it * nb + b] = bn[b];
      }
      norms[it] = s;
      exchange_faces_f(nb, dims, nbr, ph);
    }
    for (int b = 0; b < nb; ++b) {
      int nx = dims[3 * b], ny = dims[3 * b + 1], nz = dims[3 * b + 2];
      for (int k = 1; k <= nz; ++k)
        for (int j = 1; j <= ny; ++j)
          for (int i = 1; i <= nx; ++i) phi[b][IDX(i, j, k)] = (double)ph[b][IDX(i, j, k)];
    }
    /* interface ghosts = neighbours' (converted) interior, as after an exchange */
    exchange_faces(nb, dims, nbr, phi);
    for (int b = 0; b < nb; ++b) free(S[b]);
    free(S);
    free(ph);
  }
  free(bn);
done:
  for (int b = 0; b < nb; ++b) free(F[b]);
  free(F);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Block-Jacobi SIP over a generated lattice, memory-lean (test driver for   */
/* the full-size BASELINE configs): same algorithm and results as           */
/* orc_solve_multi on orc_generate's systems, but each block's system is     */
/* regenerated and refactored on the fly every iteration (the work arrays    */
/* of a block live only while a thread relaxes it), so a 128-block lattice   */
/* needs ~1 phi per block instead of 16 arrays per block.  Block b's system  */
/* is orc_generate(kind, seed0 + b, g, org[3b..], dims[3b..]).  phi[b]:      */
/* Field3 fp64, interior written back at the end (fp32: converted once at    */
/* entry / exit, interface ghosts = neighbours' converted interior).         */
/* ------------------------------------------------------------------------ */
int orc_solve_multi_gen(int kind, uint64_t seed0, const int g[3], int nb, const int* org,
                        const int* dims, const int* nbr, int precision, double alpha, int iters,
                        double* const* phi, double* norms, double* block_norms, int nthreads,
                        long long* bad) {
  int rc = 0;
  double* bn = (double*)xalloc((size_t)nb * 8);
  float** ph = NULL;
  if (precision != 0) {
    ph = (float**)calloc(nb, sizeof(float*));
    for (int b = 0; b < nb; ++b) {
      size_t G = (size_t)(dims[3 * b] + 2) * (dims[3 * b + 1] + 2) * (dims[3 * b + 2] + 2);
      ph[b] = (float*)xalloc(G * 4);
      for (size_t n = 0; n < G; ++n) ph[b][n] = (float)phi[b][n];
    }
    exchange_faces_f(nb, dims, nbr, ph);
  } else {
    exchange_faces(nb, dims, nbr, phi);
  }
  for (int it = 0; it < iters && !rc; ++it) {
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1) if (nthreads > 1)
    for (int b = 0; b < nb; ++b) {
      int nx = dims[3 * b], ny = dims[3 * b + 1], nz = dims[3 * b + 2];
      size_t G = (size_t)(nx + 2) * (ny + 2) * (nz + 2);
      double* A = (double*)xalloc(16 * G * 8); /* 8 arrays + 7 factors + work */
      double* F = A + 8 * G;
      orc_generate(kind, seed0 + (uint64_t)b, g, org + 3 * b, nx, ny, nz, A, A + G, A + 2 * G,
                   A + 3 * G, A + 4 * G, A + 5 * G, A + 6 * G, A + 7 * G);
      long long bb = -1;
      int r = orc_factor(nx, ny, nz, alpha, A, A + G, A + 2 * G, A + 3 * G, A + 4 * G, A + 5 * G,
                         A + 6 * G, F, F + G, F + 2 * G, F + 3 * G, F + 4 * G, F + 5 * G, F + 6 * G,
                         &bb);
      if (r) {
#pragma omp critical
        {
          rc = 1;
          if (bad) *bad = bb;
        }
      } else if (precision == 0) {
        bn[b] = orc_sweep_d(nx, ny, nz, A, A + G, A + 2 * G, A + 3 * G, A + 4 * G, A + 5 * G,
                            A + 6 * G, A + 7 * G, F, F + G, F + 2 * G, F + 3 * G, F + 4 * G,
                            F + 5 * G, F + 6 * G, phi[b], F + 7 * G);
      } else {
        float* S = (float*)xalloc(16 * G * 4);
        for (int a = 0; a < 15; ++a)
          for (size_t n = 0; n < G; ++n) S[a * G + n] = (float)A[a * G + n];
        bn[b] = orc_sweep_f(nx, ny, nz, S, S + G, S + 2 * G, S + 3 * G, S + 4 * G, S + 5 * G,
                            S + 6 * G, S + 7 * G, S + 8 * G, S + 9 * G, S + 10 * G, S + 11 * G,
                            S + 12 * G, S + 13 * G, S + 14 * G, ph[b], S + 15 * G);
        free(S);
      }
      free(A);
    }
    if (rc) break;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) {
      s += bn[b];
      if (block_norms) block_norms[(size_t)it * nb + b] = bn[b];
    }
    norms[it] = s;
    if (precision != 0) exchange_faces_f(nb, dims, nbr, ph);
    else exchange_faces(nb, dims, nbr, phi);
  }
  if (precision != 0) {
    for (int b = 0; b < nb; ++b) {
      int nx = dims[3 * b], ny = dims[3 * b + 1], nz = dims[3 * b + 2];
      for (int k = 1; k <= nz; ++k)
        for (int j = 1; j <= ny; ++j)
          for (int i = 1; i <= nx; ++i) phi[b][IDX(i, j, k)] = (double)ph[b][IDX(i, j, k)];
      free(ph[b]);
    }
    free(ph);
    exchange_faces(nb, dims, nbr, phi);
  }
  free(bn);
  return rc;
}
