/*
 * sip_c.h -- C-ABI of the B200-native SIP (Stone's strongly implicit
 * procedure) hot path.  Plain pointers and sizes only; no CUDA / torch types.
 *
 * The reference (arXiv 1303.4538 artifact "bsfv", /root/reference) defines
 * SIP only as a specification; the entry points below replace the SPEC's sip
 * module operations one for one:
 *
 *   reference                         this ABI
 *   ------------------------------------------  -------------------------------
 *   StencilSystem          SPEC.md:116-119       sip_set_system / sip_set_source
 *   SipFactors + stamp     SPEC.md:120-123       factor state inside sip_ctx
 *   SipConfig              SPEC.md:124-127       alpha / max_iters / target / precision args
 *   SolveReport            SPEC.md:128-131       norms_out / iters_used / sip_report
 *   sip_factor             SPEC.md:143-151       sip_factor
 *   residual_general       SPEC.md:152-160       sip_residual
 *   residual_symmetric     SPEC.md:161-169       sip_residual (symmetric = 1)
 *   sip_sweep              SPEC.md:170-178       sip_iterate (iters = 1)
 *   solve                  SPEC.md:179-187       sip_solve
 *   decompose / with_ranks proj/src/grid.cpp:50-102   sip_create_lattice
 *   Endpoint::all_reduce   proj/include/bsfv/net.hpp:131  (inside; NCCL)
 *   exchange_nonblocking   SPEC.md:263-271       (inside; device copies + NCCL)
 *   Field3<double>         proj/include/bsfv/field.hpp:21-44  host array layout
 *   assemble_poisson       SPEC.md:134-142       sip_assemble_poisson
 *   pressure_correct       SPEC.md:341-349       sip_flow_* / sip_pressure_correct
 *   build_transfers (periodic wraps) transfers.cpp:15-25  sip_plan_halo_periodic
 *
 * Host arrays use the reference's Field3 layout: (nx+2)*(ny+2)*(nz+2) doubles,
 * index i + (nx+2)*(j + (ny+2)*k), interior 1..n, one ghost layer.  The sign
 * convention is the matrix-entry one (FASTEST / Ferziger-Peric):
 *   AP*phi_P + AW*phi_W + AE*phi_E + AS*phi_S + AN*phi_N + AB*phi_B + AT*phi_T = Q
 * i.e. SPEC's a_nb = -A_nb.
 *
 * Every function returns a SIP_* status and never throws.  The C++ shim
 * include/bsfv_sip.hpp maps statuses onto the reference's exception classes
 * (proj/include/bsfv/error.hpp:10-50).  Threading: one context per host
 * thread / rank; calls only from the owning thread.
 */
#ifndef SIP_C_H_
#define SIP_C_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes -> bsfv exception classes (error.hpp). */
#define SIP_OK 0
#define SIP_ERR_SINGULAR 1 /* SingularFactorError  error.hpp:34-37 */
#define SIP_ERR_STALE 2    /* StaleFactorsError    error.hpp:40-43 */
#define SIP_ERR_MISUSE 3   /* MisuseError          error.hpp:47-50 */
#define SIP_ERR_CONFIG 4   /* ConfigError          error.hpp:16-19 */
#define SIP_ERR_CUDA 5     /* Error (device failure)               */
#define SIP_ERR_NCCL 6     /* Error (collective failure)           */
#define SIP_ERR_NOMEM 7    /* Error (device allocation)            */
#define SIP_ERR_FORMAT 8   /* FormatError          error.hpp:22-31 (byte offset) */
#define SIP_ERR_PROTOCOL 9 /* ProtocolError        error.hpp:53-57 */
#define SIP_ERR_NOCONV 10  /* pressure_correct: outer cap reached above the mass threshold
                              (non-convergence error carrying the defect norm) */

/* bsfv::Precision (field.hpp:10): relaxation precision. */
#define SIP_PREC_DOUBLE 0
#define SIP_PREC_SINGLE 1

typedef struct sip_ctx sip_ctx;

/* Library version string and build flags ("sm_100a ..."). */
const char* sip_version(void);
const char* sip_status_string(int status);
/* Last error message of a context (or of the last failed create if ctx NULL). */
const char* sip_last_error(const sip_ctx* ctx);

/*
 * Single block of nx*ny*nz interior cells on CUDA device `device`.
 */
int sip_create(int device, int nx, int ny, int nz, int precision, sip_ctx** out);

/*
 * Block-structured grid gnx*gny*gnz split into px*py*pz blocks exactly as
 * bsfv::decompose (grid.cpp:50-89: even split, remainder to the last block
 * per axis; block id = bx + px*(by + py*bz)).  block_rank[nblocks] assigns
 * blocks to ranks (NULL: compact sub-lattices, see sip_plan_block_ranks);
 * this process is `rank` of `nranks` and owns the blocks mapped to it.
 * nccl_id: 128-byte ncclUniqueId shared by all ranks (NULL when nranks == 1).
 */
int sip_create_lattice(int device, int gnx, int gny, int gnz, int px, int py, int pz,
                       const int* block_rank, int rank, int nranks, const void* nccl_id,
                       int precision, sip_ctx** out);
int sip_destroy(sip_ctx* ctx);

/* Local blocks of this rank, ascending block id. */
int sip_num_local_blocks(const sip_ctx* ctx, int* n);
int sip_local_block(const sip_ctx* ctx, int local, int* block_id, int dims[3], int origin[3]);

/*
 * Stencil system of one local block (Field3 host arrays, G doubles each).
 * Bumps the system revision (stale factors are detected).
 */
int sip_set_system(sip_ctx* ctx, int local, const double* ap, const double* aw,
                   const double* ae, const double* as, const double* an, const double* ab,
                   const double* at, const double* q);
/* Source term only (su changes per RK stage; factors stay valid). */
int sip_set_source(sip_ctx* ctx, int local, const double* q);
/* Seeded synthetic system generated on the device:
 * kind 0 = configs 0/1/3/4 generator, kind 2 = config 2, kind 3 = symmetric
 * (one coefficient per face; sip_set_symmetric accepts it); seed per block =
 * seed + block id.  Same values as sip_generate_host. */
int sip_generate_system(sip_ctx* ctx, int kind, uint64_t seed);

/*
 * Stone incomplete-LU factorisation of every local block.
 * On SIP_ERR_SINGULAR, *bad_block / *bad_cell name the first singular cell
 * (block id, Field3 index) in lexicographic order.
 */
int sip_factor(sip_ctx* ctx, double alpha, long long* bad_block, long long* bad_cell);

/*
 * solve on the reuse path: phi[local] (Field3 host arrays,
 * in/out) converted once at entry / exit; iterate until norm/norm[0] <=
 * target or max_iters (target <= 0: fixed count; target >= 1: no-op, 0
 * iterations).  norms_out[max_iters] receives the per-iteration L1 norm of
 * the pre-update residual, summed over all blocks of all ranks in block order.
 */
int sip_solve(sip_ctx* ctx, double* const* phi, int max_iters, double target, double* norms_out,
              int* iters_used);
/* sip_solve with the norm-evaluation interval of the target-reduction mode
 * (SPEC.md DESIGN DECISIONS: "every s-th sweep").  Single rank: the stop is
 * exact (the forward sweep's finaliser tests norm/norm[0] <= target on the
 * device and the remaining sweeps return at once); check_every only sets how
 * often the host polls the stop flag (<= 0: never before the end).  Several
 * ranks: the global norm is all-gathered and tested every check_every sweeps
 * (>= 1), so the solve stops at the first tested sweep meeting the target.
 * sip_solve = check_every 8 (single rank) / 1 (several ranks). */
int sip_solve_ex(sip_ctx* ctx, double* const* phi, int max_iters, double target, int check_every,
                 double* norms_out, int* iters_used);

/* Device-resident path (used for the HBM-resident throughput number). */
int sip_load_phi(sip_ctx* ctx, double* const* phi);      /* host Field3 -> device */
int sip_store_phi(sip_ctx* ctx, double* const* phi);     /* device -> host Field3 */
int sip_iterate(sip_ctx* ctx, int iters);                 /* enqueue, no host sync */
int sip_read_norms(sip_ctx* ctx, int first, int count, double* norms, double* block_norms);
/* Waits for the context's stream; completes the pending sip_solve_async calls
 * (their norms_out are filled here). */
int sip_synchronize(sip_ctx* ctx);

/*
 * Pipelined solves (single rank).  A caller that knows the next step's source
 * can upload it while the current solve runs, and keep two solves in flight:
 *   sip_set_source_async(q_0); sip_solve_async(phi, iters, norms_0);
 *   for each step i:
 *     if (i + 1 < steps) { sip_set_source_async(q_{i+1});
 *                          sip_solve_async(phi, iters, norms_{i+1}); }
 *     sip_wait_async();      (step i complete: phi written, norms_i filled)
 * sip_set_source_async copies q (pinned host memory for overlap) on a copy
 * stream into one of two staging buffers per block and applies it on the
 * context's stream after the work already enqueued there.  sip_solve_async
 * is sip_solve with a fixed iteration count and no host synchronisation; at
 * most two are pending.  When its phi buffers are the ones the previous
 * pending solve writes its result into, the upload of phi0 follows that
 * download chunk by chunk (both directions of the link at once).  Results are
 * those of the sequential calls.  sip_wait_async completes the oldest pending
 * solve, sip_synchronize all of them.
 */
int sip_set_source_async(sip_ctx* ctx, int local, const double* q);
int sip_solve_async(sip_ctx* ctx, double* const* phi, int iters, double* norms_out);
int sip_wait_async(sip_ctx* ctx);

/* Flag (symmetric = 1) or unflag the system of local block `local` as
 * symmetric (StencilSystem invariant: ae(i) = aw(i+1),
 * an(j) = as(j+1), at(k) = ab(k+1), checked exactly on the device;
 * SIP_ERR_CONFIG if violated).  sip_set_system clears the flag. */
int sip_set_symmetric(sip_ctx* ctx, int local, int symmetric);

/* residual_general / residual_symmetric of the current
 * device phi into res[local] (Field3 host arrays, interior written).
 * symmetric = 1 reads only AE/AN/AT (+ shifted), AP, Q (Listing 1) and
 * requires every local system to be flagged (SIP_ERR_MISUSE otherwise,
 * SPEC.md:165). */
int sip_residual(sip_ctx* ctx, int symmetric, double* const* res);

/* ---- FTT1 transfer tables (proj/include/bsfv/tables.hpp:62-71)
 * Entry rows are int[12]: dir (0 local, 1 send, 2 recv), kind (0 face,
 * 1 edge, 2 corner), face (E W N S T B = 0..5), peer rank, owner block,
 * neighbor block, ilo, ihi, jlo, jhi, klo, khi; the ranks' tables are
 * concatenated, counts[r] entries for rank r.
 * sip_ftt1_read parses an in-memory image (tables.cpp:140-183): pass NULL
 * counts/entries to query *nranks / *total first.  SIP_ERR_FORMAT with the
 * reference's message (sip_last_error(NULL)) and *err_offset on a defect.
 * sip_ftt1_write produces the image (buf NULL: size query into *len).
 * sip_ftt1_validate checks send/recv matching (tables.cpp:185-235):
 * SIP_ERR_PROTOCOL with the reference's message. */
int sip_ftt1_read(const void* buf, size_t len, int* nranks, int* counts, int* entries,
                  long long cap_entries, long long* total, long long* err_offset);
int sip_ftt1_write(int nranks, const int* counts, const int* entries, void* buf, size_t cap,
                   size_t* len);
int sip_ftt1_validate(int nranks, const int* counts, const int* entries);

/* Replace the context's face-halo plan by the face entries of this rank's
 * table (arbitrary decompositions and periodic wraps, transfers.cpp:15-25):
 * local entries become device face copies, send/recv entries the per-peer
 * NCCL pack/unpack lists in table order.  The tables are validated first
 * (SIP_ERR_PROTOCOL); face entries must cover whole block faces of this
 * context's lattice (SIP_ERR_CONFIG otherwise).  Edge / corner entries are
 * ignored: the 7-point stencil reads face ghosts only. */
int sip_set_halo_tables(sip_ctx* ctx, int nranks, const int* counts, const int* entries);

/* Run on a caller-provided cudaStream_t (NULL: the context's own stream).
 * Work already enqueued on the previous stream stays ordered before anything
 * enqueued afterwards (the new stream waits on an event of the old one). */
int sip_set_stream(sip_ctx* ctx, void* stream);
void* sip_get_stream(const sip_ctx* ctx);

/* Per-kernel CUDA-event timing of subsequent sip_iterate calls (0 = off).
 * Totals over the iterations since enabling: forward (K2), backward (K3),
 * halo (K4) in ms, and the number of kernel launches enqueued. */
int sip_set_profiling(sip_ctx* ctx, int on);
int sip_get_profile(sip_ctx* ctx, double* fwd_ms, double* bwd_ms, double* halo_ms,
                    long long* launches);
/* Total kernel launches enqueued by this context so far. */
long long sip_launch_count(const sip_ctx* ctx);
/* Brick geometry of the wavefront kernels: brick extents along i and j
 * (kW, kL), number of bricks, slices of the forward / backward packs. */
int sip_geometry(const sip_ctx* ctx, int* ti, int* tj, long long* tiles, long long* slices);
/* Factorisation counter: K1 launches of this context so far. */
long long sip_factor_count(const sip_ctx* ctx);
/* Blocks of the whole lattice (all ranks): sizes sip_read_norms' block_norms. */
int sip_num_global_blocks(const sip_ctx* ctx, int* n);

/* ---- debugging / test helpers (not part of the reference interface) ---- */
/* One forward sweep (K2) on the current device phi (writes R). */
int sip_debug_forward(sip_ctx* ctx);
/* Gather a device pack of one local block into a Field3 array: which = 0 phi,
 * 1 R, 2..13 forward pack (AP,AW,AE,AS,AN,AB,AT,Q,LB,LW,LS,LP), 14..16 UN,UE,UT. */
int sip_debug_field(sip_ctx* ctx, int local, int which, double* out);

/* ---- host-only helpers (no device needed) ---- */
/* 128-byte ncclUniqueId for sip_create_lattice (rank 0 creates, all share). */
int sip_nccl_unique_id(void* out128);
/* Host copy of the synthetic generator (Field3 arrays of one block). */
int sip_generate_host(int kind, uint64_t seed, const int g[3], const int o[3], int nx, int ny,
                      int nz, double* ap, double* aw, double* ae, double* as, double* an,
                      double* ab, double* at, double* q);
/* Compact block -> rank map: each rank gets a near-cubic sub-lattice of the
 * px*py*pz block lattice (replaces with_ranks' slabs, grid.cpp:91-102). */
int sip_plan_block_ranks(int px, int py, int pz, int nranks, int* block_rank);
/* Face-halo plan of one rank (faces only; the 7-point stencil reads no edge or
 * corner ghosts).  Each entry is 12 ints in the field order of
 * the reference's TransferEntry / FTT1 record (tables.hpp:18-28,55-59):
 *   dir (0 local, 1 send, 2 recv), kind (0 = face), face (E,W,N,S,T,B = 0..5),
 *   peer rank, owner block, neighbor block, ilo, ihi, jlo, jhi, klo, khi
 * in the canonical order of transfers.cpp:148-165 restricted to faces.
 * block_rank NULL = one block per rank (decompose()).  *n_entries is the
 * capacity on input (entries may be NULL to query the count). */
int sip_plan_halo(int gnx, int gny, int gnz, int px, int py, int pz, const int* block_rank,
                  int rank, int* n_entries, int* entries /* [n][12] */);

/* Same with periodic wraps: bit a of periodic_mask makes axis a (x, y, z)
 * periodic (GridSpec bc, transfers.cpp:15-25); px = 1 wraps a block onto itself. */
int sip_plan_halo_periodic(int gnx, int gny, int gnz, int px, int py, int pz,
                           const int* block_rank, int rank, int periodic_mask, int* n_entries,
                           int* entries /* [n][12] */);

/* ---- the caller: pressure correction with factor reuse ----
 * Boundary kinds per domain face, order W,E,S,N,B,T (GridSpec bc). */
#define SIP_BC_WALL 0
#define SIP_BC_PERIODIC 1
#define SIP_BC_SYMMETRY 2

/*
 * assemble_poisson: the 7-point Laplacian of the pressure
 * correction on the context's lattice, domain lengths len[3] (cell sizes
 * h = len / global cells), boundary kinds bc[6].  Coefficients a_nb = face
 * area / distance (uniform cubes of size h: a_nb = h, AP = 6h), zero through a
 * wall or symmetry face (homogeneous Neumann, AP reduced accordingly),
 * coupled across periodic faces; Q = 0.  The system is singular (pure
 * Neumann / periodic), so global cell (0,0,0) is pinned as an identity row
 * (AP = 1, A_nb = 0, Q = 0).  Periodic axes install the wrapped
 * face-halo plan (sip_plan_halo_periodic).  Bumps the system revision: call
 * sip_factor once; sip_pressure_correct then reuses the factors for every
 * step (factorization counter = 1).  Periodic faces must come in
 * opposite pairs (SIP_ERR_CONFIG otherwise).
 */
int sip_assemble_poisson(sip_ctx* ctx, const double len[3], const int bc[6]);

/* FlowState: u, v, w, p as fp64 Field3 arrays per local
 * block, resident on the context's device. */
typedef struct sip_flow sip_flow;
#define SIP_FLOW_U 0
#define SIP_FLOW_V 1
#define SIP_FLOW_W 2
#define SIP_FLOW_P 3
int sip_flow_create(sip_ctx* ctx, sip_flow** out);  /* after sip_assemble_poisson */
/* Destroy every flow of a context before sip_destroy(ctx); a later
 * sip_assemble_poisson (new halo plan) also requires a new flow. */
int sip_flow_destroy(sip_flow* flow);
/* Host Field3 arrays (one per local block, interior used) -> device field. */
int sip_flow_set(sip_flow* flow, int field, double* const* per_block);
/* Device field -> host Field3 arrays (interior + face ghosts of the last update). */
int sip_flow_get(sip_flow* flow, int field, double* const* per_block);
/* Discrete divergence L1 = sum over cells of |div u| * cell volume (all ranks). */
int sip_flow_divergence(sip_flow* flow, double* l1);
/*
 * pressure_correct: outer loop of
 *   check  d = L1(div u); stop when d <= threshold
 *   su     Q = -(V * div u) / dt        (pinned cell: 0)
 *   solve  p' = 0, `sweeps` SIP iterations on the factored system (no refactor)
 *   update u -= dt * dp'/dx, v -= dt * dp'/dy, w -= dt * dp'/dz, p += p'
 * with co-located central differences and face ghosts from the
 * halo plan (walls: u_n ghost = -u_n, p' ghost = p').  *outer_used = solves
 * run; div_hist[0..outer_used] = L1 before each check (capacity max_outer+1,
 * may be NULL).  Returns SIP_ERR_NOCONV with the last defect in div_hist when
 * max_outer solves leave it above threshold.
 */
int sip_pressure_correct(sip_flow* flow, double dt, double threshold, int max_outer, int sweeps,
                         int* outer_used, double* div_hist);

#ifdef __cplusplus
}
#endif
#endif /* SIP_C_H_ */
