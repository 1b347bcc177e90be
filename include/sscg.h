/*
 * sscg.h -- C ABI of the B200-native Chebyshev-basis s-step PCG with
 * nu-sweep Forward Gauss-Seidel (FGS) Gram solves.
 *
 * Method: Thomas & D'Ambra, "Inexact Gauss-Seidel Coarse Solvers for AMG and
 * s-step CG", arxiv 2512.09642.  One outer iteration k computes
 *   1. the Chebyshev basis P = [p_0..p_{s-1}] of K_s(M^{-1}A, r_k)
 *        p_0 = r_k, p_1 = theta (M^{-1}A - sigma I) p_0,
 *        p_{j+1} = 2 theta (M^{-1}A - sigma I) p_j - p_{j-1}
 *      with theta = 2/(lmax-lmin), sigma = (lmax+lmin)/2,
 *      together with W = A P (the default schedule stores only w_{s-1}: the
 *      Gram pass and the update recover every other w_j per point from the
 *      recurrence, R21/R23);
 *   2. Ghat = P^T A P and c = P^T r_k in one pass, summed over all ranks with
 *      exactly one allreduce of the s x (s+1) block;
 *   3. the Ruhe scaling d_i = Ghat_ii^{-1/2}, G = S Ghat S = I + L + L^T,
 *      c~ = S c, and nu FGS sweeps (I + L) a^(l+1) = c~ - L^T a^(l), a^(0) = 0
 *                                                          (PAPER.md:47-55);
 *   4. alpha = S a~;  x += P alpha;  r -= W alpha.
 * Restart form, recurrence residual, stopping test ||r_k|| <= rtol ||r_0|| with
 * ||r_k||^2 = c_0 taken from the Gram block (readings R3-R5).
 *
 * Data decomposition: the nx*ny*nz grid is split in z into
 * nranks*slabs_per_rank slabs (sscg_partition); each process owns a
 * contiguous run of slabs_per_rank slabs.  Halo planes move by NCCL
 * send/recv between processes and by device copies between the slabs of one
 * process; the Gram block is reduced over local slabs in a fixed order and
 * then by one ncclAllReduce.
 *
 * Conventions
 *  - All double* / int* arguments documented "device" are CUDA device
 *    pointers valid on the calling process's current device; "host" pointers
 *    are ordinary host memory.
 *  - Grid functions (b, x, diag_M, face coefficients) are process-local,
 *    dense, x fastest: index (x, y, zl) -> x + nx*(y + ny*zl), zl in
 *    [0, nz_proc).  CSR vectors are indexed by row.
 *  - Ownership: the caller owns b, x, diag_M and all operator arrays and keeps
 *    them valid for the lifetime of the context; the library never frees
 *    them.  The library owns its workspace (basis, Gram buffers, history,
 *    NCCL communicator) and releases it in sscg_destroy.
 *  - Every call returns an sscg_status; on failure sscg_last_error() returns
 *    a thread-local message.  No exception or abort crosses the ABI.
 *  - A context is not re-entrant; use one per process and device.
 */
#ifndef SSCG_H
#define SSCG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SSCG_API __attribute__((visibility("default")))
#else
#define SSCG_API
#endif

typedef struct sscg_ctx sscg_ctx;

typedef enum {
    SSCG_OK = 0,
    SSCG_ERR_INVALID = 1,      /* argument out of range / inconsistent sizes        */
    SSCG_ERR_CUDA = 2,         /* a CUDA runtime call failed (incl. no device)      */
    SSCG_ERR_NCCL = 3,         /* an NCCL call failed                               */
    SSCG_ERR_OOM = 4,          /* device allocation failed                          */
    SSCG_ERR_BREAKDOWN = 5,    /* some Ghat_ii <= 0 or non-finite (R19); x = best so far */
    SSCG_ERR_NONFINITE = 6,    /* ||r_k|| became NaN/Inf                            */
    SSCG_ERR_UNSUPPORTED = 7   /* valid request this build does not implement       */
} sscg_status;

typedef enum {
    SSCG_OP_STENCIL5_2D = 0,   /* 2D 5-point: 4 / -1, nz must be 1 (BASELINE cfg 1) */
    SSCG_OP_STENCIL7 = 1,      /* 3D 7-point: 6 / -1 (cfg 2, 5)                     */
    SSCG_OP_STENCIL27 = 2,     /* 3D 27-point: 26 / -1 for all 26 neighbours (cfg 3) */
    SSCG_OP_VARCOEF7 = 3,      /* 3D variable-coefficient 7-point FV (cfg 4; R12)   */
    SSCG_OP_CSR = 4            /* general symmetric CSR, single slab only           */
} sscg_op_kind;

/* Operator A ("sparse SPD A"; stencils of PAPER.md:308 and the
 * BASELINE configs).  Homogeneous Dirichlet: values outside the global grid
 * are zero.  For VARCOEF7, the face arrays cover this process's planes
 * [z0, z0+nz_proc) (device, row-major):
 *   kx[(zl*ny + y)*(nx+1) + f]   face between x=f-1 and x=f, f in [0, nx]
 *   ky[(zl*(ny+1) + f)*nx + x]   face between y=f-1 and y=f, f in [0, ny]
 *   kz[(fl*ny + y)*nx + x]       face between global planes z0+fl-1 and z0+fl,
 *                                fl in [0, nz_proc]
 * A_ii = sum of the six faces of cell i, A_i,nbr = -k_face.
 * For CSR: n rows, int64 rowptr[n+1], int32 colind[nnz], double val[nnz]
 * (device), both triangles stored. */
typedef struct {
    int32_t kind;              /* sscg_op_kind                                      */
    int64_t nx, ny, nz;        /* GLOBAL interior grid; nz = 1 for STENCIL5_2D      */
    const double *kx, *ky, *kz;/* VARCOEF7 faces (device), else NULL                */
    int64_t n;                 /* CSR rows, else 0                                  */
    const int64_t *rowptr;     /* CSR (device)                                      */
    const int32_t *colind;     /* CSR (device)                                      */
    const double *val;         /* CSR (device)                                      */
} sscg_operator;

/* Process group.  nranks == 1 needs no NCCL.  For nranks > 1, every rank
 * passes the same 128-byte ncclUniqueId (host) obtained by rank 0 with
 * sscg_nccl_unique_id and broadcast by the caller (e.g. torch.distributed).
 * slabs_per_rank > 1 splits this process's planes further into that many
 * slabs on the same GPU (in-process halo copies; used to test the
 * decomposition on one device). */
typedef struct {
    int32_t rank, nranks;
    int32_t slabs_per_rank;    /* >= 1                                              */
    const void *nccl_id;       /* host, 128 bytes; ignored when nranks == 1         */
} sscg_comm;

/* Planes [z0, z0+nzl) owned by process `rank` when nz planes are split into
 * nranks*slabs_per_rank slabs, slab g = [floor(g nz/S), floor((g+1) nz/S)).
 * Pure host arithmetic; needs no GPU.  Returns SSCG_ERR_INVALID if some slab
 * would be empty. */
SSCG_API sscg_status sscg_partition(int64_t nz, int32_t nranks, int32_t slabs_per_rank, int32_t rank,
                           int64_t *z0, int64_t *nzl);

/* Halo plan of local slab `slab` (0..slabs_per_rank-1) of process `rank`:
 * out[6] = {peer_lo, send_lo_z, recv_lo_z, peer_hi, send_hi_z, recv_hi_z}
 * where peer_* is the process that owns the neighbouring slab (-1 at the
 * global Dirichlet boundary; == rank for an in-process neighbour) and *_z
 * are GLOBAL plane indices: the interior plane sent to that neighbour and
 * the plane received into the halo.  One plane per side per basis step
 * (7/27-point stencils reach one plane).  Pure host arithmetic. */
SSCG_API sscg_status sscg_halo_plan(int64_t nz, int32_t nranks, int32_t slabs_per_rank, int32_t rank,
                                    int32_t slab, int64_t *out6);

/* Fill `out` (host, 128 bytes) with a fresh ncclUniqueId.  Needs no GPU. */
SSCG_API sscg_status sscg_nccl_unique_id(void *out);

/* Create a solver context (PAPER.md:33-55 fixes theta, sigma, s, nu).
 *   A          operator (arrays device, see sscg_operator)
 *   diag_M     device, process-local grid function: the Jacobi diagonal M;
 *              NULL => M = diag(A) (BASELINE configs).  Copied at setup.
 *   lambda_min, lambda_max  bounds of the spectrum of M^{-1}A, 0 < lmin < lmax
 *              (PAPER.md:34); theta = 2/(lmax-lmin), sigma = (lmax+lmin)/2.
 *   s          basis size, 1 <= s <= 64;   nu  FGS sweeps, nu >= 1.
 *   comm       NULL => single process, one slab.
 *   stream     cudaStream_t to run on (NULL => the library creates one).
 * Allocates the basis P and W = AP (2 s vectors with one halo plane each
 * side), Gram partials and history; zeroes the global-boundary halos.
 * Errors: SSCG_ERR_INVALID for out-of-range arguments (incl. a slab with no
 * planes, STENCIL5_2D with nz != 1, CSR with more than one slab),
 * SSCG_ERR_OOM, SSCG_ERR_CUDA, SSCG_ERR_NCCL.  *out is NULL on failure. */
SSCG_API sscg_status sscg_setup(const sscg_operator *A, const double *diag_M, double lambda_min,
                       double lambda_max, int32_t s, int32_t nu, const sscg_comm *comm,
                       void *stream, sscg_ctx **out);

#define SSCG_SOLVE_X0_ZERO 1u  /* flag: treat x as 0 on entry (r_0 = b, no SpMV)   */

/* Solve A x = b by restart s-step CG until
 * ||r_k|| <= rtol ||r_0|| or max_outer updates.  b, x: device, process-local.
 * x holds x_0 on entry (ignored with SSCG_SOLVE_X0_ZERO) and x_k on return.
 * Synchronous on return.  rtol = 0 runs exactly max_outer outer iterations.
 * Non-convergence is not an error (SSCG_OK, stats.converged = 0).
 * Breakdown returns SSCG_ERR_BREAKDOWN with the last good x. */
SSCG_API sscg_status sscg_solve(sscg_ctx *ctx, const double *b, double *x, double rtol, int32_t max_outer,
                       uint32_t flags);

/* Same as sscg_solve with HOST b and x (process-local, pageable or pinned):
 * b is copied to the device, x is copied in (unless X0_ZERO) and back out.
 * The copies are part of the call (end-to-end path).  With a page-locked
 * x_host (cudaMallocHost / cudaHostRegister) the copy of x out overlaps the
 * last outer iteration (the one that only evaluates the stopping test); a
 * pageable x_host is copied after the solve completes. */
SSCG_API sscg_status sscg_solve_host(sscg_ctx *ctx, const double *b_host, double *x_host, double rtol,
                            int32_t max_outer, uint32_t flags);

/* Run exactly `nsteps` further outer iterations (basis, Gram + allreduce,
 * FGS, update: every step of PAPER.md:31/33-55) from the state the last
 * sscg_solve left (r_k inside the context, x_k in `x`), with the stopping
 * test disabled and no host round trip between iterations.  x: device, the
 * vector the last sscg_solve returned.  Used to time a fixed number of outer
 * iterations (BASELINE cfg 3-5).  SSCG_ERR_INVALID if no solve preceded. */
SSCG_API sscg_status sscg_iterate(sscg_ctx *ctx, double *x, int32_t nsteps);

/* Per-kernel device time: with profiling on, every launch group is bracketed
 * by CUDA events on the solver stream and accumulated per category.  When the
 * schedule runs fused basis kernels (K1M triples / K1F pairs), SSCG_PROF_BASIS
 * counts those and SSCG_PROF_BASIS_SINGLE the single basis steps around them
 * (the last step j = s-1, boundary planes); otherwise every basis launch is
 * SSCG_PROF_BASIS. */
enum { SSCG_PROF_BASIS = 0, SSCG_PROF_GRAM = 1, SSCG_PROF_ALLREDUCE = 2, SSCG_PROF_FGS = 3,
       SSCG_PROF_UPDATE = 4, SSCG_PROF_HALO = 5, SSCG_PROF_BASIS_SINGLE = 6, SSCG_PROF_N = 7 };
typedef struct {
    double ms[SSCG_PROF_N];          /* accumulated device milliseconds           */
    int64_t launches[SSCG_PROF_N];   /* events pairs (= launches, or NCCL groups)  */
} sscg_profile_t;
SSCG_API sscg_status sscg_set_profiling(sscg_ctx *ctx, int32_t on);   /* also resets */
SSCG_API sscg_status sscg_profile(sscg_ctx *ctx, sscg_profile_t *out); /* synchronises */

typedef struct {
    int32_t outer_iterations;  /* updates applied                                   */
    int32_t converged;         /* ||r_k|| <= rtol ||r_0|| reached                    */
    int32_t breakdown;         /* Ghat_ii <= 0 or non-finite                         */
    int32_t nonfinite;         /* ||r_k|| not finite                                 */
    double r0_norm;            /* ||r_0||_2                                          */
    double relres_final;       /* ||r_k|| / ||r_0|| at exit (recurrence residual)    */
    int32_t history_len;       /* entries in relres_history (outer_iterations + 1)  */
    const double *relres_history; /* host, owned by ctx, valid until next solve     */
    const double *delta_history;  /* host: ||c~ - G a~||/||c~|| per update */
    double ms_total;           /* device time of the last solve (CUDA events)        */
    int64_t kernel_launches;   /* library kernels launched by the last solve        */
    int64_t allreduces;        /* NCCL allreduces issued by the last solve          */
    double budget;             /* with SSCG_OPT_DIAGNOSTICS: sum_k delta_k ||A|| ||P_k||_F
                                  (PAPER.md:259-266 Thm Inexact Convergence), else 0 */
} sscg_stats_t;

SSCG_API sscg_status sscg_stats(const sscg_ctx *ctx, sscg_stats_t *out);

/* Parity hooks: copy internal state of the LAST solve to host memory.
 *   SSCG_INSPECT_P, _W     column `index` of P / W = AP of the last basis built
 *                          (process-local grid layout, nx*ny*nz_proc doubles)
 *   SSCG_INSPECT_GRAM      outer `index`: [Ghat (s*s, row-major, mirrored) | c (s)]
 *                          after the allreduce
 *   SSCG_INSPECT_D, _ALPHA_T, _ALPHA   outer `index`: s doubles
 *   SSCG_INSPECT_DELTA     outer `index`: 1 double (||c~ - G a~|| / ||c~||)
 *   SSCG_INSPECT_LNORM     outer `index`: 1 double (||L||_F of the scaled Gram matrix)
 * `capacity` is the byte size of host_out; too small => SSCG_ERR_INVALID.
 * History entries exist for outer indices 0..max_outer of the last solve
 * (GRAM, D, ALPHA_T, ALPHA: the first 2048 outer iterations only). */
enum {
    SSCG_INSPECT_P = 0, SSCG_INSPECT_W = 1, SSCG_INSPECT_GRAM = 2, SSCG_INSPECT_D = 3,
    SSCG_INSPECT_ALPHA_T = 4, SSCG_INSPECT_ALPHA = 5, SSCG_INSPECT_DELTA = 6,
    SSCG_INSPECT_LNORM = 7,    /* outer `index`: ||L||_F of G = I + L + L^T, 1 double */
    SSCG_INSPECT_KAPPA = 8,    /* outer `index`: kappa(G) (with SSCG_OPT_DIAGNOSTICS, else 0), 1 double */
    SSCG_INSPECT_PNORM = 9,    /* outer `index`: ||P_k||_F (diagnostics), 1 double */
    SSCG_INSPECT_BUDGET = 10   /* outer `index`: delta_k ||A|| ||P_k||_F, ||A|| the Gershgorin bound (diagnostics) */
};
SSCG_API sscg_status sscg_inspect(const sscg_ctx *ctx, int32_t what, int32_t index, void *host_out,
                         int64_t capacity);

/* Process-local sizes: planes [z0, z0+nz_proc) (CSR: n rows, z0 = 0). */
SSCG_API sscg_status sscg_local_shape(const sscg_ctx *ctx, int64_t *z0, int64_t *nz_proc, int64_t *n_local);

/* Replace the spectral bounds of M^{-1}A (0 < lmin < lmax):
 * theta = 2/(lmax-lmin), sigma = (lmax+lmin)/2 for later
 * solves.  A context created with lambda_min = lambda_max = 0 has no bounds;
 * sscg_solve with the Chebyshev basis then returns SSCG_ERR_INVALID until
 * this is called (e.g. with the result of sscg_estimate_bounds).
 * Errors: SSCG_ERR_INVALID. */
SSCG_API sscg_status sscg_set_bounds(sscg_ctx *ctx, double lambda_min, double lambda_max);

/* Spectral bounds of M^{-1}A by `iters` Lanczos steps (
 * PAPER.md:311 "Lanczos ... with a safety margin"; BASELINE cfg 3/4 use 50
 * steps and margin 0.05) on D^{-1/2} A D^{-1/2} (D = M, the Jacobi diagonal
 * of the context) from v0/||v0||, without reorthogonalisation; the extreme
 * Ritz values are widened to lmin (1 - margin), lmax (1 + margin).
 *   v0         device, process-local grid function (layout as b), not all 0
 *   iters      1..100000;  margin in [0, 1)
 *   lmin, lmax host outputs;  alpha_out, beta_out: optional host arrays of
 *              `iters` doubles receiving the tridiagonal (a_k, b_k); entries
 *              past an early stop (b_k = 0) are 0.
 * Runs on the context's stream with two reductions per step (one NCCL
 * allreduce each for nranks > 1); synchronous on return.  Uses its own
 * workspace (3 vectors + D + w per slab, allocated on first use): the basis
 * and the state of the last solve are untouched.
 * Errors: SSCG_ERR_INVALID, SSCG_ERR_CUDA, SSCG_ERR_NCCL, SSCG_ERR_OOM,
 * SSCG_ERR_BREAKDOWN if the Ritz interval is not positive. */
SSCG_API sscg_status sscg_estimate_bounds(sscg_ctx *ctx, const double *v0, int32_t iters, double margin,
                                          double *lmin, double *lmax, double *alpha_out, double *beta_out);

/* Variants on the same boundary, for later solves:
 *   SSCG_OPT_GRAM_SOLVER  SSCG_GRAM_FGS (default): nu Forward Gauss-Seidel
 *                         sweeps;  SSCG_GRAM_CHOLESKY: the
 *                         exact O(s^3) solve by dense Cholesky of the scaled
 *                         Gram matrix; a non-positive pivot
 *                         is reported as SSCG_ERR_BREAKDOWN.
 *   SSCG_OPT_BASIS        SSCG_BASIS_CHEBYSHEV (default) or
 *                         SSCG_BASIS_MONOMIAL p_{j+1} = M^{-1}A p_j
 *                         (kappa(G) grows like
 *                         kappa(M^{-1}A)^{s-1}, so only small s is usable).
 *   SSCG_OPT_DIAGNOSTICS  0 (default) / 1: after every update also compute
 *                         kappa(G) of the scaled Gram matrix (one-warp Jacobi
 *                         eigensolver), ||P_k||_F (one extra pass over P) and
 *                         the budget term delta_k ||A|| ||P_k||_F of
 *                         PAPER.md:259-266 (||A||: Gershgorin bound, computed
 *                         once), read back with SSCG_INSPECT_KAPPA / _PNORM /
 *                         _BUDGET and stats.budget.  Off the hot path.
 *   SSCG_OPT_BLOCKCG      0 (default): the restart form x += P~ alpha
 *                         (PAPER.md:31);  1: block-conjugate s-step CG
 *                         (R24): each outer block
 *                         Q_k = P_k - Q_{k-1} B_k is made A-conjugate to the
 *                         previous one, B_k = G_{k-1}^{-1} (A Q_{k-1})^T P_k;
 *                         the cross-block entries come from the same single
 *                         Gram pass and allreduce (over the 2s vectors
 *                         [P_k | Q_{k-1}]), K4 solves Q_k^T A Q_k a =
 *                         Q_k^T r_k with the selected Gram solver (pair it
 *                         with SSCG_GRAM_CHOLESKY: inexact FGS solves break
 *                         the conjugacy), and the update is x += Q_k alpha,
 *                         r -= A Q_k alpha.  Needs s <= 32; twice the basis
 *                         storage (reallocated here; the next solve starts a
 *                         new block sequence); W_k = A P_k is recovered from
 *                         the basis recurrence (not stored) for the 7- and
 *                         27-point stencils with a constant diagonal and
 *                         s <= 16, A Q_{k-1} is kept (stored-W schedule
 *                         otherwise).  With nranks > 1 every rank sets it
 *                         (the reallocation re-maps the neighbours' basis
 *                         for the peer-store halos: NCCL calls with them).
 *                         SSCG_INSPECT_GRAM then returns [G_k | c_k] of the
 *                         conjugated system.
 * Errors: SSCG_ERR_INVALID for an unknown key or value. */
enum { SSCG_OPT_GRAM_SOLVER = 0, SSCG_OPT_BASIS = 1, SSCG_OPT_DIAGNOSTICS = 2, SSCG_OPT_BLOCKCG = 3 };
enum { SSCG_GRAM_FGS = 0, SSCG_GRAM_CHOLESKY = 1 };
enum { SSCG_BASIS_CHEBYSHEV = 0, SSCG_BASIS_MONOMIAL = 1 };
SSCG_API sscg_status sscg_set_option(sscg_ctx *ctx, int32_t key, int32_t value);

/* Introspection of the schedule the context runs (host, no GPU work):
 *   SSCG_QUERY_BASIS_FUSED    basis steps per launch of the schedule's main
 *                             basis kernel: 3 (K1M triples, p_{j+1}, p_{j+2}
 *                             kept on chip; one 7-point slab), 2 (K1F pairs),
 *                             1 (single steps)
 *   SSCG_QUERY_BASIS_VECTORS  FP64 vectors of n_local the basis kernels read
 *                             and write per outer iteration (algorithmic;
 *                             variable-coefficient face arrays not included)
 *   SSCG_QUERY_UPDATE_VECTORS FP64 vectors the update kernel moves per outer
 *                             iteration: 2s+3 (r -= W alpha from the stored
 *                             W), or s+4 when W alpha is formed from the
 *                             Chebyshev recurrence (R21; s+5 when
 *                             the Jacobi diagonal varies and is read too)
 *   SSCG_QUERY_GRAM_VECTORS   FP64 vectors the Gram pass reads per outer
 *                             iteration: 2s (P and the stored W = AP), or s+1
 *                             (+1 for a varying diagonal) when W is recovered
 *                             from the basis recurrence (R23);
 *                             4s in the block-conjugate mode
 *   SSCG_QUERY_BASIS_SINGLE_VECTORS  the part of BASIS_VECTORS moved by the
 *                             single steps of a fused schedule (0 without)
 *   SSCG_QUERY_PEER_HALO      how the deep-halo triples reach their neighbours'
 *                             ghost planes: 0 exchange (NCCL
 *                             send/recv or device copies after each triple),
 *                             1 peer stores into in-process slabs, 2 peer
 *                             stores into basis vectors mapped at setup (other
 *                             ranks' through CUDA IPC; SSCG_NCCL_SELF: the
 *                             in-process slabs after the same NCCL round trip),
 *                             ordered by a one-double token per triple
 * Errors: SSCG_ERR_INVALID. */
enum { SSCG_QUERY_BASIS_FUSED = 0, SSCG_QUERY_BASIS_VECTORS = 1, SSCG_QUERY_UPDATE_VECTORS = 2,
       SSCG_QUERY_GRAM_VECTORS = 3, SSCG_QUERY_BASIS_SINGLE_VECTORS = 4, SSCG_QUERY_PEER_HALO = 5 };
SSCG_API sscg_status sscg_query(const sscg_ctx *ctx, int32_t what, int64_t *out);

SSCG_API void sscg_destroy(sscg_ctx *ctx);

/* ------------------------------------------------------------------------
 * AMG coarse-grid Forward Gauss-Seidel (§6 "AMG Coarse-Grid
 * Extension": FGS on A_c = P^T A_f P, "implemented in a streaming
 * (matrix-free) fashion to avoid forming A_c explicitly"
 * §8: nu_coarse = 20 at the coarsest level, n_c ~ 5000; R25).
 *
 * One coarse level of unsmoothed aggregation: P is piecewise constant on
 * bx x by x bz blocks of fine cells (the last block of an axis may be
 * partial); coarse point (I, J, K), I < ncx = ceil(nx/bx) etc., has index
 * I + ncx (J + ncy K) and aggregates fine cells x in [bx I, min(bx I + bx, nx)),
 * likewise y, z.  A_f: SSCG_OP_STENCIL5_2D (bz must be 1), SSCG_OP_STENCIL7
 * or SSCG_OP_VARCOEF7 on one process (z0 = 0, nz_proc = nz; face arrays as
 * for sscg_setup, device, owned by the caller and kept valid for the
 * handle's lifetime).  Their A_c couples only face-adjacent aggregates.
 *
 * Modes:
 *   SSCG_COARSE_STREAMING  A_c is never stored: every visit of a coarse row
 *                          recomputes its (at most 7) entries from the fine
 *                          operator -- entry (I, J) is the sum over the cells
 *                          a of aggregate I of (A_f p_J)_a, p_J = P e_J.
 *   SSCG_COARSE_ASSEMBLED  the entries are formed once at create (7 n_c
 *                          doubles padded to 8 per row, the same arithmetic)
 *                          and read by FGS.
 * For the 5- and 7-point operators the streaming entries are integers (face
 * areas, 4 / 6 x cells - 2 x internal couplings) formed in closed form --
 * exact, hence the same doubles as any summation order.
 * Both give results bitwise equal to the definition written out in the
 * oracle (entry sums in ascending fine index, Gauss-Seidel row sums in
 * ascending coarse index, no fused multiply-add).
 *
 * Calls are asynchronous on `stream` (a cudaStream_t; NULL = the legacy
 * default stream); vectors are device pointers.  The FGS kernel keeps r_c and
 * y in one CTA's shared memory: n_c <= SSCG_COARSE_MAX_N.
 * Errors: SSCG_ERR_INVALID (null pointers, b < 1, nu < 0, bz != 1 for the 2D
 * operator), SSCG_ERR_UNSUPPORTED (other operator kinds, n_c too large),
 * SSCG_ERR_CUDA / SSCG_ERR_OOM.
 * ------------------------------------------------------------------------ */
typedef struct sscg_coarse sscg_coarse;
enum { SSCG_COARSE_STREAMING = 0, SSCG_COARSE_ASSEMBLED = 1 };
#define SSCG_COARSE_MAX_N 11000
SSCG_API sscg_status sscg_coarse_create(const sscg_operator *A_f, int32_t bx, int32_t by, int32_t bz, int32_t mode,
                                        sscg_coarse **out);
/* r_c = P^T r_f (n_f -> n_c; each aggregate summed in ascending fine index) */
SSCG_API sscg_status sscg_coarse_restrict(sscg_coarse *h, const double *r_f, double *r_c, void *stream);
/* x_f += P y (n_c -> n_f) */
SSCG_API sscg_status sscg_coarse_prolong_add(sscg_coarse *h, const double *y, double *x_f, void *stream);
/* nu forward Gauss-Seidel sweeps on A_c y = r_c; y holds the initial guess on
 * entry and the result on return (nu = 10-30) */
SSCG_API sscg_status sscg_coarse_fgs(sscg_coarse *h, const double *r_c, double *y, int32_t nu, void *stream);
/* the (at most 7) entries of every coarse row, device out[7 * n_c]: out[d *
 * n_c + c] = A_c(c, neighbour d of c), d = 0..6 for the neighbours at
 * z-1, y-1, x-1, c itself, x+1, y+1, z+1 (0 where absent) -- computed by the
 * routine the assembly runs (the closed form of the constant stencils gives
 * the same integers) */
SSCG_API sscg_status sscg_coarse_entries(sscg_coarse *h, double *out, void *stream);
/*   SSCG_COARSE_QUERY_N              n_c
 *   SSCG_COARSE_QUERY_NCX / _NCY / _NCZ  the coarse grid
 *   SSCG_COARSE_QUERY_WAVEFRONTS     T = ncx + ncy + ncz - 2 wavefronts t = I + J + K;
 *                                    an FGS call of nu sweeps runs T + 2 (nu - 1)
 *                                    barrier-separated steps (sweeps pipelined)
 *   SSCG_COARSE_QUERY_MATRIX_BYTES   device bytes holding A_c (0 when streaming) */
enum { SSCG_COARSE_QUERY_N = 0, SSCG_COARSE_QUERY_NCX = 1, SSCG_COARSE_QUERY_NCY = 2, SSCG_COARSE_QUERY_NCZ = 3,
       SSCG_COARSE_QUERY_WAVEFRONTS = 4, SSCG_COARSE_QUERY_MATRIX_BYTES = 5 };
SSCG_API sscg_status sscg_coarse_query(const sscg_coarse *h, int32_t what, int64_t *out);
SSCG_API void sscg_coarse_destroy(sscg_coarse *h);

/* Thread-local description of the last error ("" if none). */
SSCG_API const char *sscg_last_error(void);

/* Library version string. */
SSCG_API const char *sscg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SSCG_H */
