// Internal declarations shared by the sm_100a kernels and the host driver of
// libsscg.  Nothing here is visible through the C ABI (include/sscg.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace sscg {

// Programmatic dependent launch (PDL).  The hot kernels are launched with the
// programmatic-stream-serialization attribute (launch_pdl), so a kernel's
// CTAs are scheduled while its predecessor in the stream (or the captured
// graph) is still running.  Each such kernel starts with PDL_ENTRY: it waits
// (griddepcontrol.wait) until the predecessor grid has completed and its
// writes are visible -- no global memory is touched before that -- then lets
// its own dependents launch, then reads the device stop flag.  The launch
// latency of every kernel boundary is hidden behind the previous kernel's
// tail.  A kernel launched without the attribute passes the wait at once.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#define PDL_ENTRY(st)                     \
    do {                                  \
        ::sscg::pdl_wait();               \
        ::sscg::pdl_trigger();            \
        if ((st) && (st)->done) return;   \
    } while (0)

template <typename... K, typename... A>
inline cudaError_t launch_pdl(bool pdl, void (*kern)(K...), dim3 grid, dim3 block, size_t smem, cudaStream_t strm,
                              A &&...args)
{
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = strm;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}

// Device-resident solver state.  K4 (FGS) is the only writer of the control
// fields; every hot kernel reads `done` first and exits if it is set, so the
// host can enqueue several outer iterations without a round trip
// (device-side stopping test).
struct DevState {
    int k;            // current outer index (basis/Gram being built)
    int done;         // 1 => stop: kernels of later outer iterations are no-ops
    int converged;
    int breakdown;
    int nonfinite;
    int outer;        // updates applied
    int hist_cap;     // scalar history slots (relres, delta, ||L||, ...)
    int gram_cap;     // per-outer vector records (Gram block, d, alpha~, alpha): min(hist_cap, 2048)
    double r0norm;    // ||r_0||
    double rtol;
    int max_outer;
    int pad2_;
};

// One z-slab of the decomposition in the workspace layout.
//   plane  = ny * pitch doubles; pitch = nx rounded up to even (16-B rows)
//   vector = (nzl + 2) planes: plane 0 = lower halo, 1..nzl interior,
//            nzl+1 = upper halo (zero at global boundaries); with deep halos
//            (Geo::guard = 2) two more ghost planes are allocated on each
//            side (planes -2, -1 and nzl+2, nzl+3), so a vector spans
//            nzl + 6 planes and its base pointer still addresses plane 0.
struct Slab {
    int64_t z0;        // first global plane
    int nzl;           // interior planes
    int has_lo, has_hi;   // a neighbour slab (this or another rank) below / above
    int64_t zoff;      // first plane relative to the process-local range
    double *P;         // s vectors, stride vstride (2s in the block-conjugate mode: [P_k | Q_{k-1}])
    double *W;         // s vectors, stride vstride (2s: [W_k | Z_{k-1} = A Q_{k-1}])
    double *Palloc, *Walloc;      // the allocations (P, W start Geo::guard planes in)
    // peer-store halos: the basis P of the neighbour below [0] /
    // above [1] that K1M stores ghost planes into -- an in-process slab, or
    // another rank's P mapped through CUDA IPC -- with its vector stride and
    // depth (null: exchange instead)
    double *nbP[2];
    int64_t nbvs[2];
    int nbnzl[2];
    int nb_remote[2];             // the neighbour is another process (K1M ends with a system-scope fence)
    bool want_k1f, want_k1m, want_k1fv;   // basis kernels whose tensor maps the store needs
    double *part;      // Gram partials [grid][nent]
    double *blk;       // this slab's reduced block (s*s + s)
    unsigned *ticket;  // last-CTA counter for K2
    const double *kx, *ky, *kz;   // VARCOEF7 faces of this slab
    const double *dinv;           // Jacobi 1/diag(M) interior layout (or nullptr)
    double *dvec;                 // diag(M) in the padded layout when it is not constant (K5 REC), else nullptr
    CUtensorMap tmP, tmW;         // K2: [s rows x interior] views of P and W
    CUtensorMap tmPd, tmWd;       // K2D (DMMA Gram, s > 16): same views, box pitch 132/68
    bool has_k2d;
    CUtensorMap tmWl, tmDv;       // K2R: the row w_{s-1} of W, diag(M) (one row)
    CUtensorMap tmPr;             // K2R: P rows, box pitch 136/72 (16-B point-pair loads)
    CUtensorMap tmPb, tmZb, tmWlb;   // K2R block mode: [P_k | Q'] rows, Z' rows, w_{s-1}
    bool has_k2r, has_k2rb;
    CUtensorMap tmP4, tmM4;       // K1T: 4-D [x][y][plane][vector] views of P (halo box / tile box)
    bool has_k1t;
    CUtensorMap tmF_P, tmF_M;     // K1F: 2-cell / 1-cell halo boxes
    CUtensorMap tmM3_P, tmM3_M;   // K1M (depth-3 basis): 3/6-cell and 2/4-cell halo boxes
    CUtensorMap tmV_KX, tmV_KY, tmV_KZ;   // K1FV: faces in the pair's boxes
    int kx_shift;                         // K1FV: the 1-D kx view starts this many elements early
    bool has_k1m;
    CUtensorMap tmKX, tmKY, tmKZ; // K1T: variable-coefficient faces (nx even)
    bool has_ftma;
    bool has_k1f;
};

// Schedule and tuning switches (DESIGN.md §1 table), read from the
// environment once per context by sscg_setup (read_knobs) and carried in Geo,
// so a context keeps the switches it was created with and two contexts of
// one process may differ (the parity tests force both sides of a choice).
struct Knobs {
    int k1_fuse = -1;      // SSCG_K1_FUSE      -1 auto, 0 forbid, 1 force (K1F pairs)
    int k1_mp3 = -1;       // SSCG_K1_MP3       same for K1M triples
    int k1_fuse_vc = -1;   // SSCG_K1_FUSE_VC   same for K1FV
    int k1_tma = 1;        // SSCG_K1_TMA       0: direct-load K1
    int k1_zc = 0;         // SSCG_K1_ZC        z-chunk length (0 auto)
    int faces_tma = 1;     // SSCG_FACES_TMA    0: direct face loads
    int k2_dmma = -1;      // SSCG_K2_DMMA      stored-W Gram on tensor cores (-1: s > 16)
    int k2s = 1;           // SSCG_K2S          0: tensor-core K2R also for s <= 8
    int k2_e = 0, k2_ns = 0, k2_grid = 0, k2_groups = 0, k2_smem_kb = 216;   // Gram-pass sweeps
    int wfree = 1;         // SSCG_WFREE        0: stored-W schedule
    int k5_recur = 1;      // SSCG_K5_RECUR     0: update with the stored W
    int deep_halo = 1;     // SSCG_DEEP_HALO    0: 1-plane halos around every K1M triple (boundary single steps)
    int deep_overlap = 0;  // SSCG_DEEP_OVERLAP 1: deep-halo exchange overlapped with the triple / update interior
    int peer_halo = 1;     // SSCG_PEER_HALO    0: in-process deep halos by copies after each triple instead of K1M peer stores
    int small = -1;        // SSCG_SMALL        -1 auto (2D grids <= 8192 points), 0 forbid, 1 force the single-cluster outer iteration
    int debug = 0;         // SSCG_DEBUG
    int pdl = 1;           // SSCG_PDL          0: plain stream-ordered launches (no programmatic dependent launch)
    int wl_fold = 1;       // SSCG_WL_FOLD      1: w_{s-1} never stored (K2R lower triangle + k_pap + K5 stencil); 2: only K5 forms it; 0: off
    int gram_space = 0;    // SSCG_GRAM_SPACE   1: the folded K2R forms E = P^T P and maps it to Ghat by the recurrence (R27: loses ~log10 kappa digits; opt-in)
    int k2_il = 1;         // SSCG_K2_IL        0: the folded two-block K2R with blocked (8J + r) instead of interleaved (2r + J) fragment rows
};
Knobs read_knobs();

struct Geo {
    Knobs kn;
    int kind;          // sscg_op_kind
    int nx, ny;        // grid in x, y
    int pitch;         // row pitch (doubles)
    int64_t plane;     // ny * pitch
    int64_t vstride;   // doubles between consecutive basis vectors
    int guard;         // ghost planes allocated beyond the 1-plane halo on each side (0, or 2 for deep halos)
    double center;     // 4, 6, 26 for constant stencils
    double dinv_c;     // 1/center
    // CSR
    int64_t n;
    const int64_t *rowptr;
    const int32_t *colind;
    const double *val;
};

// K1: fused SpMV + Jacobi + Chebyshev recurrence over planes [zb, ze)
//   mode 0: w = A p                                   (j = s-1)
//   mode 1: w = A p; pn = coef * (dinv w - sigma p)   (j = 0, coef = theta)
//   mode 2: w = A p; pn = coef * (dinv w - sigma p) - pm   (coef = 2 theta)
//   mode 3: w = b - A p (residual r_0 = b - A x_0; b in process layout)
struct K1Args {
    const double *p;
    const double *pm;
    double *w;
    double *pn;
    const double *b;       // mode 3 only (process layout, slab offset applied)
    const double *kx, *ky, *kz;
    const double *dinv;    // interior layout with pitch, or nullptr => dinv_c
    double dinv_c;
    double coef, sigma;
    int zb, ze;            // padded plane indices (1..nzl)
    int zb2, ze2;          // optional second plane range (boundary launches), empty if ze2 <= zb2
    int sm_cap;            // > 0: use at most this many SMs (leave room for NCCL kernels)
    int mode;
    int nzl;
    int j;                 // basis step (K1T: vector coordinate of p_j in the tensor maps)
    int skip_w;            // 1: w_j is not stored (the Gram pass recovers it, R23; K1T/K1F)
    int skip_w2;           // K1F: same for w_{j+1}
    const CUtensorMap *tmP4, *tmM4;   // K1T tensor maps of this slab (host memory), or nullptr
    const CUtensorMap *tmKX, *tmKY, *tmKZ;   // K1T variable-coefficient face maps, or nullptr
    double *w2, *pn2;                 // K1F: w_{j+1}, p_{j+2} (nullptr at j+1 = s-1)
    // K1T mode 0 with the w_{s-1} fold: accumulate p^T A p over the launch's own
    // cells instead of storing w (skip_w): per-CTA partials, a ticket, and the
    // entry the last CTA writes (the slab's Gram block entry (s-1, s-1)); else null
    double *dot_part, *dot_entry;
    unsigned *dot_ticket;
    int kx_shift;                     // K1FV: see Slab::kx_shift
    const CUtensorMap *tmF_P, *tmF_M; // K1F tensor maps
};

void launch_k1(const Geo &g, const K1Args &a, const DevState *st, cudaStream_t s);

// K1T: TMA-staged 7-/27-point basis step (k_stencil_tma.cu)
bool k1t_supported(const Geo &g, const K1Args &a);
bool k1t_prepare(const Geo &g, const double *P, int nzl, int s, CUtensorMap *tmP4, CUtensorMap *tmM4);
void launch_k1t(const Geo &g, const K1Args &a, const DevState *st, cudaStream_t s);
bool k1t_prepare_faces(const Geo &g, const double *kx, const double *ky, const double *kz, int nzl, CUtensorMap *mx,
                       CUtensorMap *my, CUtensorMap *mz);

// K1F: two 7-point basis steps per launch, single slab (k_stencil_fused.cu)
bool k1f_enabled(const Geo &g, int nzl);
// K1FV: the pair for variable coefficients (k_stencil_fused_vc.cu; maps in tmF_P / tmF_M)
bool k1fv_enabled(const Geo &g, int nzl);
bool k1fv_prepare(const Geo &g, const double *P, int nzl, int s, CUtensorMap *tmP, CUtensorMap *tmM);
bool k1fv_prepare_faces(const Geo &g, const double *kx, const double *ky, const double *kz, int nzl, CUtensorMap *mx,
                        CUtensorMap *my, CUtensorMap *mz, int *kx_shift);
void launch_k1fv(const Geo &g, const K1Args &a, double theta, int s, const DevState *st, cudaStream_t strm);

// K1M: three basis steps per launch (7-point, constant diagonal; k_stencil_mp3.cu)
struct K1MArgs {
    double *w[3];          // w_j, w_{j+1}, w_{j+2} (null: not stored)
    double *pn[3];         // p_{j+1}, p_{j+2}, p_{j+3} (null: not stored)
    int zb[3], ze[3];      // padded planes each level writes
    int zb2[3], ze2[3];    // optional second range (deep-halo boundary launch), empty if ze2[2] <= zb2[2]
    int nzl, j, sm_cap;
    // deep halos: a side with deep_* set has p_j current on 3
    // ghost planes and p_{j-1} on 2; levels 1 and 2 are then formed on 2 / 1
    // ghost planes there instead of taking the Dirichlet value
    int deep_lo, deep_hi;
    int guard;             // guard planes allocated below plane 0 (tensor-map offset)
    // peer-store halos: p_{j+2} / p_{j+3} of the neighbouring
    // slab below (lo) / above (hi), null for none.  Level 2 also stores its
    // planes 1, 2 (nzl-1, nzl) and level 3 its planes 1..3 (nzl-2..nzl) into the
    // neighbour's ghost planes (its nzl_lo+1.. / -2..0), which replaces the
    // exchange after the triple
    double *peer_lo[2], *peer_hi[2];
    int peer_nzl_lo;       // nzl of the slab below
    int peer_sys_fence;    // a neighbour is another process: fence.sc.sys after the peer stores
    double sigma;
    const CUtensorMap *tmP, *tmM;
};
bool k1m_enabled(const Geo &g, int nzl);
bool k1m_prepare(const Geo &g, const double *P, int nzl, int s, CUtensorMap *tmP, CUtensorMap *tmM, int guard);
void launch_k1m(const Geo &g, const K1MArgs &a, double theta, const DevState *st, cudaStream_t strm);
bool k1f_prepare(const Geo &g, const double *P, int nzl, int s, CUtensorMap *tmP, CUtensorMap *tmM);
void launch_k1f(const Geo &g, const K1Args &a, double theta, int s, const DevState *st, cudaStream_t strm);

// copy a process-layout grid function into the padded interior of `dst`
void launch_pack(const Geo &g, const double *src, double *dst, int nzl, const DevState *st,
                 cudaStream_t s);
// copy the padded interior of `src` back to process layout
void launch_unpack(const Geo &g, const double *src, double *dst, int nzl, cudaStream_t s);

// K2: fused Gram Ghat = P^T W (upper incl. diagonal) and c = P^T p_0
void launch_k2(const Geo &g, const Slab &sl, int s, const DevState *st, double *out_blk,
               cudaStream_t stream);
int k2_grid();
bool k2_prepare(const Geo &g, Slab &sl, int s);   // encode the TMA tensor maps
int k2_num_entries(int s);
// K2D: the Gram pass on FP64 tensor cores (k_gram_dmma.cu), s > 16 by default
bool k2d_enabled(const Geo &g, int s);
// K2R: DMMA Gram pass recovering W = AP from the basis recurrence (W not stored, R23)
bool k2r_prepare(const Geo &g, Slab &sl, int s, int nvec = 0);
// the block-conjugate mode's Gram pass with W_k recovered (sl.has_k2rb)
void launch_k2r_block(const Geo &g, const Slab &sl, int s, double theta, double sigma, const DevState *st,
                      double *out_blk, cudaStream_t stream);
void launch_k2r(const Geo &g, const Slab &sl, int s, double theta, double sigma, const DevState *st, double *out_blk,
                cudaStream_t stream, bool fold = false);
// the w_{s-1} fold: Ghat_{s-1,s-1} = p_{s-1}^T A p_{s-1} of one slab
// into its Gram block (after launch_k2r with fold = true)
void launch_pap(const Geo &g, const Slab &sl, int s, const DevState *st, double *out_blk, cudaStream_t stream);
// w_j (j < s-1) from the recurrence into `out` (a vector in the padded layout) -- parity hooks
void launch_wrec(const Geo &g, const Slab &sl, int j, double theta, double sigma, double *out, cudaStream_t stream);
bool k2d_prepare(const Geo &g, Slab &sl, int s);
void launch_k2d(const Geo &g, const Slab &sl, int s, const DevState *st, double *out_blk, cudaStream_t stream);

// fixed-order sum of per-slab blocks into `blk`
void launch_slab_sum(const double *const *blks_dev, int nslab, int len, double *blk,
                     const DevState *st, cudaStream_t s);

// K4: Ruhe scaling + nu FGS sweeps (single CTA) + stopping test + history
struct K4Args {
    const double *blk;     // [Ghat (s*s) | c (s)] after allreduce
    double *alpha;         // out: alpha = d o a~ (s)
    int s, nu;
    int solver;            // 0 = nu FGS sweeps, 1 = dense Cholesky
    int pdl;               // launch with programmatic dependent launch (Knobs::pdl)
    const double *rn2;     // ||r_k||^2 for the stopping test, or nullptr: c_0 of blk (the block-conjugate
                           // mode solves Q_k^T A Q_k a = Q_k^T r_k, whose c_0 is not ||r_k||^2)
    double *h_gram, *h_d, *h_at, *h_al, *h_delta, *h_relres;  // history [cap][...]
    double *h_lnorm;       // ||L||_F of the scaled Gram matrix G = I + L + L^T per outer
};
void launch_k4(const K4Args &a, DevState *st, cudaStream_t s);

// diagnostics: kappa(G) of the scaled Gram matrix of the last update (one warp)
void launch_kappa(const double *blk, int s, const DevState *st, double *h_kappa, cudaStream_t stream);
// diagnostics: ||P_k||_F (per-block partials, then phase 0: ordered sum, phase 1: budget term)
void launch_pnorm(const Geo &g, const Slab &sl, int s, double *part, int nblk, const DevState *st, cudaStream_t stream);
void launch_budget(const double *part, int nparts, double *sum, double anorm, bool allreduce_needed,
                   const DevState *st, const double *h_delta, double *h_pnorm, double *h_budget, cudaStream_t stream,
                   int phase);
void launch_anorm(const Geo &g, const Slab &sl, double *bmax, int nblk, cudaStream_t stream);

// K5: x += P alpha;  p_0 -= W alpha over padded planes [zb, ze) (ze < 0: to nzl+1)
//   rec: form W alpha from the Chebyshev recurrence (constant diagonal, vector path only)
void launch_k5(const Geo &g, const Slab &sl, int s, const double *alpha, double *const *xpp, int64_t xoff,
               const DevState *st, cudaStream_t stream, int zb, int ze, double theta, double sigma, bool rec,
               bool fold = false);

// KS: one whole outer iteration in one launch of one 8-CTA cluster for small problems (k_small.cu)
bool ks_supported(const Geo &g, int s, int64_t npts);
bool ks_prepare();   // opt in to the shared-memory ring (once per process)
void launch_ks(const Geo &g, const Slab &sl, int s, double theta, double sigma, double *const *xpp, double *blk,
               const K4Args &k4, DevState *st, cudaStream_t stream);

// block-conjugate s-step CG (k_blockcg.cu, R24)
void launch_bcg_prep(const double *big, int s, double *blk2, double *Bm, DevState *st, bool pdl, cudaStream_t strm);
void launch_k5_block(const Geo &g, const Slab &sl, int s, const double *alpha, const double *B, double *const *xpp,
                     int64_t xoff, const DevState *st, cudaStream_t stream, int zb, int ze, bool rec = false,
                     double theta = 0.0, double sigma = 0.0);

// Lanczos spectral bounds (k_lanczos.cu)
int lz_grid();
void lz_diag(const Geo &g, const Slab &sl, double *D, cudaStream_t s);
void lz_init(const Geo &g, const Slab &sl, const double *v0, const double *D, const double *nrm2, double *y,
             cudaStream_t s);
void lz_dot(const double *x, const double *y, const double *D, int64_t N, int mode, double *part, unsigned *ticket,
            double *out, const int *stop, cudaStream_t s);
void lz_sum(const double *vals, int n, double *out, const int *stop, cudaStream_t s);
void lz_update(const double *w, const double *D, const double *y, const double *yp, double *z, int64_t N,
               const double *a, const double *bprev, const int *stop, cudaStream_t s);
void lz_record(const double *a, const double *b2, double *alpha, double *beta, double *bprev, int k, int *stop, int *m,
               cudaStream_t s);
void lz_scale(double *z, int64_t N, const double *bprev, const int *stop, cudaStream_t s);
void lz_extremes(const double *alpha, const double *beta, const int *m, double margin, double *out, cudaStream_t s);

}  // namespace sscg
