// Host driver and C ABI of libsscg (include/sscg.h).
//
// Per outer iteration k (restart form, R3):
//   for j = 0..s-1:  halo(p_j) ; K1(j)            basis + W = AP
//   K2 per slab -> [slab sum] -> one ncclAllReduce  Gram block [Ghat | c]
//   K4                                              stop test, scaling, FGS
//   K5 per slab                                     x += P alpha, r -= W alpha
// The stopping decision is taken on the device (K4 sets DevState::done and
// every later kernel exits at once), so the host enqueues several outer
// iterations before it reads the flag back.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>
#include <unistd.h>
#include <chrono>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sscg.h"
#include "sscg_internal.cuh"

using namespace sscg;

static thread_local std::string g_err;

static sscg_status fail(sscg_status st, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

// for the other C-ABI translation units (k_coarse.cu)
namespace sscg {
sscg_status api_fail(sscg_status st, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}
}  // namespace sscg

#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return fail(e_ == cudaErrorMemoryAllocation ? SSCG_ERR_OOM : SSCG_ERR_CUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                        \
    } while (0)

#define NC(call)                                                                                   \
    do {                                                                                           \
        ncclResult_t r_ = (call);                                                                  \
        if (r_ != ncclSuccess)                                                                     \
            return fail(SSCG_ERR_NCCL, "%s: %s (%s:%d)", #call, ncclGetErrorString(r_), __FILE__, __LINE__); \
    } while (0)

struct sscg_ctx {
    Geo g{};
    int s = 0, nu = 0;
    double lmin = 0, lmax = 0, theta = 0, sigma = 0;
    int rank = 0, nranks = 1, spr = 1;
    bool nccl_self = false;   // SSCG_NCCL_SELF=1 with one rank: the NCCL paths on a 1-rank communicator
    int64_t nz_global = 1, z0_proc = 0, nzl_proc = 1, n_local = 0;
    std::vector<Slab> slabs;
    std::vector<void *> allocs;
    double *blk = nullptr;            // final [Ghat | c]
    int nvec = 0;                     // vectors of P and W per slab (s; 2s in the block-conjugate mode)
    bool blockcg = false;             // block-conjugate s-step CG (SSCG_OPT_BLOCKCG, R24)
    double *blk2 = nullptr;           // block mode: [G_k | c_k], the conjugated system K4 solves
    double *bmat = nullptr;           // block mode: B_k (s x s)
    double **blkptrs = nullptr;       // device array of slab block pointers
    double *alpha = nullptr;
    DevState *st = nullptr;
    DevState *st_host = nullptr;      // pinned
    // history (device) and host copies
    int hist_cap = 0, gram_cap = 0;
    double *h_lnorm = nullptr;
    double *h_gram = nullptr, *h_d = nullptr, *h_at = nullptr, *h_al = nullptr, *h_delta = nullptr,
           *h_relres = nullptr;
    std::vector<double> relres_host, delta_host;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // halo overlap: boundary planes first, then the exchange of
    // the next basis vector's boundary planes on `cstream` while the interior
    // planes run on `stream`
    cudaStream_t cstream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_xready = nullptr;
    double *x_host_out = nullptr;   // sscg_solve_host: copy x out as soon as it is final
    bool x_copied = false;
    bool overlap = true;
    bool failed = false;            // an NCCL abort left the context unusable (every call: SSCG_ERR_NCCL)
    // the fused basis schedules every rank can run (AND over ranks at setup: slabs of
    // different depth may cross a kernel's size threshold, and the halo exchanges of
    // all ranks must match step for step)
    bool all_mp3 = true, all_fused = true;
    double nccl_timeout_s = 600.0;  // SSCG_NCCL_TIMEOUT_S, read at setup
    int k1_sm_cap = 0;
    // variants on the same boundary
    int gram_solver = SSCG_GRAM_FGS;
    int basis = SSCG_BASIS_CHEBYSHEV;
    bool bounds_set = false;
    bool diagnostics = false;
    double *h_kappa = nullptr, *h_pnorm = nullptr, *h_budget = nullptr;
    double *diag_part = nullptr, *diag_sum = nullptr;   // ||P||_F partials [slab][DIAG_BLK], sum
    double anorm = 0.0;                                  // Gershgorin bound of ||A||_2 (global)
    // Lanczos workspace (sscg_estimate_bounds): 3 vectors + D per slab, lazily
    std::vector<double *> lz_vec;     // [slab * 5 + {y0, y1, y2, w, D}]
    double *lz_scal = nullptr;        // device scalars, see sscg_estimate_bounds
    int lz_iters = 0;
    int *lz_flags = nullptr;          // {stop, m}
    double *lz_part = nullptr;        // dot partials [slab][grid]
    unsigned *lz_ticket = nullptr;    // [slab]
    ncclComm_t comm = nullptr;
    // cross-rank peer-store halos: the neighbours' P mapped through
    // CUDA IPC (or, SSCG_NCCL_SELF, the in-process slabs' descriptors after the
    // same NCCL round trip); after each deep triple a one-double token to every
    // such neighbour orders its next triple after this one's stores
    bool peer_remote = false;
    int peer_rank[2] = {-1, -1};      // rank below slab 0 / above the last slab (-1: none)
    std::vector<void *> ipc_open;     // mappings to close at destroy
    double *token = nullptr;          // [send, recv lo, recv hi]
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    double *bbuf = nullptr, *xbuf = nullptr;   // device buffers of sscg_solve_host
    double *scratch = nullptr;                 // process-layout scratch for inspect
    sscg_stats_t stats{};
    int64_t launches = 0, allreduces = 0;
    int last_max_outer = -1;
    bool solved = false;
    // profiling
    bool prof_on = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
    std::vector<int> prof_cat;
    size_t prof_used = 0;
    sscg_profile_t prof{};
    // CUDA graph of one outer iteration
    bool use_graph = true;
    cudaGraphExec_t gexec = nullptr;
    double **xdev = nullptr;      // device cell with the current x (K5 reads it per launch)
    double **xhost = nullptr;     // pinned staging of that pointer
    int64_t graph_launches = 0, graph_allreduces = 0;
};

static const char *kVersion = "sscg-b200 0.1 (sm_100a)";
static const int DIAG_BLK = 592;   // blocks of the ||P||_F diagnostic per slab
static const int GRAM_HIST = 2048; // outer iterations whose Gram block / d / alpha are recorded

extern "C" const char *sscg_version(void) { return kVersion; }
extern "C" const char *sscg_last_error(void) { return g_err.c_str(); }

extern "C" sscg_status sscg_partition(int64_t nz, int32_t nranks, int32_t spr, int32_t rank, int64_t *z0,
                                      int64_t *nzl)
{
    if (nz < 1 || nranks < 1 || spr < 1 || rank < 0 || rank >= nranks || !z0 || !nzl)
        return fail(SSCG_ERR_INVALID, "sscg_partition: bad arguments");
    const int64_t S = (int64_t)nranks * spr;
    if (nz < S) return fail(SSCG_ERR_INVALID, "sscg_partition: %lld planes < %lld slabs", (long long)nz, (long long)S);
    const int64_t g0 = (int64_t)rank * spr, g1 = g0 + spr;
    *z0 = g0 * nz / S;
    *nzl = g1 * nz / S - *z0;
    return SSCG_OK;
}

extern "C" sscg_status sscg_halo_plan(int64_t nz, int32_t nranks, int32_t spr, int32_t rank, int32_t slab,
                                      int64_t *out6)
{
    if (!out6 || slab < 0 || slab >= spr) return fail(SSCG_ERR_INVALID, "sscg_halo_plan: bad slab");
    int64_t z0p, nzp;
    const sscg_status ps = sscg_partition(nz, nranks, spr, rank, &z0p, &nzp);
    if (ps != SSCG_OK) return ps;
    const int64_t S = (int64_t)nranks * spr, g = (int64_t)rank * spr + slab;
    const int64_t z0 = g * nz / S, z1 = (g + 1) * nz / S;   // this slab: [z0, z1)
    out6[0] = (g > 0) ? (g - 1) / spr : -1;
    out6[1] = z0;
    out6[2] = z0 - 1;
    out6[3] = (g + 1 < S) ? (g + 1) / spr : -1;
    out6[4] = z1 - 1;
    out6[5] = z1;
    return SSCG_OK;
}

extern "C" sscg_status sscg_nccl_unique_id(void *out)
{
    if (!out) return fail(SSCG_ERR_INVALID, "null output");
    ncclUniqueId id;
    NC(ncclGetUniqueId(&id));
    memcpy(out, &id, sizeof id);
    return SSCG_OK;
}

template <class T>
static sscg_status dalloc(sscg_ctx *c, T **p, size_t count)
{
    void *q = nullptr;
    cudaError_t e = cudaMalloc(&q, count * sizeof(T) + 16);
    if (e != cudaSuccess) {
        *p = nullptr;
        return fail(SSCG_ERR_OOM, "cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
    }
    c->allocs.push_back(q);
    *p = static_cast<T *>(q);
    return SSCG_OK;
}

#define TRY(x)                           \
    do {                                 \
        sscg_status t_ = (x);            \
        if (t_ != SSCG_OK) return t_;    \
    } while (0)

__global__ void k_recip_pack(Geo g, const double *diag, double *dinv, int nzl)
{
    // dinv (padded vector layout) = 1 / diag (process layout)
    const int64_t nxy = (int64_t)g.nx * g.ny, tot = nxy * nzl;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t zl = e / nxy, rem = e - zl * nxy;
        const int64_t y = rem / g.nx, x = rem - y * g.nx;
        dinv[(zl + 1) * g.plane + y * g.pitch + x] = 1.0 / diag[e];
    }
}

__global__ void k_csr_dinv(Geo g, double *dinv)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= g.n) return;
    double d = 0.0;
    for (int64_t q = g.rowptr[r]; q < g.rowptr[r + 1]; ++q)
        if (g.colind[q] == r) d += g.val[q];
    dinv[g.plane + r] = 1.0 / d;
}

static void dfree(sscg_ctx *c, void *p);

// (Re)build the basis store of every slab: P and W with nvec vectors (s; 2s in
// the block-conjugate mode, whose upper halves hold Q_{k-1} and A Q_{k-1}) and
// every tensor map over them.  Device work is ordered on the solver stream.
static sscg_status build_basis_store(sscg_ctx *c, int nvec)
{
    Geo &g = c->g;
    const int s = c->s;
    for (auto &sl : c->slabs) {
        if (sl.Palloc) {
            CU(cudaStreamSynchronize(c->stream));
            dfree(c, sl.Palloc);
            dfree(c, sl.Walloc);
        }
        TRY(dalloc(c, &sl.Palloc, (size_t)g.vstride * nvec));
        TRY(dalloc(c, &sl.Walloc, (size_t)g.vstride * nvec));
        CU(cudaMemsetAsync(sl.Palloc, 0, (size_t)g.vstride * nvec * sizeof(double), c->stream));
        CU(cudaMemsetAsync(sl.Walloc, 0, (size_t)g.vstride * nvec * sizeof(double), c->stream));
        sl.P = sl.Palloc + (int64_t)g.guard * g.plane;   // vectors address plane 0; planes -guard.. lie before it
        sl.W = sl.Walloc + (int64_t)g.guard * g.plane;
        // the stored-W Gram pass runs over all nvec rows ([P | Q'] x [W | Z'] in the block mode)
        if (!k2_prepare(g, sl, nvec)) return fail(SSCG_ERR_CUDA, "cuTensorMapEncodeTiled failed for the Gram pass");
        const int kind = g.kind;
        if (kind == SSCG_OP_STENCIL7 || kind == SSCG_OP_STENCIL27 || kind == SSCG_OP_VARCOEF7) {
            if (!k1t_prepare(g, sl.P, sl.nzl, s, &sl.tmP4, &sl.tmM4))
                return fail(SSCG_ERR_CUDA, "cuTensorMapEncodeTiled failed for the basis step");
            sl.has_k1t = true;
        }
        if (sl.want_k1f) {
            if (!k1f_prepare(g, sl.P, sl.nzl, s, &sl.tmF_P, &sl.tmF_M))
                return fail(SSCG_ERR_CUDA, "cuTensorMapEncodeTiled failed for the fused basis step");
            sl.has_k1f = true;
        }
        if (sl.want_k1m) {
            if (!k1m_prepare(g, sl.P, sl.nzl, s, &sl.tmM3_P, &sl.tmM3_M, g.guard))
                return fail(SSCG_ERR_CUDA, "cuTensorMapEncodeTiled failed for the depth-3 basis step");
            sl.has_k1m = true;
        }
        if (sl.want_k1fv) {
            if (!k1fv_prepare(g, sl.P, sl.nzl, s, &sl.tmF_P, &sl.tmF_M))
                return fail(SSCG_ERR_CUDA, "cuTensorMapEncodeTiled failed for the fused variable-coefficient step");
            sl.has_k1f = true;
        }
        if (kind == SSCG_OP_STENCIL7 || kind == SSCG_OP_STENCIL27 || kind == SSCG_OP_VARCOEF7 || kind == SSCG_OP_CSR) {
            if (!k2r_prepare(g, sl, s, nvec)) return fail(SSCG_ERR_CUDA, "tensor maps for the recovered-W Gram pass");
            sl.has_k2r = true;
        }
    }
    c->nvec = nvec;
    return SSCG_OK;
}

// Gram-pass partials and blocks for `rows` basis rows (rows^2 + rows entries)
static sscg_status alloc_gram_buffers(sscg_ctx *c, int rows)
{
    const int nent = rows * rows + rows;
    const int64_t npart = (int64_t)k2_grid() * 8 * nent;
    CU(cudaStreamSynchronize(c->stream));
    for (auto &sl : c->slabs) {
        dfree(c, sl.part);
        dfree(c, sl.blk);
        TRY(dalloc(c, &sl.part, (size_t)npart));
        TRY(dalloc(c, &sl.blk, (size_t)nent));
    }
    dfree(c, c->blk);
    TRY(dalloc(c, &c->blk, (size_t)nent));
    std::vector<double *> ptrs;
    for (auto &sl : c->slabs) ptrs.push_back(sl.blk);
    dfree(c, c->blkptrs);
    TRY(dalloc(c, &c->blkptrs, ptrs.size()));
    CU(cudaMemcpyAsync(c->blkptrs, ptrs.data(), ptrs.size() * sizeof(double *), cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return SSCG_OK;
}

Knobs sscg::read_knobs()
{
    Knobs k;
    auto tri = [](const char *name, int dflt) {
        const char *e = getenv(name);
        return e ? (e[0] == '1' ? 1 : e[0] == '0' ? 0 : dflt) : dflt;
    };
    auto num = [](const char *name, int dflt) {
        const char *e = getenv(name);
        return e ? atoi(e) : dflt;
    };
    k.k1_fuse = tri("SSCG_K1_FUSE", -1);
    k.k1_mp3 = tri("SSCG_K1_MP3", -1);
    k.k1_fuse_vc = tri("SSCG_K1_FUSE_VC", -1);
    k.k1_tma = tri("SSCG_K1_TMA", 1) != 0;
    k.k1_zc = std::max(0, num("SSCG_K1_ZC", 0));
    k.faces_tma = tri("SSCG_FACES_TMA", 1) != 0;
    k.k2_dmma = tri("SSCG_K2_DMMA", -1);
    k.k2s = tri("SSCG_K2S", 1) != 0;
    k.k2_e = num("SSCG_K2_E", 0);
    k.k2_ns = num("SSCG_K2_NS", 0);
    k.k2_grid = num("SSCG_K2_GRID", 0);
    k.k2_groups = std::max(0, num("SSCG_K2_GROUPS", 0));
    k.k2_smem_kb = std::min(224, std::max(64, num("SSCG_K2_SMEM_KB", 216)));
    k.wfree = tri("SSCG_WFREE", 1) != 0;
    k.k5_recur = tri("SSCG_K5_RECUR", 1) != 0;
    k.deep_halo = tri("SSCG_DEEP_HALO", 1) != 0;
    k.deep_overlap = tri("SSCG_DEEP_OVERLAP", 0) != 0;
    k.peer_halo = tri("SSCG_PEER_HALO", 1) != 0;
    k.small = tri("SSCG_SMALL", -1);
    k.debug = getenv("SSCG_DEBUG") != nullptr;
    k.pdl = tri("SSCG_PDL", 1) != 0;
    k.wl_fold = std::min(2, std::max(0, num("SSCG_WL_FOLD", 1)));
    k.gram_space = tri("SSCG_GRAM_SPACE", 0) == 1;
    k.k2_il = tri("SSCG_K2_IL", 1) != 0;
    return k;
}

static sscg_status setup_peers(sscg_ctx *c);

static sscg_status setup_impl(const sscg_operator *A, const double *diag_M, double lmin, double lmax, int s,
                              int nu, const sscg_comm *cm, void *stream, sscg_ctx *c)
{
    if (!A) return fail(SSCG_ERR_INVALID, "null operator");
    if (s < 1 || s > 64) return fail(SSCG_ERR_INVALID, "s = %d outside [1, 64]", s);
    if (nu < 1) return fail(SSCG_ERR_INVALID, "nu = %d < 1", nu);
    if (lmin == 0.0 && lmax == 0.0) {
        c->bounds_set = false;   // to be estimated (sscg_estimate_bounds) and set (sscg_set_bounds)
    } else if (!(lmin > 0.0) || !(lmax > lmin) || !std::isfinite(lmax)) {
        return fail(SSCG_ERR_INVALID, "need 0 < lambda_min < lambda_max (got %g, %g)", lmin, lmax);
    } else {
        c->bounds_set = true;
    }
    if (A->kind < 0 || A->kind > 4) return fail(SSCG_ERR_INVALID, "unknown operator kind %d", A->kind);
    c->s = s;
    c->nu = nu;
    c->lmin = lmin;
    c->lmax = lmax;
    c->theta = 2.0 / (lmax - lmin);
    c->sigma = (lmax + lmin) / 2.0;
    if (cm) {
        c->rank = cm->rank;
        c->nranks = cm->nranks;
        c->spr = cm->slabs_per_rank;
    }
    if (c->nranks < 1 || c->rank < 0 || c->rank >= c->nranks || c->spr < 1)
        return fail(SSCG_ERR_INVALID, "bad comm (rank %d of %d, %d slabs per rank)", c->rank, c->nranks, c->spr);

    Geo &g = c->g;
    g.kn = read_knobs();
    g.kind = A->kind;
    if (A->kind == SSCG_OP_CSR) {
        if (c->nranks * c->spr != 1) return fail(SSCG_ERR_INVALID, "CSR operator supports a single slab only");
        if (A->n < 1 || !A->rowptr || !A->colind || !A->val) return fail(SSCG_ERR_INVALID, "CSR arrays missing");
        g.n = A->n;
        g.rowptr = A->rowptr;
        g.colind = A->colind;
        g.val = A->val;
        g.nx = (int)A->n;   // one "row" of n doubles per plane
        g.ny = 1;
        g.pitch = (int)A->n + (int)(A->n & 1);
        c->nz_global = 1;
    } else {
        if (A->nx < 1 || A->ny < 1 || A->nz < 1 || A->nx > (1 << 30) || A->ny > (1 << 30))
            return fail(SSCG_ERR_INVALID, "bad grid %lld x %lld x %lld", (long long)A->nx, (long long)A->ny,
                        (long long)A->nz);
        if (A->kind == SSCG_OP_STENCIL5_2D && A->nz != 1) return fail(SSCG_ERR_INVALID, "5-point stencil needs nz = 1");
        if (A->kind == SSCG_OP_VARCOEF7 && (!A->kx || !A->ky || !A->kz))
            return fail(SSCG_ERR_INVALID, "VARCOEF7 needs kx, ky, kz");
        g.nx = (int)A->nx;
        g.ny = (int)A->ny;
        g.pitch = g.nx + (g.nx & 1);
        c->nz_global = A->nz;
    }
    g.plane = (int64_t)g.ny * g.pitch;
    g.center = (A->kind == 0) ? 4.0 : (A->kind == 1) ? 6.0 : (A->kind == 2) ? 26.0 : 0.0;
    g.dinv_c = (g.center > 0) ? 1.0 / g.center : 0.0;

    TRY(sscg_partition(c->nz_global, c->nranks, c->spr, c->rank, &c->z0_proc, &c->nzl_proc));
    c->n_local = (A->kind == SSCG_OP_CSR) ? A->n : (int64_t)g.nx * g.ny * c->nzl_proc;

    if (stream) {
        c->stream = static_cast<cudaStream_t>(stream);
    } else {
        // a BLOCKING stream: it orders after the caller's work on the legacy
        // default stream (e.g. torch producing b), so inputs are complete
        // before the first kernel reads them
        CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamDefault));
        c->own_stream = true;
    }
    if (const char *e = getenv("SSCG_NO_GRAPH")) c->use_graph = (e[0] == '0');
    if (const char *e = getenv("SSCG_NO_OVERLAP")) c->overlap = (e[0] == '0');
    if (const char *e = getenv("SSCG_NCCL_TIMEOUT_S")) c->nccl_timeout_s = atof(e);
    {
        int lo = 0, hi = 0;
        CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        CU(cudaStreamCreateWithPriority(&c->cstream, cudaStreamNonBlocking, hi));
        CU(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&c->ev_xready, cudaEventDisableTiming));
    }
    CU(cudaEventCreate(&c->ev0));
    CU(cudaEventCreate(&c->ev1));
    CU(cudaMallocHost(&c->st_host, sizeof(DevState)));
    TRY(dalloc(c, &c->st, 1));

    // slabs of this process
    const int S = c->nranks * c->spr;
    int max_nzl = 0;
    for (int l = 0; l < c->spr; ++l) {
        const int gidx = c->rank * c->spr + l;
        Slab sl{};
        sl.z0 = (int64_t)gidx * c->nz_global / S;
        sl.nzl = (int)((int64_t)(gidx + 1) * c->nz_global / S - sl.z0);
        sl.zoff = sl.z0 - c->z0_proc;
        sl.has_lo = gidx > 0;
        sl.has_hi = gidx + 1 < S;
        max_nzl = std::max(max_nzl, sl.nzl);
        c->slabs.push_back(sl);
    }
    // deep halos: 7-point slabs with neighbours keep 3 ghost
    // planes per side for the K1M triples -- two guard planes allocated beyond
    // the 1-plane halo on each side of every vector
    g.guard = (A->kind == SSCG_OP_STENCIL7 && !diag_M && S > 1 && g.kn.deep_halo) ? 2 : 0;
    g.vstride = ((int64_t)(max_nzl + 2 + 2 * g.guard) * g.plane + 31) / 32 * 32;   // 256-B aligned vectors
    if (getenv("SSCG_VPAD") && (g.vstride / 32) % 2 == 0) g.vstride += 32;   // odd multiple of 256 B
    for (auto &sl : c->slabs) {
        if (A->kind == SSCG_OP_VARCOEF7) {
            sl.kx = A->kx + sl.zoff * g.ny * (g.nx + 1);
            sl.ky = A->ky + sl.zoff * (g.ny + 1) * g.nx;
            sl.kz = A->kz + sl.zoff * g.ny * g.nx;
            sl.has_ftma = g.kn.faces_tma &&
                          k1t_prepare_faces(g, sl.kx, sl.ky, sl.kz, sl.nzl, &sl.tmKX, &sl.tmKY, &sl.tmKZ);
            sl.want_k1fv = !diag_M && k1fv_enabled(g, sl.nzl) &&
                           k1fv_prepare_faces(g, sl.kx, sl.ky, sl.kz, sl.nzl, &sl.tmV_KX, &sl.tmV_KY, &sl.tmV_KZ,
                                              &sl.kx_shift);
        }
        sl.want_k1f = (A->kind == SSCG_OP_STENCIL7 || A->kind == SSCG_OP_STENCIL27) && !diag_M && k1f_enabled(g, sl.nzl);
        sl.want_k1m = A->kind == SSCG_OP_STENCIL7 && !diag_M && k1m_enabled(g, sl.nzl);
        if (diag_M || A->kind == SSCG_OP_CSR) {
            double *dv = nullptr;
            TRY(dalloc(c, &dv, (size_t)g.vstride));
            CU(cudaMemsetAsync(dv, 0, (size_t)g.vstride * sizeof(double), c->stream));
            if (diag_M) {
                const int nzl = (A->kind == SSCG_OP_CSR) ? 1 : sl.nzl;
                const int64_t tot = (int64_t)g.nx * g.ny * nzl;
                k_recip_pack<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 16), 256, 0, c->stream>>>(
                    g, diag_M + sl.zoff * (int64_t)g.nx * g.ny, dv, nzl);
            } else {
                k_csr_dinv<<<(unsigned)((g.n + 255) / 256), 256, 0, c->stream>>>(g, dv);
            }
            CU(cudaGetLastError());
            sl.dinv = dv;
        }
        if (diag_M || A->kind == SSCG_OP_VARCOEF7 || A->kind == SSCG_OP_CSR) {
            // diag(M) per point for the recurrence form of the update (R21) and the
            // W-free Gram pass (R23); for CSR 1 / the D^{-1} the basis uses
            double *dd = nullptr;
            TRY(dalloc(c, &dd, (size_t)g.vstride));
            CU(cudaMemsetAsync(dd, 0, (size_t)g.vstride * sizeof(double), c->stream));
            lz_diag(g, sl, dd, c->stream);
            CU(cudaGetLastError());
            sl.dvec = dd;
        }
        TRY(dalloc(c, &sl.ticket, 1));
        CU(cudaMemsetAsync(sl.ticket, 0, sizeof(unsigned), c->stream));
    }
    TRY(build_basis_store(c, s));
    TRY(alloc_gram_buffers(c, s));
    if ((A->kind == SSCG_OP_STENCIL5_2D || A->kind == SSCG_OP_STENCIL7) && !ks_prepare())
        return fail(SSCG_ERR_CUDA, "shared-memory opt-in of the single-CTA outer iteration");
    TRY(dalloc(c, &c->xdev, 1));
    CU(cudaMallocHost(&c->xhost, sizeof(double *)));
    TRY(dalloc(c, &c->alpha, 64));
    TRY(dalloc(c, &c->scratch, (size_t)c->n_local));
    if (c->nranks > 1) {
        // interior K1 launches leave two SMs free so the NCCL send/recv kernels
        // of the overlapped halo exchange can be scheduled next to them
        c->k1_sm_cap = k2_grid() - 2;
        if (!cm->nccl_id) return fail(SSCG_ERR_INVALID, "nranks > 1 needs nccl_id");
        ncclUniqueId id;
        memcpy(&id, cm->nccl_id, sizeof id);
        NC(ncclCommInitRank(&c->comm, c->nranks, id, c->rank));
        // agree on the fused basis schedules (minimum over ranks of the local capability)
        int flags[2] = {1, 1};
        for (const auto &sl : c->slabs) {
            if (!sl.has_k1m || sl.nzl < 8) flags[0] = 0;
            if (!sl.has_k1f || sl.nzl < 4) flags[1] = 0;
        }
        int *dflags = nullptr;
        TRY(dalloc(c, &dflags, 2));
        CU(cudaMemcpyAsync(dflags, flags, sizeof flags, cudaMemcpyHostToDevice, c->stream));
        NC(ncclAllReduce(dflags, dflags, 2, ncclInt32, ncclMin, c->comm, c->stream));
        CU(cudaMemcpyAsync(flags, dflags, sizeof flags, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        c->all_mp3 = flags[0] != 0;
        c->all_fused = flags[1] != 0;
    } else if (const char *e = getenv("SSCG_NCCL_SELF"); e && e[0] == '1') {
        // test mode for a one-GPU box: a one-rank communicator carries the
        // allreduces, and the halos of in-process slabs move by NCCL send/recv
        // to self -- the NCCL calls, their graph capture and the polled waits
        // of the multi-rank path, on data that makes the result bitwise equal
        // to the plain in-process run
        c->k1_sm_cap = k2_grid() - 2;
        ncclUniqueId id;
        NC(ncclGetUniqueId(&id));
        NC(ncclCommInitRank(&c->comm, 1, id, 0));
        c->nccl_self = true;
    }
    TRY(setup_peers(c));
    CU(cudaStreamSynchronize(c->stream));
    return SSCG_OK;
}

extern "C" sscg_status sscg_setup(const sscg_operator *A, const double *diag_M, double lambda_min,
                                  double lambda_max, int32_t s, int32_t nu, const sscg_comm *comm, void *stream,
                                  sscg_ctx **out)
{
    if (!out) return fail(SSCG_ERR_INVALID, "null out");
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(SSCG_ERR_CUDA, "no CUDA device");
    sscg_ctx *c = new sscg_ctx();
    sscg_status st = setup_impl(A, diag_M, lambda_min, lambda_max, s, nu, comm, stream, c);
    if (st != SSCG_OK) {
        std::string keep = g_err;
        sscg_destroy(c);
        g_err = keep;
        return st;
    }
    *out = c;
    return SSCG_OK;
}

extern "C" void sscg_destroy(sscg_ctx *c)
{
    if (!c) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->cstream) cudaStreamSynchronize(c->cstream);
    // the captured outer iteration holds NCCL's persistent plans: release it
    // before the communicator (ncclCommDestroy waits for them otherwise)
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    c->gexec = nullptr;
    if (c->comm) ncclCommDestroy(c->comm);
    for (void *p : c->ipc_open) cudaIpcCloseMemHandle(p);
    for (void *p : c->allocs) cudaFree(p);
    if (c->st_host) cudaFreeHost(c->st_host);
    if (c->xhost) cudaFreeHost(c->xhost);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    for (auto &e : c->prof_events) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->ev_xready) cudaEventDestroy(c->ev_xready);
    if (c->cstream) cudaStreamDestroy(c->cstream);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

// ---------------------------------------------------------------------------
// halo exchange of one basis vector: np planes per side --
// the slab's planes [1, np] go to the lower neighbour's planes [nzl'+1,
// nzl'+np], its planes [nzl-np+1, nzl] to the upper neighbour's [1-np, 0].
// np = 1 is the 1-plane halo of a single basis step; np = 3 (p_j) and 2
// (p_{j-1}) the deep halo of a K1M triple (planes below 0 and
// above nzl+1 are the guard planes, Geo::guard >= np - 1)
static sscg_status exchange(sscg_ctx *c, double *const *vec_of_slab, cudaStream_t strm, int np = 1)
{
    const Geo &g = c->g;
    if (g.kind == SSCG_OP_CSR) return SSCG_OK;
    const size_t cnt = (size_t)np * g.plane, pb = cnt * sizeof(double);
    const int L = (int)c->slabs.size();
    // in-process neighbours (SSCG_NCCL_SELF: by NCCL send/recv to self, in order)
    if (c->nccl_self && L > 1) NC(ncclGroupStart());
    for (int l = 0; l + 1 < L; ++l) {
        double *lo = vec_of_slab[l], *hi = vec_of_slab[l + 1];
        const int nzl = c->slabs[l].nzl;
        double *lo_src = lo + (int64_t)(nzl - np + 1) * g.plane, *hi_dst = hi + (int64_t)(1 - np) * g.plane;
        double *hi_src = hi + g.plane, *lo_dst = lo + (int64_t)(nzl + 1) * g.plane;
        if (c->nccl_self) {
            NC(ncclSend(lo_src, cnt, ncclDouble, 0, c->comm, strm));
            NC(ncclRecv(hi_dst, cnt, ncclDouble, 0, c->comm, strm));
            NC(ncclSend(hi_src, cnt, ncclDouble, 0, c->comm, strm));
            NC(ncclRecv(lo_dst, cnt, ncclDouble, 0, c->comm, strm));
            continue;
        }
        CU(cudaMemcpyAsync(hi_dst, lo_src, pb, cudaMemcpyDeviceToDevice, strm));
        CU(cudaMemcpyAsync(lo_dst, hi_src, pb, cudaMemcpyDeviceToDevice, strm));
    }
    if (c->nccl_self && L > 1) NC(ncclGroupEnd());
    if (c->nranks > 1) {
        // remote neighbours of the first and last local slab (sscg_halo_plan)
        int64_t lo[6], hi[6];
        TRY(sscg_halo_plan(c->nz_global, c->nranks, c->spr, c->rank, 0, lo));
        TRY(sscg_halo_plan(c->nz_global, c->nranks, c->spr, c->rank, L - 1, hi));
        NC(ncclGroupStart());
        if (lo[0] >= 0 && lo[0] != c->rank) {
            // send planes from lo[1] (local 1) up, receive the planes below lo[2] + 1 (local 0 down)
            double *v = vec_of_slab[0];
            NC(ncclSend(v + g.plane, cnt, ncclDouble, (int)lo[0], c->comm, strm));
            NC(ncclRecv(v + (int64_t)(1 - np) * g.plane, cnt, ncclDouble, (int)lo[0], c->comm, strm));
        }
        if (hi[3] >= 0 && hi[3] != c->rank) {
            // send the planes up to hi[4] (local nzl), receive from hi[5] (local nzl+1) up
            double *v = vec_of_slab[L - 1];
            const int nzl = c->slabs[L - 1].nzl;
            NC(ncclSend(v + (int64_t)(nzl - np + 1) * g.plane, cnt, ncclDouble, (int)hi[3], c->comm, strm));
            NC(ncclRecv(v + (int64_t)(nzl + 1) * g.plane, cnt, ncclDouble, (int)hi[3], c->comm, strm));
        }
        NC(ncclGroupEnd());
    }
    return SSCG_OK;
}

// profiling: CUDA event pairs around launch groups, resolved on demand
static sscg_status prof_mark(sscg_ctx *c, int cat, bool begin, cudaStream_t strm = nullptr)
{
    if (!strm) strm = c->stream;
    if (!c->prof_on) return SSCG_OK;
    if (begin) {
        if (c->prof_used == c->prof_events.size()) {
            cudaEvent_t e0, e1;
            CU(cudaEventCreate(&e0));
            CU(cudaEventCreate(&e1));
            c->prof_events.push_back({e0, e1});
            c->prof_cat.push_back(cat);
        }
        c->prof_cat[c->prof_used] = cat;
        CU(cudaEventRecord(c->prof_events[c->prof_used].first, strm));
    } else {
        CU(cudaEventRecord(c->prof_events[c->prof_used].second, strm));
        ++c->prof_used;
    }
    return SSCG_OK;
}

static sscg_status prof_resolve(sscg_ctx *c)
{
    if (!c->prof_used) return SSCG_OK;
    CU(cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < c->prof_used; ++i) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, c->prof_events[i].first, c->prof_events[i].second));
        c->prof.ms[c->prof_cat[i]] += ms;
        c->prof.launches[c->prof_cat[i]] += 1;
    }
    c->prof_used = 0;
    return SSCG_OK;
}

static void drop_graph(sscg_ctx *c)
{
    if (c->gexec) {
        cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
    }
}

// Wait for `strm`.  With ranks, poll instead of blocking so that an NCCL
// failure (ncclCommGetAsyncError) or a peer that never arrives (timeout
// SSCG_NCCL_TIMEOUT_S, default 600 s) aborts the communicator and returns
// SSCG_ERR_NCCL instead of hanging (SURVEY §5 failure detection).
static sscg_status wait_stream(sscg_ctx *c, cudaStream_t strm)
{
    if (!c->comm) {
        CU(cudaStreamSynchronize(strm));
        return SSCG_OK;
    }
    const double limit = c->nccl_timeout_s;
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        const cudaError_t q = cudaStreamQuery(strm);
        if (q == cudaSuccess) return SSCG_OK;
        if (q != cudaErrorNotReady) return fail(SSCG_ERR_CUDA, "stream: %s", cudaGetErrorString(q));
        ncclResult_t ae = ncclSuccess;
        ncclCommGetAsyncError(c->comm, &ae);
        const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (ae != ncclSuccess || (limit > 0.0 && dt > limit)) {
            // the captured outer iteration holds NCCL nodes of this communicator:
            // drop it with the communicator, and refuse every later call
            drop_graph(c);
            ncclCommAbort(c->comm);
            c->comm = nullptr;
            c->failed = true;
            return fail(SSCG_ERR_NCCL, "NCCL %s after %.1f s (communicator aborted)",
                        ae != ncclSuccess ? ncclGetErrorString(ae) : "timeout", dt);
        }
        usleep(20);
    }
}

// halo of basis column j of every local slab; with overlap the exchange runs
// on the comm stream after the work already enqueued on the solver stream
// (fork) and `ev_join` marks its completion
// np planes of basis column j; with j2 >= 0 also np2 planes of column j2 (the
// deep halo of a K1M triple: p_j on 3 planes, p_{j-1} on 2)
static sscg_status halo_fork(sscg_ctx *c, int j, bool fork, int np = 1, int j2 = -1, int np2 = 0)
{
    const int L = (int)c->slabs.size();
    std::vector<double *> vj(L), vj2(L);
    for (int l = 0; l < L; ++l) {
        vj[l] = c->slabs[l].P + (int64_t)j * c->g.vstride;
        vj2[l] = c->slabs[l].P + (int64_t)std::max(j2, 0) * c->g.vstride;
    }
    cudaStream_t strm = fork ? c->cstream : c->stream;
    if (fork) {
        CU(cudaEventRecord(c->ev_fork, c->stream));
        CU(cudaStreamWaitEvent(c->cstream, c->ev_fork, 0));
    }
    TRY(prof_mark(c, SSCG_PROF_HALO, true, strm));
    TRY(exchange(c, vj.data(), strm, np));
    if (j2 >= 0 && np2 > 0) TRY(exchange(c, vj2.data(), strm, np2));
    TRY(prof_mark(c, SSCG_PROF_HALO, false, strm));
    if (fork) CU(cudaEventRecord(c->ev_join, c->cstream));
    return SSCG_OK;
}

static sscg_status halo_join(sscg_ctx *c)
{
    CU(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    return SSCG_OK;
}

// K5 forms W alpha from the Chebyshev recurrence (R21) for the
// constant-coefficient stencils with M = diag(A) and a Chebyshev basis
// (SSCG_K5_RECUR=0 keeps the stored-W form everywhere)
static bool uses_rec_update(const sscg_ctx *c)
{
    const Geo &g = c->g;
    if (!g.kn.k5_recur || c->blockcg) return false;
    if (c->basis != SSCG_BASIS_CHEBYSHEV || c->s < 2 || g.pitch != g.nx) return false;
    for (const auto &sl : c->slabs)
        if (!sl.dvec && !(g.center > 0.0 && !sl.dinv)) return false;   // need m or diag(M) per point
    return true;
}

// W = AP is not stored (except w_{s-1}) and the Gram pass recovers it from the
// basis recurrence (K2R, R23) when the basis kernels are K1T/K1F
// and the basis is Chebyshev (SSCG_WFREE=0 keeps the stored-W schedule)
static bool uses_wfree(const sscg_ctx *c)
{
    if (!c->g.kn.wfree) return false;
    if (c->basis != SSCG_BASIS_CHEBYSHEV || c->s < 2) return false;
    if (c->blockcg) {
        // the block mode (R24): W_k recovered in the 2s-row Gram pass (K2R BLK) and in
        // K5B; Z' = A Q' stays stored.  Constant diagonal, 2s <= 32 rows.
        const Geo &g = c->g;
        if (g.kind == SSCG_OP_CSR || !(g.center > 0.0) || g.pitch != g.nx) return false;
        for (const auto &sl : c->slabs)
            if (!sl.has_k2rb || !sl.has_k1t || sl.dvec || sl.dinv) return false;
        return true;
    }
    for (const auto &sl : c->slabs)   // (CSR: the row-per-thread K1, which skips w_j too)
        if (!sl.has_k2r || (!sl.has_k1t && c->g.kind != SSCG_OP_CSR)) return false;
    return uses_rec_update(c);   // the update must not need the stored W either
}

static bool uses_mp3(const sscg_ctx *c);
static bool uses_fused(const sscg_ctx *c);
static bool uses_wlfold(const sscg_ctx *c);

// KS (k_small.cu): the whole outer iteration in one launch of one 8-CTA
// cluster, for a single slab of at most 8192 points (its P and W fit the
// cluster's shared memory), 5-/7-point constant stencil, Chebyshev basis,
// s <= 8, FGS solver (auto: the 2D 5-point operator -- BASELINE cfg 1;
// SSCG_SMALL=1 forces it for any supported slab)
static bool uses_small(const sscg_ctx *c)
{
    const Geo &g = c->g;
    if (c->g.kn.small == 0 || c->slabs.size() != 1 || c->comm || c->basis != SSCG_BASIS_CHEBYSHEV ||
        c->gram_solver != SSCG_GRAM_FGS || c->blockcg || c->diagnostics || c->slabs[0].dinv)
        return false;
    const int64_t npts = (int64_t)g.nx * g.ny * c->slabs[0].nzl;
    if (!ks_supported(g, c->s, npts)) return false;
    return c->g.kn.small == 1 || g.kind == SSCG_OP_STENCIL5_2D;
}

// K1 for step j over the planes of every local slab selected by `part`:
//   0 = all planes, 1 = the two boundary planes (1 and nzl), 2 = the interior
//   planes [2, nzl) that do not read a halo plane, 3 = the two planes next to
//   each boundary (1, 2, nzl-1, nzl; the third step of a K1M triple)
static sscg_status launch_basis(sscg_ctx *c, int j, int part, bool ignore_stop = false)
{
    const Geo &g = c->g;
    const int s = c->s;
    for (auto &sl : c->slabs) {
        K1Args a{};
        a.p = sl.P + (int64_t)j * g.vstride;
        a.pm = (j > 0) ? sl.P + (int64_t)(j - 1) * g.vstride : nullptr;
        a.w = sl.W + (int64_t)j * g.vstride;
        a.pn = (j < s - 1) ? sl.P + (int64_t)(j + 1) * g.vstride : nullptr;
        a.kx = sl.kx; a.ky = sl.ky; a.kz = sl.kz;
        a.dinv = sl.dinv;
        a.dinv_c = g.dinv_c;
        a.sigma = c->sigma;
        a.coef = (j == 0) ? c->theta : 2.0 * c->theta;
        a.mode = (j == s - 1) ? 0 : (j == 0 ? 1 : 2);
        if (c->basis == SSCG_BASIS_MONOMIAL) {   // p_{j+1} = M^{-1} A p_j
            a.sigma = 0.0;
            a.coef = 1.0;
            a.mode = (j == s - 1) ? 0 : 1;
        }
        a.nzl = sl.nzl;
        a.j = j;
        a.skip_w = (uses_wfree(c) && j < s - 1) ? 1 : 0;
        if (sl.has_k1t) {
            a.tmP4 = &sl.tmP4;
            a.tmM4 = &sl.tmM4;
        }
        if (sl.has_ftma) {
            a.tmKX = &sl.tmKX;
            a.tmKY = &sl.tmKY;
            a.tmKZ = &sl.tmKZ;
        }
        if (part == 0) {
            a.zb = 1; a.ze = sl.nzl + 1;
        } else if (part == 1) {
            a.zb = 1; a.ze = 2;
            a.zb2 = std::max(2, sl.nzl); a.ze2 = sl.nzl + 1;
        } else if (part == 3) {
            a.zb = 1; a.ze = std::min(3, sl.nzl + 1);
            a.zb2 = std::max(a.ze, sl.nzl - 1); a.ze2 = sl.nzl + 1;
        } else {
            a.zb = 2; a.ze = sl.nzl;
            a.sm_cap = c->k1_sm_cap;
            if (a.ze <= a.zb) continue;
        }
        const int cat = (uses_mp3(c) || uses_fused(c)) ? SSCG_PROF_BASIS_SINGLE : SSCG_PROF_BASIS;
        TRY(prof_mark(c, cat, true));
        launch_k1(g, a, ignore_stop ? nullptr : c->st, c->stream);   // (no state: runs after the stop too)
        TRY(prof_mark(c, cat, false));
        ++c->launches;
    }
    return SSCG_OK;
}

// w_{s-1} fold: under the W-free schedule on the 7-point
// constant-centre stencil, w_{s-1} = A p_{s-1} is never stored: the Gram pass
// takes column s-1 from the transposed products w_i^T p_{s-1} (K2R PAP), one
// reduction pass over p_{s-1} gives p_{s-1}^T A p_{s-1} (k_pap), and the
// update forms w_{s-1} per point from p_{s-1} and its neighbours (K5 FOLD), so
// the basis schedules stop at p_{s-1} and the single step j = s-1 disappears
// (SSCG_WL_FOLD=0 keeps it)
static bool uses_wlfold(const sscg_ctx *c)
{
    const Geo &g = c->g;
    if (g.kn.wl_fold != 1 || g.kind != SSCG_OP_STENCIL7 || c->blockcg || !uses_wfree(c)) return false;
    if (c->s > 32 || (c->s <= 8 && g.kn.k2s)) return false;   // K2R with at most 4 row blocks; K2S reads the stored w_{s-1}
    if ((g.nx & 1) || g.pitch != g.nx) return false;             // k_pap and K5 run on point pairs
    for (const auto &sl : c->slabs)
        if (sl.dvec || sl.dinv) return false;
    // K1F pairs with s even end on a pair that stores p_{s-1} and w_{s-1}; the fold
    // would replace it by a single step plus the dot pass (one more launch for the
    // same bytes: cfg 2 measured 0.2509 vs 0.2488 ms per outer), so there only
    // the update half applies (uses_k5fold)
    if (!uses_mp3(c) && uses_fused(c) && c->s % 2 == 0) return false;
    return true;
}

// the update half of the fold alone (SSCG_WL_FOLD=2, or with the full fold):
// K5 forms w_{s-1} from p_{s-1} and its neighbours instead of reading it
static bool uses_k5fold(const sscg_ctx *c)
{
    const Geo &g = c->g;
    if (g.kn.wl_fold == 0 || g.kind != SSCG_OP_STENCIL7 || !uses_rec_update(c) || (g.nx & 1)) return false;
    for (const auto &sl : c->slabs)
        if (sl.dvec || sl.dinv) return false;
    return true;
}

// K1F pairs are used when every slab has the fused tensor maps (7-point,
// constant diagonal) and, with neighbours, enough planes for an interior
static bool uses_fused(const sscg_ctx *c)
{
    if (c->basis != SSCG_BASIS_CHEBYSHEV ||
        (c->g.kind != SSCG_OP_STENCIL7 && c->g.kind != SSCG_OP_STENCIL27 && c->g.kind != SSCG_OP_VARCOEF7))
        return false;
    if (!c->all_fused) return false;   // some rank's slabs cannot (every rank must run the same schedule)
    const bool halo = c->slabs.size() > 1 || c->nranks > 1;
    for (const auto &sl : c->slabs)
        if (!sl.has_k1f || (halo && sl.nzl < 4)) return false;
    return true;
}

// K1M triples (three basis steps per launch): 7-point; with neighbours each
// slab needs an interior for the third level ([3, nzl-1))
static bool uses_mp3(const sscg_ctx *c)
{
    if (c->basis != SSCG_BASIS_CHEBYSHEV || c->g.kind != SSCG_OP_STENCIL7 || !c->all_mp3) return false;
    const bool halo = c->slabs.size() > 1 || c->nranks > 1;
    for (const auto &sl : c->slabs)
        if (!sl.has_k1m || (halo && sl.nzl < 8)) return false;
    return true;
}

// deep halos: with neighbours, the K1M triples run on slabs
// whose p_j carries 3 ghost planes and p_{j-1} 2 (one exchange per triple, no
// boundary single steps); needs the guard planes allocated at setup
static bool uses_deep(const sscg_ctx *c)
{
    const bool halo = c->slabs.size() > 1 || c->nranks > 1;
    return halo && c->g.guard >= 2 && uses_mp3(c);
}

// peer-store halos: each deep triple stores the planes its
// neighbours need straight into their ghost planes (K1M), so no exchange
// follows it -- in-process neighbours by pointer; other ranks' basis mapped
// through CUDA IPC at setup (peer_remote), then a token orders the triples
static bool uses_peer(const sscg_ctx *c)
{
    if (!c->g.kn.peer_halo || c->g.kn.deep_overlap || !uses_deep(c)) return false;
    return (c->nranks == 1 && c->slabs.size() > 1 && !c->nccl_self) || c->peer_remote;
}

// the descriptor of one slab's P that a neighbour needs to store into it
struct PeerInfo {
    cudaIpcMemHandle_t h;
    int64_t off, vstride;   // P - the allocation (bytes), vector stride (doubles)
    int32_t nzl, pid;
    uint64_t nonce, base;   // this process, and the allocation's address in it
};

static uint64_t proc_nonce()
{
    static int anchor;
    return (uint64_t)(uintptr_t)&anchor ^ ((uint64_t)getpid() << 32);
}

// a neighbour's P: its own pointer in this process (the SSCG_NCCL_SELF test
// mode), else the allocation opened through CUDA IPC (null if that fails)
static double *peer_map(sscg_ctx *c, const PeerInfo &pi, bool *remote)
{
    void *base = nullptr;
    *remote = !(pi.pid == (int32_t)getpid() && pi.nonce == proc_nonce());
    if (!*remote) {
        base = (void *)(uintptr_t)pi.base;
    } else {
        if (cudaIpcOpenMemHandle(&base, pi.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        c->ipc_open.push_back(base);
    }
    return reinterpret_cast<double *>(static_cast<char *>(base) + pi.off);
}

// neighbour descriptors of every slab: in-process neighbours by pointer; with a
// communicator and the deep peer-store schedule, the other ranks' first / last
// slab exchanged by NCCL and mapped (SSCG_NCCL_SELF: the in-process pairs make
// the same round trip to self).  All ranks agree (min over the communicator)
// or every rank keeps the NCCL exchange of the ghost planes.
static sscg_status setup_peers(sscg_ctx *c)
{
    const Geo &g = c->g;
    const int L = (int)c->slabs.size();
    for (void *p : c->ipc_open) cudaIpcCloseMemHandle(p);   // a rebuilt store (SSCG_OPT_BLOCKCG): map again
    c->ipc_open.clear();
    for (int l = 0; l < L; ++l) {
        Slab &sl = c->slabs[l];
        for (int d = 0; d < 2; ++d) {
            sl.nbP[d] = nullptr;
            sl.nbvs[d] = 0;
            sl.nbnzl[d] = 0;
            sl.nb_remote[d] = 0;
        }
        if (l > 0) {
            sl.nbP[0] = c->slabs[l - 1].P;
            sl.nbvs[0] = g.vstride;
            sl.nbnzl[0] = c->slabs[l - 1].nzl;
        }
        if (l + 1 < L) {
            sl.nbP[1] = c->slabs[l + 1].P;
            sl.nbvs[1] = g.vstride;
            sl.nbnzl[1] = c->slabs[l + 1].nzl;
        }
    }
    c->peer_remote = false;
    if (!c->comm || !g.kn.peer_halo || g.kn.deep_overlap || !uses_deep(c)) return SSCG_OK;
    // messages: (slab whose descriptor is sent, peer rank) and (slab, side, peer rank) received
    struct Tx { int slab, peer; };
    struct Rx { int slab, side, peer; };
    std::vector<Tx> tx;
    std::vector<Rx> rx;
    if (c->nranks > 1) {
        int64_t lo[6], hi[6];
        TRY(sscg_halo_plan(c->nz_global, c->nranks, c->spr, c->rank, 0, lo));
        TRY(sscg_halo_plan(c->nz_global, c->nranks, c->spr, c->rank, L - 1, hi));
        c->peer_rank[0] = (lo[0] >= 0 && lo[0] != c->rank) ? (int)lo[0] : -1;
        c->peer_rank[1] = (hi[3] >= 0 && hi[3] != c->rank) ? (int)hi[3] : -1;
        if (c->peer_rank[0] >= 0) {
            tx.push_back({0, c->peer_rank[0]});
            rx.push_back({0, 0, c->peer_rank[0]});
        }
        if (c->peer_rank[1] >= 0) {
            tx.push_back({L - 1, c->peer_rank[1]});
            rx.push_back({L - 1, 1, c->peer_rank[1]});
        }
    } else if (c->nccl_self && L > 1) {
        for (int l = 0; l + 1 < L; ++l) {   // in order: slab l+1's to slab l, slab l's to slab l+1
            tx.push_back({l + 1, 0});
            rx.push_back({l, 1, 0});
            tx.push_back({l, 0});
            rx.push_back({l + 1, 0, 0});
        }
    }
    const size_t nb = sizeof(PeerInfo);
    std::vector<PeerInfo> hin(tx.size()), hout(rx.size());
    for (size_t i = 0; i < tx.size(); ++i) {
        const Slab &sl = c->slabs[tx[i].slab];
        PeerInfo &pi = hin[i];
        memset(&pi, 0, nb);
        CU(cudaIpcGetMemHandle(&pi.h, sl.Palloc));
        pi.off = (int64_t)(reinterpret_cast<char *>(sl.P) - reinterpret_cast<char *>(sl.Palloc));
        pi.vstride = g.vstride;
        pi.nzl = sl.nzl;
        pi.pid = (int32_t)getpid();
        pi.nonce = proc_nonce();
        pi.base = (uint64_t)(uintptr_t)sl.Palloc;
    }
    char *dbuf = nullptr;
    int *dok = nullptr;
    TRY(dalloc(c, &dbuf, (tx.size() + rx.size()) * nb + 1));
    TRY(dalloc(c, &dok, 1));
    if (!c->token) TRY(dalloc(c, &c->token, 3));
    if (!tx.empty()) CU(cudaMemcpyAsync(dbuf, hin.data(), tx.size() * nb, cudaMemcpyHostToDevice, c->stream));
    NC(ncclGroupStart());
    for (size_t i = 0; i < tx.size(); ++i) {
        NC(ncclSend(dbuf + i * nb, nb, ncclUint8, tx[i].peer, c->comm, c->stream));
        NC(ncclRecv(dbuf + (tx.size() + i) * nb, nb, ncclUint8, rx[i].peer, c->comm, c->stream));
    }
    NC(ncclGroupEnd());
    if (!rx.empty())
        CU(cudaMemcpyAsync(hout.data(), dbuf + tx.size() * nb, rx.size() * nb, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    std::vector<double *> ptr(rx.size());
    std::vector<int> remote(rx.size());
    int ok = 1;
    for (size_t i = 0; i < rx.size(); ++i) {
        bool rem = false;
        ptr[i] = peer_map(c, hout[i], &rem);
        remote[i] = rem;
        if (!ptr[i]) ok = 0;
    }
    CU(cudaMemcpyAsync(dok, &ok, sizeof ok, cudaMemcpyHostToDevice, c->stream));
    NC(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, c->comm, c->stream));
    CU(cudaMemcpyAsync(&ok, dok, sizeof ok, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    dfree(c, dbuf);
    dfree(c, dok);
    if (!ok) {   // every rank keeps the NCCL exchange
        for (void *p : c->ipc_open) cudaIpcCloseMemHandle(p);
        c->ipc_open.clear();
        return SSCG_OK;
    }
    for (size_t i = 0; i < rx.size(); ++i) {
        Slab &sl = c->slabs[rx[i].slab];
        const int d = rx[i].side;
        sl.nbP[d] = ptr[i];
        sl.nbvs[d] = hout[i].vstride;
        sl.nbnzl[d] = hout[i].nzl;
        sl.nb_remote[d] = remote[i];
    }
    c->peer_remote = !rx.empty();
    return SSCG_OK;
}

// the ordering step of the cross-rank peer-store halo: one double to and from
// every neighbour that was stored into (graph-captured like the exchange)
static sscg_status peer_token(sscg_ctx *c)
{
    if (!c->peer_remote) return SSCG_OK;
    TRY(prof_mark(c, SSCG_PROF_HALO, true));
    NC(ncclGroupStart());
    if (c->nranks > 1) {
        for (int d = 0; d < 2; ++d)
            if (c->peer_rank[d] >= 0) {
                NC(ncclSend(c->token, 1, ncclDouble, c->peer_rank[d], c->comm, c->stream));
                NC(ncclRecv(c->token + 1 + d, 1, ncclDouble, c->peer_rank[d], c->comm, c->stream));
            }
    } else {
        NC(ncclSend(c->token, 1, ncclDouble, 0, c->comm, c->stream));
        NC(ncclRecv(c->token + 1, 1, ncclDouble, 0, c->comm, c->stream));
    }
    NC(ncclGroupEnd());
    TRY(prof_mark(c, SSCG_PROF_HALO, false));
    return SSCG_OK;
}

// deep-halo triple of steps j..j+2 on every slab.  part 0: all planes (levels 1
// and 2 formed on the ghost planes of a side with a neighbour); part 1: the
// planes the next exchange sends (level 3 on [1, 4) and [nzl-2, nzl], levels 1
// and 2 on [1, 3) and [nzl-1, nzl]); part 2: the rest (level 3 [4, nzl-2),
// levels 1 and 2 [3, nzl-1))
static sscg_status launch_basis_triple_deep(sscg_ctx *c, int j, int part)
{
    const Geo &g = c->g;
    const int s = c->s;
    const bool wf = uses_wfree(c);
    for (auto &sl : c->slabs) {
        K1MArgs a{};
        const int n = sl.nzl;
        for (int l = 0; l < 3; ++l) {
            const int jl = j + l;
            a.w[l] = (!wf || jl == s - 1) ? sl.W + (int64_t)jl * g.vstride : nullptr;
            a.pn[l] = (jl + 1 <= s - 1) ? sl.P + (int64_t)(jl + 1) * g.vstride : nullptr;
            if (part == 0) {
                a.zb[l] = 1;
                a.ze[l] = n + 1;
            } else if (part == 1) {
                a.zb[l] = 1;
                a.ze[l] = (l == 2) ? 4 : 3;
                a.zb2[l] = (l == 2) ? n - 2 : n - 1;
                a.ze2[l] = n + 1;
            } else {
                a.zb[l] = (l == 2) ? 4 : 3;
                a.ze[l] = (l == 2) ? n - 2 : n - 1;
            }
        }
        if (part == 2) a.sm_cap = c->k1_sm_cap;
        if (part == 0 && uses_peer(c)) {
            const size_t l = &sl - c->slabs.data();
            (void)l;
            for (int v = 0; v < 2; ++v) {
                const int jv = j + 2 + v;   // p_{j+2}, p_{j+3}
                if (jv > s - 1) continue;
                if (sl.nbP[0]) a.peer_lo[v] = sl.nbP[0] + (int64_t)jv * sl.nbvs[0];
                if (sl.nbP[1]) a.peer_hi[v] = sl.nbP[1] + (int64_t)jv * sl.nbvs[1];
            }
            a.peer_nzl_lo = sl.nbnzl[0];
            a.peer_sys_fence = sl.nb_remote[0] || sl.nb_remote[1];
        }
        a.deep_lo = sl.has_lo;
        a.deep_hi = sl.has_hi;
        a.guard = g.guard;
        a.nzl = n;
        a.j = j;
        a.sigma = c->sigma;
        a.tmP = &sl.tmM3_P;
        a.tmM = &sl.tmM3_M;
        TRY(prof_mark(c, SSCG_PROF_BASIS, true));
        launch_k1m(g, a, c->theta, c->st, c->stream);
        TRY(prof_mark(c, SSCG_PROF_BASIS, false));
        ++c->launches;
    }
    return SSCG_OK;
}

// halo = false: all planes of a slab bounded by Dirichlet planes; true: the
// planes each level can form from p_j with its halo planes current (level 1
// [2, nzl) -- its planes 1 and nzl come from the boundary single step --,
// level 2 [2, nzl), level 3 [3, nzl-1)); the rest runs as single steps
// around the exchanges (enqueue_outer)
static sscg_status launch_basis_triple(sscg_ctx *c, int j, bool halo = false)
{
    const Geo &g = c->g;
    const int s = c->s;
    const bool wf = uses_wfree(c);
    for (auto &sl : c->slabs) {
        K1MArgs a{};
        for (int l = 0; l < 3; ++l) {
            const int jl = j + l;   // step of level l+1
            a.w[l] = (!wf || jl == s - 1) ? sl.W + (int64_t)jl * g.vstride : nullptr;
            a.pn[l] = (jl + 1 <= s - 1) ? sl.P + (int64_t)(jl + 1) * g.vstride : nullptr;
            a.zb[l] = halo ? (l == 2 ? 3 : 2) : 1;
            a.ze[l] = halo ? (l == 2 ? sl.nzl - 1 : sl.nzl) : sl.nzl + 1;
        }
        if (halo) a.sm_cap = c->k1_sm_cap;
        a.guard = g.guard;
        a.nzl = sl.nzl;
        a.j = j;
        a.sigma = c->sigma;
        a.tmP = &sl.tmM3_P;
        a.tmM = &sl.tmM3_M;
        TRY(prof_mark(c, SSCG_PROF_BASIS, true));
        launch_k1m(g, a, c->theta, c->st, c->stream);
        TRY(prof_mark(c, SSCG_PROF_BASIS, false));
        ++c->launches;
    }
    return SSCG_OK;
}

// K1F: basis steps j, j+1 in one launch per slab, over all planes (part 0,
// a slab bounded by the global Dirichlet planes) or the planes [2, nzl) that
// need no halo of p_{j+1} (part 2)
static sscg_status launch_basis_pair(sscg_ctx *c, int j, int part)
{
    const Geo &g = c->g;
    const int s = c->s;
    for (auto &sl : c->slabs) {
        K1Args a{};
        a.p = sl.P + (int64_t)j * g.vstride;
        a.pm = (j > 0) ? sl.P + (int64_t)(j - 1) * g.vstride : nullptr;
        a.w = sl.W + (int64_t)j * g.vstride;
        a.pn = sl.P + (int64_t)(j + 1) * g.vstride;
        a.w2 = sl.W + (int64_t)(j + 1) * g.vstride;
        a.pn2 = (j + 2 < s) ? sl.P + (int64_t)(j + 2) * g.vstride : nullptr;
        a.sigma = c->sigma;
        a.nzl = sl.nzl;
        a.skip_w = uses_wfree(c) ? 1 : 0;                         // j <= s-2 here
        a.skip_w2 = (uses_wfree(c) && j + 1 < s - 1) ? 1 : 0;
        a.zb = (part == 0) ? 1 : 2;
        a.ze = (part == 0) ? sl.nzl + 1 : sl.nzl;
        if (part == 2) a.sm_cap = c->k1_sm_cap;
        a.j = j;
        a.tmF_P = &sl.tmF_P;
        a.tmF_M = &sl.tmF_M;
        a.kx = sl.kx; a.ky = sl.ky; a.kz = sl.kz;
        a.tmKX = &sl.tmV_KX; a.tmKY = &sl.tmV_KY; a.tmKZ = &sl.tmV_KZ;
        a.kx_shift = sl.kx_shift;
        TRY(prof_mark(c, SSCG_PROF_BASIS, true));
        if (g.kind == SSCG_OP_VARCOEF7) launch_k1fv(g, a, c->theta, s, c->st, c->stream);
        else launch_k1f(g, a, c->theta, s, c->st, c->stream);
        TRY(prof_mark(c, SSCG_PROF_BASIS, false));
        ++c->launches;
    }
    return SSCG_OK;
}

// One outer iteration.  Precondition: the halo planes of p_0 are current.
//   for j: K1 boundary planes -> fork halo(p_{j+1}) -> K1 interior -> join
//   K2 (+ slab sum) -> allreduce -> K4 -> K5 boundary -> fork halo(p_0) -> K5 interior -> join
// the fold's diagonal entry p_{s-1}^T A p_{s-1} of one slab into its Gram block
// (after K2R): the TMA single step (K1T) in its dot mode -- it streams p_{s-1}
// as the single step it replaces did, stores nothing and reduces -- else k_pap
static void launch_pap_dot(sscg_ctx *c, const Slab &sl, double *blk)
{
    const Geo &g = c->g;
    const int s = c->s;
    K1Args a{};
    a.p = sl.P + (int64_t)(s - 1) * g.vstride;
    a.w = sl.W + (int64_t)(s - 1) * g.vstride;   // (not written: skip_w)
    a.dinv = sl.dinv;
    a.dinv_c = g.dinv_c;
    a.sigma = c->sigma;
    a.mode = 0;
    a.nzl = sl.nzl;
    a.j = s - 1;
    a.skip_w = 1;
    a.zb = 1;
    a.ze = sl.nzl + 1;
    if (sl.has_k1t) {
        a.tmP4 = &sl.tmP4;
        a.tmM4 = &sl.tmM4;
    }
    a.dot_part = sl.part;
    a.dot_ticket = sl.ticket;
    a.dot_entry = blk + (int64_t)(s - 1) * s + (s - 1);
    if (k1t_supported(g, a)) launch_k1(g, a, c->st, c->stream);
    else launch_pap(g, sl, s, c->st, blk, c->stream);
}

static sscg_status enqueue_outer(sscg_ctx *c, double *x)
{
    const Geo &g = c->g;
    const int s = c->s;
    const int L = (int)c->slabs.size();
    const bool halo = (L > 1 || c->nranks > 1) && g.kind != SSCG_OP_CSR;
    const bool ovl = halo && c->overlap;
    const bool fuse = uses_fused(c), mp3 = uses_mp3(c), deep = uses_deep(c);
    if (uses_small(c)) {   // the whole outer iteration in one launch (KS)
        K4Args a4{};
        a4.blk = c->blk;
        a4.alpha = c->alpha;
        a4.s = s;
        a4.nu = c->nu;
        a4.pdl = g.kn.pdl;
        a4.h_gram = c->h_gram; a4.h_d = c->h_d; a4.h_at = c->h_at; a4.h_al = c->h_al;
        a4.h_delta = c->h_delta; a4.h_relres = c->h_relres; a4.h_lnorm = c->h_lnorm;
        TRY(prof_mark(c, SSCG_PROF_BASIS, true));
        launch_ks(g, c->slabs[0], s, c->theta, c->sigma, c->xdev, c->blk, a4, c->st, c->stream);
        TRY(prof_mark(c, SSCG_PROF_BASIS, false));
        ++c->launches;
        CU(cudaGetLastError());
        return SSCG_OK;
    }
    // with the w_{s-1} fold the basis kernels stop at p_{s-1}: steps j < s_end
    const bool fold = uses_wlfold(c);
    const int s_end = fold ? s - 1 : s;
    bool pend_last = false;   // p_{s-1} produced by a single step whose exchange is still due (fold)
    nvtxRangePushA("basis");
    for (int j = 0; j < s_end; ++j) {
        if (mp3 && j + 2 < s_end) {   // steps j, j+1, j+2 in one pass (K1M)
            if (!halo) {
                TRY(launch_basis_triple(c, j));
            } else if (deep) {
                // p_j is current on 3 ghost planes, p_{j-1} on 2: the triple forms
                // levels 1 and 2 on the ghost planes itself.  Its outputs feed the next
                // triple (p_{j+3} on 3 planes, p_{j+2} on 2) or the remaining single /
                // paired steps (p_{j+3} on 1 plane): one exchange after the triple.
                // SSCG_DEEP_OVERLAP=1: the planes the exchange sends go first and the
                // exchange overlaps the rest of the triple (an extra launch per triple;
                // measured slower on one GPU, tools/slab_overhead.py)
                const bool next3 = j + 5 < s_end;
                const int np3 = (j + 3 < s) ? (next3 ? 3 : 1) : 0, np2 = next3 ? 2 : 0;
                if (ovl && np3 > 0 && g.kn.deep_overlap) {
                    TRY(launch_basis_triple_deep(c, j, 1));
                    TRY(halo_fork(c, j + 3, true, np3, j + 2, np2));
                    TRY(launch_basis_triple_deep(c, j, 2));
                    TRY(halo_join(c));
                } else {
                    TRY(launch_basis_triple_deep(c, j, 0));
                    if (np3 > 0 && !uses_peer(c)) TRY(halo_fork(c, j + 3, false, np3, j + 2, np2));
                    if (np3 > 0 && uses_peer(c)) TRY(peer_token(c));
                }
            } else {
                // boundary planes of step j, exchange of p_{j+1} (overlapped with the
                // interior triple), boundary planes of step j+1, exchange of p_{j+2},
                // the two planes next to each boundary of step j+2, exchange of p_{j+3}
                TRY(launch_basis(c, j, 1));
                TRY(halo_fork(c, j + 1, ovl));
                TRY(launch_basis_triple(c, j, true));
                if (ovl) TRY(halo_join(c));
                TRY(launch_basis(c, j + 1, 1));
                TRY(halo_fork(c, j + 2, false));
                TRY(launch_basis(c, j + 2, 3));
                if (j + 3 < s) TRY(halo_fork(c, j + 3, false));
            }
            j += 2;
        } else if (fuse && j + 1 < s_end) {   // steps j and j+1 in one pass (K1F)
            if (!halo) {
                TRY(launch_basis_pair(c, j, 0));
            } else {
                // boundary planes of step j, exchange of p_{j+1} (overlapped with
                // the interior pair), boundary planes of step j+1, exchange of p_{j+2}
                TRY(launch_basis(c, j, 1));
                TRY(halo_fork(c, j + 1, ovl));
                TRY(launch_basis_pair(c, j, 2));
                if (ovl) TRY(halo_join(c));
                TRY(launch_basis(c, j + 1, 1));
                if (j + 2 < s) TRY(halo_fork(c, j + 2, false));
            }
            ++j;
        } else if (!halo) {
            TRY(launch_basis(c, j, 0));
        } else if (!ovl) {
            if (j > 0) TRY(halo_fork(c, j, false));
            TRY(launch_basis(c, j, 0));
            pend_last = j == s_end - 1;
        } else {
            TRY(launch_basis(c, j, 1));
            if (j < s - 1) TRY(halo_fork(c, j + 1, true));
            TRY(launch_basis(c, j, 2));
            if (j < s - 1) TRY(halo_join(c));
        }
    }
    if (fold && halo && pend_last) TRY(halo_fork(c, s - 1, false));   // K2R / K5 read p_{s-1}'s ghost planes
    nvtxRangePop();
    nvtxRangePushA("gram+allreduce+fgs");
    const bool wfree = uses_wfree(c);
    K4Args a4{};
    a4.blk = c->blk;
    a4.alpha = c->alpha;
    a4.s = s;
    a4.nu = c->nu;
    a4.solver = (c->gram_solver == SSCG_GRAM_CHOLESKY) ? 1 : 0;
    a4.pdl = g.kn.pdl;
    a4.h_gram = c->h_gram; a4.h_d = c->h_d; a4.h_at = c->h_at; a4.h_al = c->h_al;
    a4.h_delta = c->h_delta; a4.h_relres = c->h_relres; a4.h_lnorm = c->h_lnorm;
    // block-conjugate mode: the Gram pass runs over the 2s rows [P_k | Q'] x [W_k | Z']
    const int rows = c->blockcg ? 2 * s : s, nent = rows * rows + rows;
    for (auto &sl : c->slabs) {
        TRY(prof_mark(c, SSCG_PROF_GRAM, true));
        if (wfree && c->blockcg) launch_k2r_block(g, sl, s, c->theta, c->sigma, c->st, L == 1 ? c->blk : sl.blk, c->stream);
        else if (wfree) launch_k2r(g, sl, s, c->theta, c->sigma, c->st, L == 1 ? c->blk : sl.blk, c->stream, fold);
        else launch_k2(g, sl, rows, c->st, L == 1 ? c->blk : sl.blk, c->stream);
        ++c->launches;
        if (fold) {   // Ghat_{s-1,s-1} = p_{s-1}^T A p_{s-1}
            launch_pap_dot(c, sl, L == 1 ? c->blk : sl.blk);
            ++c->launches;
        }
        TRY(prof_mark(c, SSCG_PROF_GRAM, false));
    }
    if (L > 1) {
        TRY(prof_mark(c, SSCG_PROF_GRAM, true));
        launch_slab_sum(c->blkptrs, L, nent, c->blk, c->st, c->stream);
        TRY(prof_mark(c, SSCG_PROF_GRAM, false));
        ++c->launches;
    }
    if (c->comm) {   // ranks (or the SSCG_NCCL_SELF test mode): the one allreduce of the outer iteration
        TRY(prof_mark(c, SSCG_PROF_ALLREDUCE, true));
        NC(ncclAllReduce(c->blk, c->blk, (size_t)nent, ncclDouble, ncclSum, c->comm, c->stream));
        TRY(prof_mark(c, SSCG_PROF_ALLREDUCE, false));
        ++c->allreduces;
    }
    if (c->blockcg) {   // B_k, then K4 on the conjugated system; the stopping test reads ||r_k||^2 of the raw block
        TRY(prof_mark(c, SSCG_PROF_FGS, true));
        launch_bcg_prep(c->blk, s, c->blk2, c->bmat, c->st, g.kn.pdl, c->stream);
        TRY(prof_mark(c, SSCG_PROF_FGS, false));
        ++c->launches;
        a4.blk = c->blk2;
        a4.rn2 = c->blk + (int64_t)rows * rows;
    }
    TRY(prof_mark(c, SSCG_PROF_FGS, true));
    launch_k4(a4, c->st, c->stream);
    if (c->diagnostics) {
        launch_kappa(a4.blk, s, c->st, c->h_kappa, c->stream);
        ++c->launches;
        for (int l = 0; l < L; ++l) {   // ||P_k||_F before K5 overwrites p_0
            launch_pnorm(g, c->slabs[l], s, c->diag_part + (size_t)l * DIAG_BLK, DIAG_BLK, c->st, c->stream);
            ++c->launches;
        }
        launch_budget(c->diag_part, L * DIAG_BLK, c->diag_sum, c->anorm, false, c->st, c->h_delta, c->h_pnorm,
                      c->h_budget, c->stream, 0);
        if (c->comm) NC(ncclAllReduce(c->diag_sum, c->diag_sum, 1, ncclDouble, ncclSum, c->comm, c->stream));
        launch_budget(c->diag_part, L * DIAG_BLK, c->diag_sum, c->anorm, false, c->st, c->h_delta, c->h_pnorm,
                      c->h_budget, c->stream, 1);
        c->launches += 2;
    }
    TRY(prof_mark(c, SSCG_PROF_FGS, false));
    ++c->launches;
    nvtxRangePop();
    nvtxRangePushA("update");
    auto k5 = [&](int zb, int ze) -> sscg_status {
        for (auto &sl : c->slabs) {
            const int e = (ze < 0) ? sl.nzl + 2 + ze : std::min(ze, sl.nzl + 1);   // ze = -m: nzl + 2 - m
            const int b = std::max(zb, 1);
            if (e <= b) continue;
            TRY(prof_mark(c, SSCG_PROF_UPDATE, true));
            if (c->blockcg)
                launch_k5_block(g, sl, s, c->alpha, c->bmat, c->xdev, sl.zoff * (int64_t)g.nx * g.ny, c->st, c->stream,
                                b, e, wfree, c->theta, c->sigma);
            else
                launch_k5(g, sl, s, c->alpha, c->xdev, sl.zoff * (int64_t)g.nx * g.ny, c->st, c->stream, b, e,
                          c->theta, c->sigma, uses_rec_update(c), uses_k5fold(c));
            TRY(prof_mark(c, SSCG_PROF_UPDATE, false));
            ++c->launches;
        }
        return SSCG_OK;
    };
    // r_{k+1} = p_0 of the next outer needs 3 ghost planes for a deep-halo triple
    const int np0 = deep ? 3 : 1;
    if (!halo) {
        TRY(k5(1, -1));
    } else if (!ovl || (deep && !g.kn.deep_overlap) || c->blockcg) {
        TRY(k5(1, -1));
        TRY(halo_fork(c, 0, false, np0));
    } else {
        // boundary planes of r_{k+1} first, their exchange overlapping the
        // interior update
        for (auto &sl : c->slabs) {
            const int top = std::max(1 + np0, sl.nzl - np0 + 1);
            for (int zb : {1, top}) {
                const int ze = std::min(zb + np0, sl.nzl + 1);
                if (zb >= ze) continue;
                TRY(prof_mark(c, SSCG_PROF_UPDATE, true));
                launch_k5(g, sl, s, c->alpha, c->xdev, sl.zoff * (int64_t)g.nx * g.ny, c->st, c->stream, zb, ze,
                          c->theta, c->sigma, uses_rec_update(c), uses_k5fold(c));
                TRY(prof_mark(c, SSCG_PROF_UPDATE, false));
                ++c->launches;
            }
        }
        TRY(halo_fork(c, 0, true, np0));
        TRY(k5(1 + np0, -(1 + np0)));
        TRY(halo_join(c));
    }
    nvtxRangePop();
    CU(cudaGetLastError());
    return SSCG_OK;
}

// One outer iteration as a CUDA graph (captured once per x pointer): the
// s + 3 launches (+ NCCL calls) replay with one cudaGraphLaunch, which removes
// the per-kernel host launch cost that dominates small problems (cfg 1/2).
// Profiling runs use plain launches so every kernel can be bracketed.
static sscg_status run_outer(sscg_ctx *c, double *x)
{
    if (c->prof_on || !c->use_graph) return enqueue_outer(c, x);
    if (!c->gexec) {
        if (c->gexec) {
            cudaGraphExecDestroy(c->gexec);
            c->gexec = nullptr;
        }
        const int64_t l0 = c->launches, a0 = c->allreduces;
        cudaGraph_t graph = nullptr;
        CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
        const sscg_status st = enqueue_outer(c, x);
        const cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
        if (st != SSCG_OK) {
            if (graph) cudaGraphDestroy(graph);
            return st;
        }
        if (e != cudaSuccess) return fail(SSCG_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
        const cudaError_t e2 = cudaGraphInstantiate(&c->gexec, graph, 0);
        cudaGraphDestroy(graph);
        if (e2 != cudaSuccess) {
            c->gexec = nullptr;
            return fail(SSCG_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(e2));
        }
        c->graph_launches = c->launches - l0;
        c->graph_allreduces = c->allreduces - a0;
        c->launches = l0;
        c->allreduces = a0;
    }
    CU(cudaGraphLaunch(c->gexec, c->stream));
    c->launches += c->graph_launches;
    c->allreduces += c->graph_allreduces;
    return SSCG_OK;
}

// free a device buffer allocated by dalloc (and forget it)
static void dfree(sscg_ctx *c, void *p)
{
    if (!p) return;
    for (auto &q : c->allocs)
        if (q == p) {
            cudaFree(q);
            q = c->allocs.back();
            c->allocs.pop_back();
            return;
        }
}

static sscg_status ensure_history(sscg_ctx *c, int cap)
{
    if (cap <= c->hist_cap) return SSCG_OK;
    cap = std::max(cap, std::min(2 * c->hist_cap, 1 << 20));   // grow geometrically
    CU(cudaStreamSynchronize(c->stream));                       // old buffers may still be written
    if (c->gexec) {   // the captured K4 holds the old history pointers
        cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
    }
    const int s = c->s, nent = s * s + s;
    // per-outer vector records (Gram block, d, alpha~, alpha) are kept for the
    // first GRAM_HIST outer iterations only: s = 64 would need 33 GB for 2^20
    const int gcap = std::min(cap, GRAM_HIST);
    if (gcap > c->gram_cap) {
        for (double *q : {c->h_gram, c->h_d, c->h_at, c->h_al}) dfree(c, q);
        TRY(dalloc(c, &c->h_gram, (size_t)gcap * nent));
        TRY(dalloc(c, &c->h_d, (size_t)gcap * s));
        TRY(dalloc(c, &c->h_at, (size_t)gcap * s));
        TRY(dalloc(c, &c->h_al, (size_t)gcap * s));
        c->gram_cap = gcap;
    }
    for (double *q : {c->h_delta, c->h_lnorm, c->h_kappa, c->h_pnorm, c->h_budget, c->h_relres}) dfree(c, q);
    TRY(dalloc(c, &c->h_delta, (size_t)cap));
    TRY(dalloc(c, &c->h_lnorm, (size_t)cap));
    TRY(dalloc(c, &c->h_kappa, (size_t)cap));
    TRY(dalloc(c, &c->h_pnorm, (size_t)cap));
    TRY(dalloc(c, &c->h_budget, (size_t)cap));
    CU(cudaMemset(c->h_kappa, 0, (size_t)cap * sizeof(double)));
    CU(cudaMemset(c->h_pnorm, 0, (size_t)cap * sizeof(double)));
    CU(cudaMemset(c->h_budget, 0, (size_t)cap * sizeof(double)));
    TRY(dalloc(c, &c->h_relres, (size_t)cap));
    c->hist_cap = cap;
    return SSCG_OK;
}

extern "C" sscg_status sscg_solve(sscg_ctx *c, const double *b, double *x, double rtol, int32_t max_outer,
                                  uint32_t flags)
{
    if (!c || !b || !x) return fail(SSCG_ERR_INVALID, "null argument");
    if (c->failed) return fail(SSCG_ERR_NCCL, "context unusable after an NCCL abort; destroy it");
    if (max_outer < 0 || !(rtol >= 0.0)) return fail(SSCG_ERR_INVALID, "bad rtol/max_outer");
    if (!c->bounds_set && c->basis == SSCG_BASIS_CHEBYSHEV)
        return fail(SSCG_ERR_INVALID, "spectral bounds not set (sscg_set_bounds / sscg_estimate_bounds)");
    const Geo &g = c->g;
    const int cap = std::min(max_outer + 1, 1 << 20);
    TRY(ensure_history(c, cap));
    c->launches = 0;
    c->allreduces = 0;
    c->last_max_outer = max_outer;
    DevState h{};
    h.hist_cap = c->hist_cap;
    h.gram_cap = c->gram_cap;
    h.rtol = rtol;
    h.max_outer = max_outer;
    *c->st_host = h;
    CU(cudaEventRecord(c->ev0, c->stream));
    CU(cudaMemcpyAsync(c->st, c->st_host, sizeof(DevState), cudaMemcpyHostToDevice, c->stream));
    *c->xhost = x;   // K5 reads x through this cell: the captured outer iteration serves any x
    CU(cudaMemcpyAsync(c->xdev, c->xhost, sizeof(double *), cudaMemcpyHostToDevice, c->stream));
    const int L = (int)c->slabs.size();
    // r_0 = b - A x_0 into p_0
    if (flags & SSCG_SOLVE_X0_ZERO) {
        CU(cudaMemsetAsync(x, 0, (size_t)c->n_local * sizeof(double), c->stream));
        for (auto &sl : c->slabs) {
            launch_pack(g, b + sl.zoff * (int64_t)g.nx * g.ny, sl.P, sl.nzl, nullptr, c->stream);
            ++c->launches;
        }
    } else {
        std::vector<double *> w0(L);
        for (int l = 0; l < L; ++l) {
            auto &sl = c->slabs[l];
            launch_pack(g, x + sl.zoff * (int64_t)g.nx * g.ny, sl.W, sl.nzl, nullptr, c->stream);
            ++c->launches;
            w0[l] = sl.W;
        }
        TRY(exchange(c, w0.data(), c->stream));
        for (auto &sl : c->slabs) {
            K1Args a{};
            a.p = sl.W;
            a.w = sl.P;
            a.b = b + sl.zoff * (int64_t)g.nx * g.ny;
            a.kx = sl.kx; a.ky = sl.ky; a.kz = sl.kz;
            a.dinv = sl.dinv;
            a.dinv_c = g.dinv_c;
            a.mode = 3;
            a.zb = 1;
            a.ze = sl.nzl + 1;
            a.nzl = sl.nzl;
            launch_k1(g, a, nullptr, c->stream);
            ++c->launches;
        }
    }
    nvtxRangePushA("sscg_solve");
    // halo planes of p_0 = r_0 (enqueue_outer's precondition)
    if ((L > 1 || c->nranks > 1) && g.kind != SSCG_OP_CSR) TRY(halo_fork(c, 0, false, uses_deep(c) ? 3 : 1));
    // outer iterations in chunks; the device decides when to stop
    int issued = 0;
    int chunk = 2;
    while (issued < max_outer + 1) {
        const int n = std::min(chunk, max_outer + 1 - issued);
        for (int i = 0; i < n; ++i) {
            TRY(run_outer(c, x));
            if (c->x_host_out && issued + i + 1 == max_outer) {
                // x is final after the max_outer-th update: copy it out (sscg_solve_host)
                // while the last outer iteration only builds the basis/Gram of the stopping test
                CU(cudaEventRecord(c->ev_xready, c->stream));
                CU(cudaStreamWaitEvent(c->cstream, c->ev_xready, 0));
                CU(cudaMemcpyAsync(c->x_host_out, x, (size_t)c->n_local * sizeof(double), cudaMemcpyDeviceToHost,
                                   c->cstream));
                c->x_copied = true;
            }
        }
        issued += n;
        CU(cudaMemcpyAsync(c->st_host, c->st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
        TRY(wait_stream(c, c->stream));
        if (c->st_host->done) break;
        chunk = std::min(chunk * 2, 16);
    }
    CU(cudaEventRecord(c->ev1, c->stream));
    CU(cudaMemcpyAsync(c->st_host, c->st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
    TRY(wait_stream(c, c->stream));
    if (c->x_copied) CU(cudaStreamSynchronize(c->cstream));
    nvtxRangePop();
    const DevState &f = *c->st_host;
    const int outer = f.outer;
    c->relres_host.assign((size_t)std::min(outer + 1, c->hist_cap), 0.0);
    c->delta_host.assign((size_t)std::min(outer, c->hist_cap), 0.0);
    if (!c->relres_host.empty())
        CU(cudaMemcpy(c->relres_host.data(), c->h_relres, c->relres_host.size() * sizeof(double),
                      cudaMemcpyDeviceToHost));
    if (!c->delta_host.empty())
        CU(cudaMemcpy(c->delta_host.data(), c->h_delta, c->delta_host.size() * sizeof(double),
                      cudaMemcpyDeviceToHost));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    sscg_stats_t &S = c->stats;
    S = sscg_stats_t{};
    S.outer_iterations = outer;
    S.converged = f.converged;
    S.breakdown = f.breakdown;
    S.nonfinite = f.nonfinite;
    S.r0_norm = f.r0norm;
    S.history_len = (int32_t)c->relres_host.size();
    S.relres_final = c->relres_host.empty() ? 0.0 : c->relres_host.back();
    S.relres_history = c->relres_host.data();
    S.delta_history = c->delta_host.data();
    S.ms_total = ms;
    S.kernel_launches = c->launches;
    S.allreduces = c->allreduces;
    S.budget = 0.0;
    if (c->diagnostics && outer > 0) {   // sum_k delta_k ||A|| ||P_k||_F over the applied updates
        std::vector<double> bt((size_t)std::min(outer, c->hist_cap));
        CU(cudaMemcpy(bt.data(), c->h_budget, bt.size() * sizeof(double), cudaMemcpyDeviceToHost));
        for (double v : bt) S.budget += v;
    }
    c->solved = true;
    TRY(prof_resolve(c));
    if (f.breakdown) return fail(SSCG_ERR_BREAKDOWN, "Gram breakdown at outer %d (Ghat_ii <= 0 or non-finite)", outer);
    if (f.nonfinite) return fail(SSCG_ERR_NONFINITE, "non-finite residual at outer %d", outer);
    g_err.clear();
    return SSCG_OK;
}

extern "C" sscg_status sscg_solve_host(sscg_ctx *c, const double *b_host, double *x_host, double rtol,
                                       int32_t max_outer, uint32_t flags)
{
    if (!c || !b_host || !x_host) return fail(SSCG_ERR_INVALID, "null argument");
    if (c->failed) return fail(SSCG_ERR_NCCL, "context unusable after an NCCL abort; destroy it");
    const size_t bytes = (size_t)c->n_local * sizeof(double);
    if (!c->bbuf) TRY(dalloc(c, &c->bbuf, (size_t)c->n_local));
    if (!c->xbuf) TRY(dalloc(c, &c->xbuf, (size_t)c->n_local));
    CU(cudaMemcpyAsync(c->bbuf, b_host, bytes, cudaMemcpyHostToDevice, c->stream));
    if (!(flags & SSCG_SOLVE_X0_ZERO)) CU(cudaMemcpyAsync(c->xbuf, x_host, bytes, cudaMemcpyHostToDevice, c->stream));
    // the early copy of x (overlapping the last stopping-test iteration) needs
    // page-locked memory; a pageable x_host is copied after the solve instead
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, x_host) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    c->x_host_out = pinned ? x_host : nullptr;
    c->x_copied = false;
    sscg_status st = sscg_solve(c, c->bbuf, c->xbuf, rtol, max_outer, flags);
    c->x_host_out = nullptr;
    if (st != SSCG_OK && st != SSCG_ERR_BREAKDOWN && st != SSCG_ERR_NONFINITE) return st;
    std::string keep = g_err;
    if (!c->x_copied) {   // converged (or stopped) before max_outer updates: copy now
        CU(cudaMemcpyAsync(x_host, c->xbuf, bytes, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
    }
    c->x_copied = false;
    g_err = keep;
    return st;
}

extern "C" sscg_status sscg_stats(const sscg_ctx *c, sscg_stats_t *out)
{
    if (!c || !out) return fail(SSCG_ERR_INVALID, "null argument");
    *out = c->stats;
    return SSCG_OK;
}

extern "C" sscg_status sscg_local_shape(const sscg_ctx *c, int64_t *z0, int64_t *nz_proc, int64_t *n_local)
{
    if (!c) return fail(SSCG_ERR_INVALID, "null ctx");
    if (z0) *z0 = c->z0_proc;
    if (nz_proc) *nz_proc = c->nzl_proc;
    if (n_local) *n_local = c->n_local;
    return SSCG_OK;
}

extern "C" sscg_status sscg_inspect(const sscg_ctx *cc, int32_t what, int32_t index, void *host_out,
                                    int64_t capacity)
{
    sscg_ctx *c = const_cast<sscg_ctx *>(cc);
    if (!c || !host_out) return fail(SSCG_ERR_INVALID, "null argument");
    const Geo &g = c->g;
    const int s = c->s, nent = s * s + s;
    CU(cudaStreamSynchronize(c->stream));
    auto need = [&](int64_t bytes) { return capacity >= bytes; };
    if (what == SSCG_INSPECT_P || what == SSCG_INSPECT_W) {
        if (index < 0 || index >= s) return fail(SSCG_ERR_INVALID, "column %d out of range", index);
        if (!need(c->n_local * 8)) return fail(SSCG_ERR_INVALID, "buffer too small");
        if (what == SSCG_INSPECT_W && index == s - 1 && uses_wlfold(c))   // not stored (fold): w_{s-1} = A p_{s-1}
            TRY(launch_basis(c, s - 1, 0, true));
        for (auto &sl : c->slabs) {
            double *v = (what == SSCG_INSPECT_P ? sl.P : sl.W) + (int64_t)index * g.vstride;
            if (what == SSCG_INSPECT_W && uses_wfree(c) && index < s - 1)   // not stored: recover it (R23)
                launch_wrec(g, sl, index, c->theta, c->sigma, v, c->stream);
            launch_unpack(g, v, c->scratch + sl.zoff * (int64_t)g.nx * g.ny, sl.nzl, c->stream);
        }
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(host_out, c->scratch, (size_t)c->n_local * 8, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        return SSCG_OK;
    }
    if (index < 0 || index >= c->hist_cap || index > c->last_max_outer)
        return fail(SSCG_ERR_INVALID, "history index %d out of range", index);
    if ((what == SSCG_INSPECT_GRAM || what == SSCG_INSPECT_D || what == SSCG_INSPECT_ALPHA_T ||
         what == SSCG_INSPECT_ALPHA) && index >= c->gram_cap)
        return fail(SSCG_ERR_INVALID, "outer %d: Gram/alpha records are kept for the first %d outer iterations",
                    index, c->gram_cap);
    const double *src = nullptr;
    int64_t cnt = 0;
    switch (what) {
    case SSCG_INSPECT_GRAM: src = c->h_gram + (int64_t)index * nent; cnt = nent; break;
    case SSCG_INSPECT_D: src = c->h_d + (int64_t)index * s; cnt = s; break;
    case SSCG_INSPECT_ALPHA_T: src = c->h_at + (int64_t)index * s; cnt = s; break;
    case SSCG_INSPECT_ALPHA: src = c->h_al + (int64_t)index * s; cnt = s; break;
    case SSCG_INSPECT_DELTA: src = c->h_delta + index; cnt = 1; break;
    case SSCG_INSPECT_LNORM: src = c->h_lnorm + index; cnt = 1; break;
    case SSCG_INSPECT_KAPPA: src = c->h_kappa + index; cnt = 1; break;
    case SSCG_INSPECT_PNORM: src = c->h_pnorm + index; cnt = 1; break;
    case SSCG_INSPECT_BUDGET: src = c->h_budget + index; cnt = 1; break;
    default: return fail(SSCG_ERR_INVALID, "unknown inspect target %d", what);
    }
    if (!need(cnt * 8)) return fail(SSCG_ERR_INVALID, "buffer too small");
    CU(cudaMemcpy(host_out, src, (size_t)cnt * 8, cudaMemcpyDeviceToHost));
    return SSCG_OK;
}

extern "C" sscg_status sscg_iterate(sscg_ctx *c, double *x, int32_t nsteps)
{
    if (!c || !x || nsteps < 0) return fail(SSCG_ERR_INVALID, "bad argument");
    if (c->failed) return fail(SSCG_ERR_NCCL, "context unusable after an NCCL abort; destroy it");
    if (!c->solved) return fail(SSCG_ERR_INVALID, "sscg_iterate needs a preceding sscg_solve");
    if (c->st_host->breakdown || c->st_host->nonfinite) return fail(SSCG_ERR_INVALID, "last solve broke down");
    c->launches = 0;
    c->allreduces = 0;
    DevState h = *c->st_host;
    h.done = 0;
    h.converged = 0;
    h.rtol = 0.0;
    h.max_outer = 0x3fffffff;
    *c->st_host = h;
    CU(cudaEventRecord(c->ev0, c->stream));
    CU(cudaMemcpyAsync(c->st, c->st_host, sizeof(DevState), cudaMemcpyHostToDevice, c->stream));
    *c->xhost = x;
    CU(cudaMemcpyAsync(c->xdev, c->xhost, sizeof(double *), cudaMemcpyHostToDevice, c->stream));
    nvtxRangePushA("sscg_iterate");
    for (int i = 0; i < nsteps; ++i) TRY(run_outer(c, x));
    CU(cudaEventRecord(c->ev1, c->stream));
    CU(cudaMemcpyAsync(c->st_host, c->st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
    TRY(wait_stream(c, c->stream));
    nvtxRangePop();
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    c->stats.ms_total = ms;
    c->stats.kernel_launches = c->launches;
    c->stats.allreduces = c->allreduces;
    c->stats.outer_iterations = c->st_host->outer;
    c->stats.history_len = 0;
    c->stats.relres_history = nullptr;
    c->stats.delta_history = nullptr;
    TRY(prof_resolve(c));
    if (c->st_host->breakdown) return fail(SSCG_ERR_BREAKDOWN, "Gram breakdown during sscg_iterate");
    if (c->st_host->nonfinite) return fail(SSCG_ERR_NONFINITE, "non-finite residual during sscg_iterate");
    return SSCG_OK;
}

extern "C" sscg_status sscg_set_profiling(sscg_ctx *c, int32_t on)
{
    if (!c) return fail(SSCG_ERR_INVALID, "null ctx");
    TRY(prof_resolve(c));
    c->prof_on = on != 0;
    c->prof = sscg_profile_t{};
    return SSCG_OK;
}

extern "C" sscg_status sscg_profile(sscg_ctx *c, sscg_profile_t *out)
{
    if (!c || !out) return fail(SSCG_ERR_INVALID, "null argument");
    TRY(prof_resolve(c));
    *out = c->prof;
    return SSCG_OK;
}

extern "C" sscg_status sscg_set_bounds(sscg_ctx *c, double lambda_min, double lambda_max)
{
    if (!c) return fail(SSCG_ERR_INVALID, "null ctx");
    if (!(lambda_min > 0.0) || !(lambda_max > lambda_min) || !std::isfinite(lambda_max))
        return fail(SSCG_ERR_INVALID, "need 0 < lambda_min < lambda_max (got %g, %g)", lambda_min, lambda_max);
    c->lmin = lambda_min;
    c->lmax = lambda_max;
    c->theta = 2.0 / (lambda_max - lambda_min);
    c->sigma = (lambda_max + lambda_min) / 2.0;
    c->bounds_set = true;
    drop_graph(c);                                // the captured K1 launches hold theta, sigma
    return SSCG_OK;
}

extern "C" sscg_status sscg_set_option(sscg_ctx *c, int32_t key, int32_t value)
{
    if (!c) return fail(SSCG_ERR_INVALID, "null ctx");
    switch (key) {
    case SSCG_OPT_GRAM_SOLVER:
        if (value != SSCG_GRAM_FGS && value != SSCG_GRAM_CHOLESKY) return fail(SSCG_ERR_INVALID, "bad Gram solver %d", value);
        c->gram_solver = value;
        break;
    case SSCG_OPT_DIAGNOSTICS:
        if (value != 0 && value != 1) return fail(SSCG_ERR_INVALID, "bad diagnostics flag %d", value);
        c->diagnostics = value == 1;
        if (c->diagnostics && !c->diag_part) {
            const int L = (int)c->slabs.size();
            TRY(dalloc(c, &c->diag_part, (size_t)L * DIAG_BLK));
            TRY(dalloc(c, &c->diag_sum, 1));
            // ||A|| (Gershgorin, max row sum of |A_ij|) over every slab and rank, once
            double *bmax = c->diag_part;
            double mx = 0.0;
            std::vector<double> h(DIAG_BLK);
            for (int l = 0; l < L; ++l) {
                launch_anorm(c->g, c->slabs[l], bmax, DIAG_BLK, c->stream);
                CU(cudaGetLastError());
                CU(cudaMemcpyAsync(h.data(), bmax, DIAG_BLK * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
                CU(cudaStreamSynchronize(c->stream));
                for (double v : h) mx = std::max(mx, v);
            }
            if (c->comm) {
                CU(cudaMemcpyAsync(c->diag_sum, &mx, sizeof(double), cudaMemcpyHostToDevice, c->stream));
                NC(ncclAllReduce(c->diag_sum, c->diag_sum, 1, ncclDouble, ncclMax, c->comm, c->stream));
                CU(cudaMemcpyAsync(&mx, c->diag_sum, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
                CU(cudaStreamSynchronize(c->stream));
            }
            c->anorm = mx;
        }
        break;
    case SSCG_OPT_BASIS:
        if (value != SSCG_BASIS_CHEBYSHEV && value != SSCG_BASIS_MONOMIAL) return fail(SSCG_ERR_INVALID, "bad basis %d", value);
        c->basis = value;
        break;
    case SSCG_OPT_BLOCKCG:
        if (value != 0 && value != 1) return fail(SSCG_ERR_INVALID, "bad block-conjugate flag %d", value);
        if (value == 1 && c->s > 32) return fail(SSCG_ERR_INVALID, "block-conjugate mode needs s <= 32 (s = %d)", c->s);
        if ((value == 1) != c->blockcg) {
            // the store holds [P | Q'] and [W | Z'] (2s vectors) in the block mode
            drop_graph(c);
            TRY(build_basis_store(c, value ? 2 * c->s : c->s));
            TRY(setup_peers(c));   // the neighbours' new stores (collective across ranks, like the option)
            TRY(alloc_gram_buffers(c, value ? 2 * c->s : c->s));
            if (value && !c->blk2) {
                TRY(dalloc(c, &c->blk2, (size_t)c->s * c->s + c->s));
                TRY(dalloc(c, &c->bmat, (size_t)c->s * c->s));
            }
            c->blockcg = value == 1;
            c->solved = false;
        }
        break;
    default:
        return fail(SSCG_ERR_INVALID, "unknown option %d", key);
    }
    drop_graph(c);
    return SSCG_OK;
}

// Lanczos on D^{-1/2} A D^{-1/2} (k_lanczos.cu; BASELINE cfg 3/4)
extern "C" sscg_status sscg_estimate_bounds(sscg_ctx *c, const double *v0, int32_t iters, double margin,
                                            double *lmin, double *lmax, double *alpha_out, double *beta_out)
{
    if (!c || !v0 || !lmin || !lmax) return fail(SSCG_ERR_INVALID, "null argument");
    if (c->failed) return fail(SSCG_ERR_NCCL, "context unusable after an NCCL abort; destroy it");
    if (iters < 1 || iters > 100000 || !(margin >= 0.0) || !(margin < 1.0))
        return fail(SSCG_ERR_INVALID, "bad iters (%d) or margin (%g)", iters, margin);
    const Geo &g = c->g;
    const int L = (int)c->slabs.size();
    cudaStream_t st = c->stream;
    if (c->lz_vec.empty()) {
        c->lz_vec.assign((size_t)L * 5, nullptr);
        for (int l = 0; l < L; ++l)
            for (int q = 0; q < 5; ++q) TRY(dalloc(c, &c->lz_vec[(size_t)l * 5 + q], (size_t)g.vstride));
        TRY(dalloc(c, &c->lz_part, (size_t)L * lz_grid()));
        TRY(dalloc(c, &c->lz_ticket, (size_t)L));
        TRY(dalloc(c, &c->lz_flags, 2));
    }
    if (iters > c->lz_iters) {
        TRY(dalloc(c, &c->lz_scal, (size_t)(16 + L + 2 * iters)));
        c->lz_iters = iters;
    }
    // scalars: 0 ||v0||^2, 1 a_k, 2 b_k^2, 3 b_{k-1}, 4-5 bounds, 16.. per-slab values, then alpha, beta
    double *S = c->lz_scal, *slabv = S + 16, *alpha = S + 16 + L, *beta = alpha + iters;
    CU(cudaMemsetAsync(S, 0, (size_t)(16 + L + 2 * iters) * sizeof(double), st));
    CU(cudaMemsetAsync(c->lz_flags, 0, 2 * sizeof(int), st));
    CU(cudaMemsetAsync(c->lz_ticket, 0, (size_t)L * sizeof(unsigned), st));
    auto vec = [&](int l, int q) { return c->lz_vec[(size_t)l * 5 + q]; };
    for (int l = 0; l < L; ++l) {
        for (int q = 0; q < 4; ++q) CU(cudaMemsetAsync(vec(l, q), 0, (size_t)g.vstride * sizeof(double), st));
        // D = diag(M) in the padded layout, 0 in pad columns and halos
        double *D = vec(l, 4);
        CU(cudaMemsetAsync(D, 0, (size_t)g.vstride * sizeof(double), st));
        lz_diag(g, c->slabs[l], D, st);
    }
    CU(cudaGetLastError());
    const int *stop = c->lz_flags;
    const int64_t npl = g.plane;
    // sum over slabs (fixed order) and ranks of per-slab dot products into S[idx]
    auto reduce = [&](int idx, int mode, int qa, int qb) -> sscg_status {
        for (int l = 0; l < L; ++l) {
            const int64_t N = (int64_t)c->slabs[l].nzl * npl;
            lz_dot(vec(l, qa) + npl, vec(l, qb) + npl, vec(l, 4) + npl, N, mode, c->lz_part + (size_t)l * lz_grid(),
                   c->lz_ticket + l, slabv + l, stop, st);
        }
        lz_sum(slabv, L, S + idx, stop, st);
        if (c->comm) NC(ncclAllReduce(S + idx, S + idx, 1, ncclDouble, ncclSum, c->comm, st));
        return SSCG_OK;
    };
    // ||v0||^2 from a packed copy, then y_0 = v0 / (||v0|| sqrt(D))
    for (int l = 0; l < L; ++l) {
        auto &sl = c->slabs[l];
        launch_pack(g, v0 + sl.zoff * (int64_t)g.nx * g.ny, vec(l, 0), sl.nzl, nullptr, st);
    }
    TRY(reduce(0, 0, 0, 0));
    for (int l = 0; l < L; ++l) {
        auto &sl = c->slabs[l];
        lz_init(g, sl, v0 + sl.zoff * (int64_t)g.nx * g.ny, vec(l, 4), S + 0, vec(l, 0), st);
    }
    int iy = 0, iyp = 1, iz = 2;
    const bool halo = (L > 1 || c->nranks > 1) && g.kind != SSCG_OP_CSR;
    std::vector<double *> yv(L);
    for (int k = 0; k < iters; ++k) {
        for (int l = 0; l < L; ++l) yv[l] = vec(l, iy);
        if (halo) TRY(exchange(c, yv.data(), st));
        for (int l = 0; l < L; ++l) {   // w = A y
            auto &sl = c->slabs[l];
            K1Args a{};
            a.p = vec(l, iy);
            a.w = vec(l, 3);
            a.kx = sl.kx; a.ky = sl.ky; a.kz = sl.kz;
            a.dinv = sl.dinv;
            a.dinv_c = g.dinv_c;
            a.mode = 0;
            a.zb = 1;
            a.ze = sl.nzl + 1;
            a.nzl = sl.nzl;
            launch_k1(g, a, nullptr, st);
        }
        TRY(reduce(1, 0, iy, 3));                                      // a_k = y^T A y
        for (int l = 0; l < L; ++l) {
            const int64_t N = (int64_t)c->slabs[l].nzl * npl;
            lz_update(vec(l, 3) + npl, vec(l, 4) + npl, vec(l, iy) + npl, vec(l, iyp) + npl, vec(l, iz) + npl, N,
                      S + 1, S + 3, stop, st);
        }
        TRY(reduce(2, 1, iz, iz));                                     // b_k^2 = z^T D z
        lz_record(S + 1, S + 2, alpha, beta, S + 3, k, c->lz_flags, c->lz_flags + 1, st);
        for (int l = 0; l < L; ++l) lz_scale(vec(l, iz) + npl, (int64_t)c->slabs[l].nzl * npl, S + 3, stop, st);
        const int t = iyp;
        iyp = iy;
        iy = iz;
        iz = t;
    }
    lz_extremes(alpha, beta, c->lz_flags + 1, margin, S + 4, st);
    CU(cudaGetLastError());
    double out[2];
    CU(cudaMemcpyAsync(out, S + 4, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (alpha_out) CU(cudaMemcpyAsync(alpha_out, alpha, (size_t)iters * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (beta_out) CU(cudaMemcpyAsync(beta_out, beta, (size_t)iters * sizeof(double), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    *lmin = out[0];
    *lmax = out[1];
    if (!(out[0] > 0.0) || !(out[1] > out[0]) || !std::isfinite(out[1]))
        return fail(SSCG_ERR_BREAKDOWN, "Lanczos gave no valid interval (%g, %g)", out[0], out[1]);
    return SSCG_OK;
}

// algorithmic bytes per outer iteration of the basis kernels under the
// schedule enqueue_outer uses

extern "C" sscg_status sscg_query(const sscg_ctx *c, int32_t what, int64_t *out)
{
    if (!c || !out) return fail(SSCG_ERR_INVALID, "null argument");
    const int s = c->s;
    const bool mono = c->basis == SSCG_BASIS_MONOMIAL;
    switch (what) {
    case SSCG_QUERY_BASIS_FUSED:   // basis steps per launch of the schedule's main kernel
        *out = uses_mp3(c) ? 3 : uses_fused(c) ? 2 : 1;
        return SSCG_OK;
    case SSCG_QUERY_PEER_HALO:
        *out = !uses_peer(c) ? 0 : c->peer_remote ? 2 : 1;
        return SSCG_OK;
    case SSCG_QUERY_BASIS_VECTORS:
    case SSCG_QUERY_BASIS_SINGLE_VECTORS: {
        // FP64 vectors of n_local read + written by the basis steps of one outer
        // (_SINGLE: by the single steps of a fused schedule, the SSCG_PROF_BASIS_SINGLE launches)
        const bool wf = uses_wfree(c), fold = uses_wlfold(c);
        const int se = fold ? s - 1 : s;   // steps run by basis kernels (fold: w_{s-1} formed in K2R / K5)
        auto wst = [&](int j) { return (!wf || (j == s - 1 && !fold)) ? 1 : 0; };   // w_j stored?
        int64_t v = 0, v1 = 0;
        if (uses_mp3(c)) {
            int j = 0;
            for (; j + 2 < se; j += 3)   // p_j, p_{j-1} in; p_{j+1..j+3} and stored w out
                v += 1 + (j > 0) + (j + 1 < s) + (j + 2 < s) + (j + 3 < s) + wst(j) + wst(j + 1) + wst(j + 2);
            if (j + 1 < se) { v += 1 + (j > 0) + 1 + (j + 2 < s) + wst(j) + wst(j + 1); j += 2; }   // a K1F pair
            if (j < se) v1 += 1 + (j > 0 && j < s - 1) + wst(j) + (j < s - 1);                      // a single step
        } else if (uses_fused(c)) {
            int j = 0;
            for (; j + 1 < se; j += 2) v += 1 + (j > 0) + 1 + (j + 2 < s) + wst(j) + wst(j + 1);
            if (j < se) v1 += 1 + (j > 0 && j < s - 1) + wst(j) + (j < s - 1);   // the last step alone
        } else {
            for (int j = 0; j < se; ++j) {
                const bool pn = j < s - 1, pm = !mono && j > 0 && pn;
                v += 1 + pm + wst(j) + pn;
            }
        }
        *out = (what == SSCG_QUERY_BASIS_VECTORS) ? v + v1 : v1;
        return SSCG_OK;
    }
    case SSCG_QUERY_GRAM_VECTORS:
        // stored W: P and W (2s); recovered W: P, w_{s-1} and diag(M) when it varies;
        // block-conjugate: [P | Q'] and [W | Z'] (4s)
        // (fold: P, then p_{s-1} again for p_{s-1}^T A p_{s-1})
        // block-conjugate, W-free: [P | Q'], Z' and w_{s-1} (3s + 1)
        *out = c->blockcg ? (uses_wfree(c) ? 3 * (int64_t)s + 1 : 4 * (int64_t)s) : uses_wlfold(c) ? (int64_t)s + 1 :
               uses_wfree(c) ? (int64_t)s + 1 + (c->slabs[0].dvec ? 1 : 0) : 2 * (int64_t)s;
        return SSCG_OK;
    case SSCG_QUERY_UPDATE_VECTORS:
        // P (s) + x in, x + r out; the stored-W form also reads W (s), the
        // recurrence form only w_{s-1}
        // block-conjugate: P, W, Q', Z', x in; Q, Z, x, r out
        // (W-free: W_k recovered, so P, Q', Z', w_{s-1}, x in; Q, Z, x, r out: 5s + 4)
        *out = c->blockcg ? (uses_wfree(c) ? 5 * (int64_t)s + 4 : 6 * (int64_t)s + 3) : uses_k5fold(c) ? (int64_t)s + 3 :
               uses_rec_update(c) ? (int64_t)s + 4 + (c->slabs[0].dvec ? 1 : 0) : 2 * (int64_t)s + 3;
        return SSCG_OK;
    default:
        return fail(SSCG_ERR_INVALID, "unknown query %d", what);
    }
}
