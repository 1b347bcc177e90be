// K2 -- fused tall-skinny Gram pass:
//   Ghat_ij = p_i^T w_j  (i <= j, W = AP)      c_i = p_i^T p_0  (= P^T r_k)
//
// One persistent CTA per SM streams a contiguous share of the basis exactly
// once from HBM.  A producer warp issues two TMA tensor loads per stage
// (cp.async.bulk.tensor.2d: a [s_pad x E] box of P and one of W, rows past s
// and elements past the slab zero-filled by the TMA unit) into an
// NS-deep shared-memory ring guarded by full/empty mbarriers.  Consumer warps
// own TB x TB register tiles of the upper block triangle of Ghat (the
// diagonal-tile warps also accumulate c) and read operands from shared
// memory with compile-time offsets.  Partials are reduced with warp shuffles,
// then across warps in a fixed order, written per CTA; the last CTA (integer
// ticket, no FP atomics) sums the CTA partials in index order, so the block
// is bitwise deterministic for a given grid.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "sscg_internal.cuh"
#include "tma.cuh"
#include "gram_reduce.cuh"

namespace sscg {
namespace {

constexpr int MAX_STAGE = 8;

struct K2Params {
    int64_t N;         // interior doubles per vector
    int s, s_pad;      // basis size, box rows (multiple of TB)
    int nb;            // s_pad / TB
    int nroles;        // roles in the grid (all role groups)
    int roles_cta;     // roles per CTA (grid.y groups)
    int nsl;           // consumer warps per role
    int nstage;
    double *part;      // [gridDim.y * gridDim.x][s*s + s]
    double *out;       // [s*s + s]
    unsigned *ticket;
};

template <int TB, int E>
__global__ void __launch_bounds__(256, 1)
    k2_gram(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmW, K2Params k,
            const DevState *st)
{
    PDL_ENTRY(st);
    extern __shared__ __align__(1024) double smem[];
    __shared__ uint64_t full[MAX_STAGE], empty[MAX_STAGE];
    __shared__ bool is_last;
    const int s = k.s, NS = k.nstage;
    const int stage_elems = 2 * k.s_pad * E;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ncw = k.roles_cta * k.nsl;            // consumer warps

    // chunks are dealt round-robin (chunk = blockIdx.x + it * gridDim.x): at any
    // moment the grid reads one contiguous ~gridDim.x*E*8-byte window of each
    // column, which keeps HBM streaming at full rate also for small vectors
    const int64_t nchunks = (k.N + E - 1) / E;
    const int nit = (int)((nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x);

    if (tid == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], ncw);
        }
        mbar_fence_init();
        tma_prefetch_desc(&tmP);
        tma_prefetch_desc(&tmW);
    }
    __syncthreads();

    // consumer role (warps 1..ncw): tile (I, J), I <= J, in block units
    const int cw = warp - 1;
    const int role_local = cw / k.nsl, slice = cw - role_local * k.nsl;
    const int role = blockIdx.y * k.roles_cta + role_local;
    int I = 0, J = 0;
    {
        int r = role;
        for (int a = 0; a < k.nb; ++a) {
            if (r < k.nb - a) { I = a; J = a + r; break; }
            r -= k.nb - a;
        }
    }
    const bool consumer = warp >= 1 && cw < ncw;
    const bool active = consumer && role < k.nroles;
    const bool diag = (I == J);

    double acc[TB][TB];
    double cac[TB];
#pragma unroll
    for (int a = 0; a < TB; ++a) {
        cac[a] = 0.0;
#pragma unroll
        for (int b = 0; b < TB; ++b) acc[a][b] = 0.0;
    }

    if (warp == 0) {
        // ---------------- producer ----------------
        // the whole warp walks the loop (lane 0 issues) so that warp 0 is
        // converged when it reaches the shuffles and the CTA barrier below: a
        // diverged warp 0 there cost ~80 us per launch (measured with %globaltimer)
        const uint32_t bytes = (uint32_t)stage_elems * 8u;
        for (int it = 0; it < nit; ++it) {
            if (lane == 0) {
                const int stg = it % NS;
                if (it >= NS) mbar_wait(&empty[stg], (uint32_t)((it / NS - 1) & 1));
                double *dst = smem + (size_t)stg * stage_elems;
                const int x = (int)((blockIdx.x + (int64_t)it * gridDim.x) * E);
                mbar_expect_tx(&full[stg], bytes);
                tma_load_2d(dst, &tmP, x, 0, &full[stg]);
                tma_load_2d(dst + k.s_pad * E, &tmW, x, 0, &full[stg]);
            }
            __syncwarp();
        }
    } else if (consumer) {
        // ---------------- consumers ----------------
        for (int it = 0; it < nit; ++it) {
            const int stg = it % NS;
            mbar_wait(&full[stg], (uint32_t)((it / NS) & 1));
            if (active) {
                const double *sP = smem + (size_t)stg * stage_elems;
                const double *pa = sP + I * TB * E;
                const double *pb = sP + (k.s_pad + J * TB) * E;
#pragma unroll 2
                for (int t = slice; t < E / 32; t += k.nsl) {
                    const int e = t * 32 + lane;
                    double av[TB], bv[TB];
#pragma unroll
                    for (int a = 0; a < TB; ++a) av[a] = pa[a * E + e];
#pragma unroll
                    for (int b = 0; b < TB; ++b) bv[b] = pb[b * E + e];
#pragma unroll
                    for (int a = 0; a < TB; ++a)
#pragma unroll
                        for (int b = 0; b < TB; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
                    if (diag) {
                        const double p0 = sP[e];
#pragma unroll
                        for (int a = 0; a < TB; ++a) cac[a] = fma(av[a], p0, cac[a]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stg]);
        }
    }

    // warp reduction (butterfly, fixed order)
#pragma unroll
    for (int a = 0; a < TB; ++a) {
#pragma unroll
        for (int b = 0; b < TB; ++b) {
            double v = acc[a][b];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            acc[a][b] = v;
        }
        double v = cac[a];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        cac[a] = v;
    }
    __syncthreads();   // all TMA traffic consumed: the ring can be reused
    constexpr int RW = TB * TB + TB;
    double *red = smem;   // [ncw][RW]
    if (consumer && lane == 0) {
#pragma unroll
        for (int a = 0; a < TB; ++a) {
#pragma unroll
            for (int b = 0; b < TB; ++b) red[cw * RW + a * TB + b] = acc[a][b];
            red[cw * RW + TB * TB + a] = cac[a];
        }
    }
    __syncthreads();
    const int nent = s * s + s;
    double *mypart = k.part + (int64_t)(blockIdx.y * gridDim.x + blockIdx.x) * nent;
    if (gridDim.y > 1) {   // entries owned by other role groups read as 0
        for (int q = tid; q < nent; q += blockDim.x) mypart[q] = 0.0;
        __syncthreads();
    }
    if (active && slice == 0) {
        const int i0 = I * TB, j0 = J * TB;
        for (int q = lane; q < RW; q += 32) {
            double v = 0.0;
            for (int sl = 0; sl < k.nsl; ++sl) v += red[(cw + sl) * RW + q];
            if (q < TB * TB) {
                const int i = i0 + q / TB, j = j0 + q % TB;
                if (i < s && j < s && i <= j) mypart[i * s + j] = v;
            } else if (diag) {
                const int i = i0 + (q - TB * TB);
                if (i < s) mypart[s * s + i] = v;
            }
        }
    }
    // last CTA sums all partials in index order
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned total = gridDim.x * gridDim.y;
        const unsigned t = atomicAdd(k.ticket, 1u);
        is_last = (t == total - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    last_cta_sum(k.part, gridDim.x * gridDim.y, s, k.out);
    if (tid == 0) *k.ticket = 0u;
}

// fixed-order sum of the per-slab blocks of one process
__global__ void k_slab_sum(const double *const *blks, int nslab, int len, double *out, const DevState *st)
{
    PDL_ENTRY(st);
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < len; q += gridDim.x * blockDim.x) {
        double v = 0.0;
        for (int b = 0; b < nslab; ++b) v += blks[b][q];
        out[q] = v;
    }
}

int g_sms = 0;

struct K2Plan {
    int TB, E, s_pad, nb, nroles, roles_cta, nsl, gy, nstage, threads;
    size_t smem;
};

K2Plan plan(const Geo &g, int s)
{
    K2Plan p;
    p.TB = (s <= 8) ? 4 : 8;
    p.E = (s <= 16) ? 256 : (s <= 32 ? 128 : 64);
    if (g.kn.k2_e) {   // tuning override (64 / 128 / 256)
        const int v = g.kn.k2_e;
        if ((v == 64 || v == 128 || v == 256) && (s > 8)) p.E = v;
    }
    p.s_pad = (s + p.TB - 1) / p.TB * p.TB;
    p.nb = p.s_pad / p.TB;
    p.nroles = p.nb * (p.nb + 1) / 2;
    // <= 7 consumer warps per CTA (255 registers per thread); more roles are
    // split evenly over gy co-resident CTA groups that stream the same chunks
    // (launch_k2 shrinks grid.x so that all gy groups are resident at once and
    // the partner group's TMA loads of a chunk are L2 hits)
    p.gy = (p.nroles + 6) / 7;
    p.roles_cta = (p.nroles + p.gy - 1) / p.gy;
    p.nsl = 1;
    while (p.roles_cta * p.nsl * 2 <= 7) p.nsl *= 2;
    const size_t stage = (size_t)2 * p.s_pad * p.E * sizeof(double);
    p.nstage = (int)std::min<size_t>(MAX_STAGE, (200 * 1024) / stage);
    if (g.kn.k2_ns) p.nstage = std::max(2, std::min(p.nstage, g.kn.k2_ns));
    p.smem = stage * p.nstage;
    p.threads = 32 * (1 + p.roles_cta * p.nsl);
    return p;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    return fn;
}

}  // namespace

int k2_grid()
{
    if (!g_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_sms <= 0) g_sms = 148;
    }
    return g_sms;
}

int k2_num_entries(int s) { return s * s + s; }

// 2-D tensor map over `rows` basis vectors starting at `base` (interior
// start), `inner` doubles each, `stride` doubles apart; box [box_rows x box_inner]
bool encode_rows_map(CUtensorMap *m, const double *base, int64_t inner, int rows, int64_t stride, int box_inner,
                     int box_rows)
{
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)stride * sizeof(double)};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool k2_prepare(const Geo &g, Slab &sl, int s)
{
    const K2Plan p = plan(g, s);
    const int64_t N = (int64_t)sl.nzl * g.plane;
    // opt in to the large dynamic shared memory once (outside any graph capture)
    const int mx = 210 * 1024;   // >= every plan's ring (<= 200 KB) + static smem fits 227 KB
    if (cudaFuncSetAttribute(k2_gram<4, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess ||
        cudaFuncSetAttribute(k2_gram<8, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess ||
        cudaFuncSetAttribute(k2_gram<8, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess ||
        cudaFuncSetAttribute(k2_gram<8, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess)
        return false;
    if (!encode_rows_map(&sl.tmP, sl.P + g.plane, N, s, g.vstride, p.E, p.s_pad) ||
        !encode_rows_map(&sl.tmW, sl.W + g.plane, N, s, g.vstride, p.E, p.s_pad))
        return false;
    sl.has_k2d = k2d_enabled(g, s);
    return !sl.has_k2d || k2d_prepare(g, sl, s);
}

template <int TB, int E>
static void launch_t(bool pdl, const CUtensorMap &a, const CUtensorMap &b, const K2Params &k, const K2Plan &p,
                     dim3 grid, const DevState *st, cudaStream_t stream)
{
    launch_pdl(pdl, k2_gram<TB, E>, dim3(grid), dim3(p.threads), p.smem, stream, a, b, k, st);
}

// partial buffer must hold k2_grid() * (s*s+s) doubles (gx * gy <= k2_grid())
void launch_k2(const Geo &g, const Slab &sl, int s, const DevState *st, double *out_blk, cudaStream_t stream)
{
    if (sl.has_k2d) {
        launch_k2d(g, sl, s, st, out_blk, stream);
        return;
    }
    const K2Plan p = plan(g, s);
    K2Params k;
    k.N = (int64_t)sl.nzl * g.plane;
    k.s = s;
    k.s_pad = p.s_pad;
    k.nb = p.nb;
    k.nroles = p.nroles;
    k.roles_cta = p.roles_cta;
    k.nsl = p.nsl;
    k.nstage = p.nstage;
    k.part = sl.part;
    k.out = out_blk;
    k.ticket = sl.ticket;
    const int64_t nchunks = (k.N + p.E - 1) / p.E;
    int gx = std::max(1, k2_grid() / p.gy);   // gx * gy CTAs: one per SM, all resident
    if (g.kn.k2_grid) gx = std::max(1, std::min(gx, g.kn.k2_grid));   // tuning
    if (nchunks < gx) gx = (int)nchunks;
    dim3 grid(gx, p.gy);
    if (p.TB == 4) launch_t<4, 256>(g.kn.pdl, sl.tmP, sl.tmW, k, p, grid, st, stream);
    else if (p.E == 256) launch_t<8, 256>(g.kn.pdl, sl.tmP, sl.tmW, k, p, grid, st, stream);
    else if (p.E == 128) launch_t<8, 128>(g.kn.pdl, sl.tmP, sl.tmW, k, p, grid, st, stream);
    else launch_t<8, 64>(g.kn.pdl, sl.tmP, sl.tmW, k, p, grid, st, stream);
}

void launch_slab_sum(const double *const *blks_dev, int nslab, int len, double *blk, const DevState *st,
                     cudaStream_t s)
{
    k_slab_sum<<<(len + 255) / 256, 256, 0, s>>>(blks_dev, nslab, len, blk, st);
}

}  // namespace sscg
