// K2 -- fused tall-skinny Gram pass:
//   Ghat_ij = p_i^T w_j  (i <= j, W = AP)      c_i = p_i^T p_0  (= P^T r_k)
// One persistent CTA per SM streams its contiguous share of the 2s basis
// columns exactly once from HBM with 1-D bulk TMA copies
// (cp.async.bulk ... mbarrier::complete_tx) into a 3-stage shared-memory
// ring; consumer warps own TB x TB register tiles of the upper block
// triangle of [Ghat | c] and read their operands from shared memory.
// Partials are reduced with warp shuffles, then across warps in a fixed
// order, written per CTA, and the last CTA to finish (integer ticket, no FP
// atomics) sums all CTA partials in index order: the result is bitwise
// deterministic for a given grid.
#include "sscg_internal.cuh"

namespace sscg {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t phase)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

constexpr int NSTAGE = 3;

struct K2Params {
    const double *P;   // interior start of p_0
    const double *W;   // interior start of w_0
    int64_t vstride;   // doubles between basis vectors
    int64_t N;         // interior doubles per vector (even)
    int s;
    int E;             // elements per stage (multiple of 64)
    int nb;            // ceil(s / TB)
    int nroles;        // roles in the grid (all CTAs)
    int roles_cta;     // roles per CTA (grid.y groups)
    int nsl;           // slices per role
    double *part;      // [gridDim.y * gridDim.x][nent]
    double *out;       // [s*s + s]
    unsigned *ticket;
};

template <int TB>
__global__ void __launch_bounds__(256, 1) k2_gram(K2Params k, const DevState *st)
{
    if (st && st->done) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ uint64_t full[NSTAGE];
    __shared__ bool is_last;
    const int s = k.s, E = k.E;
    const int ncol = 2 * s;
    double *stage0 = reinterpret_cast<double *>(smem_raw);
    const int64_t stage_elems = (int64_t)ncol * E;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // role of this warp: (I, J) with I <= J in block units
    const int role_local = warp / k.nsl, slice = warp % k.nsl;
    const int role = blockIdx.y * k.roles_cta + role_local;
    int I = 0, J = 0;
    {
        int r = role;
        for (int a = 0; a < k.nb; ++a) {
            if (r < k.nb - a) { I = a; J = a + r; break; }
            r -= k.nb - a;
        }
    }
    const bool active = role_local < k.roles_cta && role < k.nroles;

    // contiguous chunk range of this CTA
    const int64_t nchunks = (k.N + E - 1) / E;
    const int64_t c_lo = nchunks * blockIdx.x / gridDim.x;
    const int64_t c_hi = nchunks * (blockIdx.x + 1) / gridDim.x;

    if (tid == 0) {
        for (int i = 0; i < NSTAGE; ++i) mbar_init(&full[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto issue = [&](int64_t c, int stg) {
        const int64_t e0 = c * E;
        const int64_t ne = (k.N - e0 < E) ? (k.N - e0) : E;
        const uint32_t bytes = (uint32_t)(ne * 8);
        double *dst = stage0 + stg * stage_elems;
        mbar_expect_tx(&full[stg], bytes * (uint32_t)ncol);
        for (int col = 0; col < ncol; ++col) {
            const double *src = (col < s ? k.P + (int64_t)col * k.vstride : k.W + (int64_t)(col - s) * k.vstride) + e0;
            bulk_g2s(dst + (int64_t)col * E, src, bytes, &full[stg]);
        }
    };
    if (tid == 0)
        for (int i = 0; i < NSTAGE && c_lo + i < c_hi; ++i) issue(c_lo + i, i);

    double acc[TB][TB];
    double cac[TB];
#pragma unroll
    for (int a = 0; a < TB; ++a) {
        cac[a] = 0.0;
#pragma unroll
        for (int b = 0; b < TB; ++b) acc[a][b] = 0.0;
    }
    const bool diag = (I == J);
    const int i0 = I * TB, j0 = J * TB;

    for (int64_t c = c_lo; c < c_hi; ++c) {
        const int it = (int)(c - c_lo);
        const int stg = it % NSTAGE;
        const uint32_t phase = (uint32_t)((it / NSTAGE) & 1);
        while (!mbar_try_wait(&full[stg], phase)) {
        }
        const int64_t e0 = c * E;
        const int ne = (int)((k.N - e0 < E) ? (k.N - e0) : E);
        const double *sb = stage0 + stg * stage_elems;
        if (active) {
            for (int e = lane + 32 * slice; e < ne; e += 32 * k.nsl) {
                double av[TB], bv[TB];
#pragma unroll
                for (int a = 0; a < TB; ++a) av[a] = (i0 + a < s) ? sb[(int64_t)(i0 + a) * E + e] : 0.0;
#pragma unroll
                for (int b = 0; b < TB; ++b) bv[b] = (j0 + b < s) ? sb[(int64_t)(s + j0 + b) * E + e] : 0.0;
#pragma unroll
                for (int a = 0; a < TB; ++a)
#pragma unroll
                    for (int b = 0; b < TB; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
                if (diag) {
                    const double p0 = sb[e];
#pragma unroll
                    for (int a = 0; a < TB; ++a) cac[a] = fma(av[a], p0, cac[a]);
                }
            }
        }
        __syncthreads();   // every warp is done with this stage
        if (tid == 0 && c + NSTAGE < c_hi) issue(c + NSTAGE, stg);
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
    // per-warp results to smem (reuse stage 0), then slices summed in order
    double *red = stage0;   // [nwarps][TB*TB + TB]
    constexpr int RW = TB * TB + TB;
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int a = 0; a < TB; ++a) {
#pragma unroll
            for (int b = 0; b < TB; ++b) red[warp * RW + a * TB + b] = acc[a][b];
            red[warp * RW + TB * TB + a] = cac[a];
        }
    }
    __syncthreads();
    const int nent = s * s + s;
    double *mypart = k.part + (int64_t)(blockIdx.y * gridDim.x + blockIdx.x) * nent;
    if (gridDim.y > 1) {   // entries owned by other role groups read as 0
        for (int q = tid; q < nent; q += blockDim.x) mypart[q] = 0.0;
        __syncthreads();
    }
    // each active role's slice-0 warp writes its entries
    if (active && slice == 0) {
        for (int q = lane; q < RW; q += 32) {
            double v = 0.0;
            for (int sl = 0; sl < k.nsl; ++sl) v += red[(warp + sl) * RW + q];
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
    const int nparts = gridDim.x * gridDim.y;
    for (int q = tid; q < nent; q += blockDim.x) {
        int i, j;
        bool valid;
        if (q < s * s) { i = q / s; j = q % s; valid = (i <= j); }
        else { i = q - s * s; j = -1; valid = true; }
        if (!valid) continue;
        double v = 0.0;
        for (int b = 0; b < nparts; ++b) v += __ldcg(k.part + (int64_t)b * nent + q);
        if (j >= 0) {
            k.out[i * s + j] = v;
            k.out[j * s + i] = v;
        } else {
            k.out[s * s + i] = v;
        }
    }
    if (tid == 0) *k.ticket = 0u;
}

// fixed-order sum of the per-slab blocks of one process
__global__ void k_slab_sum(const double *const *blks, int nslab, int len, double *out, const DevState *st)
{
    if (st && st->done) return;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < len; q += gridDim.x * blockDim.x) {
        double v = 0.0;
        for (int b = 0; b < nslab; ++b) v += blks[b][q];
        out[q] = v;
    }
}

int g_sms = 0;

struct K2Plan {
    int TB, nb, nroles, roles_cta, nsl, E, gy, threads;
    size_t smem;
};

K2Plan plan(int s)
{
    K2Plan p;
    p.TB = (s <= 8) ? 4 : 8;
    p.nb = (s + p.TB - 1) / p.TB;
    p.nroles = p.nb * (p.nb + 1) / 2;
    p.roles_cta = p.nroles < 8 ? p.nroles : 8;
    p.gy = (p.nroles + p.roles_cta - 1) / p.roles_cta;
    p.nsl = 1;
    while (p.roles_cta * p.nsl * 2 <= 8) p.nsl *= 2;
    // stage of about 64 KB: 2s columns x E doubles
    int E = 65536 / (16 * s);
    E = (E / 64) * 64;
    if (E < 64) E = 64;
    if (E > 1024) E = 1024;
    p.E = E;
    p.threads = 32 * p.roles_cta * p.nsl;
    p.smem = (size_t)NSTAGE * 2 * s * E * sizeof(double);
    return p;
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

// partial buffer must hold k2_grid() * gy * (s*s+s) doubles; gy <= 4 for s <= 64
void launch_k2(const Geo &g, const Slab &sl, int s, const DevState *st, double *out_blk,
               cudaStream_t stream)
{
    const K2Plan p = plan(s);
    K2Params k;
    k.P = sl.P + g.plane;
    k.W = sl.W + g.plane;
    k.vstride = g.vstride;
    k.N = (int64_t)sl.nzl * g.plane;
    k.s = s;
    k.E = p.E;
    k.nb = p.nb;
    k.nroles = p.nroles;
    k.roles_cta = p.roles_cta;
    k.nsl = p.nsl;
    k.part = sl.part;
    k.out = out_blk;
    k.ticket = sl.ticket;
    const int64_t nchunks = (k.N + p.E - 1) / p.E;
    int gx = k2_grid();
    if (nchunks < gx) gx = (int)nchunks;
    dim3 grid(gx, p.gy);
    if (p.TB == 4) {
        cudaFuncSetAttribute(k2_gram<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
        k2_gram<4><<<grid, p.threads, p.smem, stream>>>(k, st);
    } else {
        cudaFuncSetAttribute(k2_gram<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
        k2_gram<8><<<grid, p.threads, p.smem, stream>>>(k, st);
    }
}

void launch_slab_sum(const double *const *blks_dev, int nslab, int len, double *blk, const DevState *st,
                     cudaStream_t s)
{
    k_slab_sum<<<(len + 255) / 256, 256, 0, s>>>(blks_dev, nslab, len, blk, st);
}

}  // namespace sscg
