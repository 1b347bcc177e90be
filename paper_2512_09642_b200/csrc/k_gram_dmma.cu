// K2D / K2R / K2S -- the tall-skinny Gram pass
//   Ghat_ij = p_i^T w_j  (i <= j, W = AP)      c_i = p_i^T p_0
// K2R (W-free schedule, the default): W recovered per point from the basis
// recurrence (R23), below; K2S: the same for s <= 8 as a streaming
// register-accumulator pass; K2D (stored W): this kernel.
// K2D on the FP64 tensor-core path (mma.sync m8n8k4 f64, "DMMA"): Ghat = P W^T is
// a dense contraction over the grid points, s x N times N x s.  Used for
// s > 16, where the FP64 FMA count per byte (s(s+3)/2 per point) makes the
// register-tiled K2 issue-bound (five consumer warps per SM at 255 registers);
// one DMMA does 256 FMAs, so a warp carries every 8 x 8 tile of the upper
// block triangle in 2 registers per tile and eight warps split the points.
//
// Same pipeline as K2: warp 0 issues two cp.async.bulk.tensor.2d boxes per
// stage (rows = basis vectors, EP points each, OOB rows/points zero-filled)
// into an mbarrier ring; consumer warps take k-steps of 4 points.  The box
// row pitch EP*8 bytes is 32 mod 128, so the 8 rows x 4 points of one
// fragment load fall on distinct banks.  Per-warp tiles are reduced across
// warps in a fixed order, per-CTA partials by the last CTA in index order
// (deterministic, no FP atomics).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "sscg_internal.cuh"
#include "tma.cuh"
#include "gram_reduce.cuh"

namespace sscg {
namespace {

// consumer warps: 16 while the accumulators are small (s <= 32), 8 above
// (register budget); one producer warp
#ifndef K2_DMMA_ASM
#define K2_DMMA_ASM asm volatile
#endif
#ifndef K2_NCW_SMALL
#define K2_NCW_SMALL 24
#endif
#ifndef K2R_U3
#define K2R_U3 2
#endif
// consumer warps: 24 for s <= 16 (few accumulator tiles), 12 for s <= 32, 8
// above (register budget); measured: cfg 5 16 warps x U=4 2.10 ms, 24 x U=2 2.06 ms;
// cfg 4 s = 32 16 warps 0.553 ms, 8 0.500, 12 0.453
#ifndef K2_NCW_MID
#define K2_NCW_MID 12
#endif
#ifndef K2_NCW_VARM
#define K2_NCW_VARM 20
#endif
// varm: K2R with a varying diagonal (more live values per fragment: fewer
// warps; cfg 4 s = 16: 24 warps 0.196 ms (spilling), 20 0.185, 16 0.193, 12 0.187)
__host__ __device__ constexpr int ncw_for(int nb, bool varm = false)
{
    return nb >= 5 ? 8 : nb >= 3 ? K2_NCW_MID : (varm ? K2_NCW_VARM : K2_NCW_SMALL);
}
__host__ __device__ constexpr int threads_for(int nb, bool varm = false) { return 32 * (ncw_for(nb, varm) + 1); }
constexpr int MAXS = 16;               // ring stages

struct K2DParams {
    int64_t N;         // interior doubles per vector
    int s, s_pad;      // s_pad = 8 * NB
    int nstage;
    int ngroups;       // consumer warp groups (a divisor of NCW, <= nstage)
    double *part;      // [gridDim.x][s*s + s]
    double *out;
    unsigned *ticket;
};

__device__ __forceinline__ double2 lds2(const double *p) { return *reinterpret_cast<const double2 *>(p); }

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    K2_DMMA_ASM("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int NB, int EP>
__global__ void __launch_bounds__(threads_for(NB), 1)
    k2d(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmW, K2DParams k,
        const DevState *st)
{
    PDL_ENTRY(st);
    constexpr int SP = 8 * NB;                 // rows per box
    constexpr int NCW = ncw_for(NB), THREADS = threads_for(NB);
    constexpr int KS = EP / 4;                 // k-steps per stage
    constexpr int NT = NB * (NB + 1) / 2;      // upper-triangle tiles
    extern __shared__ __align__(1024) double smem[];
    __shared__ uint64_t full[MAXS], empty[MAXS];
    __shared__ bool is_last;
    const int s = k.s, NS = k.nstage;
    const int stage_elems = 2 * SP * EP;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t nchunks = (k.N + EP - 1) / EP;
    const int nit = (int)((nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x);

    if (tid == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NCW / k.ngroups);
        }
        mbar_fence_init();
        tma_prefetch_desc(&tmP);
        tma_prefetch_desc(&tmW);
    }
    __syncthreads();

    // U accumulator sets: k-steps rotate over them so that U*NT independent
    // DMMA chains hide the tensor-core latency when the tile count is small
    constexpr int U = (NT >= 10) ? 1 : (NT >= 6) ? 2 : (NT >= 3) ? 4 : 8;
    double acc[U][NT][2];
    double cac[NB];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[u][t][0] = acc[u][t][1] = 0.0;
#pragma unroll
    for (int i = 0; i < NB; ++i) cac[i] = 0.0;

    if (warp == 0) {
        const uint32_t bytes = (uint32_t)stage_elems * 8u;
        for (int it = 0; it < nit; ++it) {
            if (lane == 0) {
                const int stg = it % NS;
                if (it >= NS) mbar_wait(&empty[stg], (uint32_t)((it / NS - 1) & 1));
                double *dst = smem + (size_t)stg * stage_elems;
                const int x = (int)((blockIdx.x + (int64_t)it * gridDim.x) * EP);
                mbar_expect_tx(&full[stg], bytes);
                tma_load_2d(dst, &tmP, x, 0, &full[stg]);
                tma_load_2d(dst + SP * EP, &tmW, x, 0, &full[stg]);
            }
            __syncwarp();
        }
    } else {
        const int cw = warp - 1;
        const int r = lane >> 2, kk = lane & 3;   // fragment row (m or n) and k index
        // warps form min(NS, NCW) groups; group g takes stages g, g + ngroups, ...
        // and its wpg warps split the k-steps of a stage
        const int ngroups = k.ngroups, wpg = NCW / ngroups;
        const int grp = cw / wpg, wig = cw - grp * wpg;
        for (int it = (grp < ngroups ? grp : nit); it < nit; it += ngroups) {
            const int stg = it % NS;
            mbar_wait(&full[stg], (uint32_t)((it / NS) & 1));
            const double *sP = smem + (size_t)stg * stage_elems;
            const double *sW = sP + SP * EP;
            for (int ks0 = wig; ks0 < KS; ks0 += wpg * U) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int ks = ks0 + u * wpg;
                    if (ks >= KS) break;
                    const int o = r * EP + ks * 4 + kk;
                    double a[NB], b[NB];
#pragma unroll
                    for (int i = 0; i < NB; ++i) a[i] = sP[o + i * 8 * EP];
#pragma unroll
                    for (int j = 0; j < NB; ++j) b[j] = sW[o + j * 8 * EP];
                    const double p0 = sP[ks * 4 + kk];
#pragma unroll
                    for (int i = 0; i < NB; ++i) cac[i] = fma(a[i], p0, cac[i]);
                    int t = 0;
#pragma unroll
                    for (int i = 0; i < NB; ++i)
#pragma unroll
                        for (int j = i; j < NB; ++j, ++t) dmma(acc[u][t][0], acc[u][t][1], a[i], b[j]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stg]);
        }
        // c: lanes with the same r hold partial sums over different k -> sum the 4
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            cac[i] += __shfl_xor_sync(0xffffffffu, cac[i], 1);
            cac[i] += __shfl_xor_sync(0xffffffffu, cac[i], 2);
        }
    }
    __syncthreads();   // ring drained: reuse it for the cross-warp reduction
    // red[cw][t][lane][2] tiles, then c: red[NCW*NT*64 + cw*SP + row]
    double *red = smem;
    if (warp > 0) {
        const int cw = warp - 1;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
#pragma unroll
            for (int u = 1; u < U; ++u) {   // fold the accumulator sets in a fixed order
                acc[0][t][0] += acc[u][t][0];
                acc[0][t][1] += acc[u][t][1];
            }
            red[((cw * NT + t) * 32 + lane) * 2 + 0] = acc[0][t][0];
            red[((cw * NT + t) * 32 + lane) * 2 + 1] = acc[0][t][1];
        }
        if ((lane & 3) == 0)
#pragma unroll
            for (int i = 0; i < NB; ++i) red[NCW * NT * 64 + cw * SP + i * 8 + (lane >> 2)] = cac[i];
    }
    __syncthreads();
    const int nent = s * s + s;
    double *mypart = k.part + (int64_t)blockIdx.x * nent;
    // tile t = (I, J), fragment element (lane, h): row I*8 + lane/4, col J*8 + 2*(lane%4) + h
    for (int q = tid; q < NT * 64; q += THREADS) {
        const int t = q >> 6, e = q & 63, ln = e >> 1, h = e & 1;
        double v = 0.0;
        for (int w = 0; w < NCW; ++w) v += red[((w * NT + t) * 32 + ln) * 2 + h];
        int I = 0, J = 0, tt = t;
        for (int a = 0; a < NB; ++a) {
            if (tt < NB - a) { I = a; J = a + tt; break; }
            tt -= NB - a;
        }
        const int i = I * 8 + (ln >> 2), j = J * 8 + 2 * (ln & 3) + h;
        if (i < s && j < s && i <= j) mypart[i * s + j] = v;
    }
    for (int i = tid; i < s; i += THREADS) {
        double v = 0.0;
        for (int w = 0; w < NCW; ++w) v += red[NCW * NT * 64 + w * SP + i];
        mypart[s * s + i] = v;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) is_last = atomicAdd(k.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    last_cta_sum(k.part, gridDim.x, s, k.out);
    if (tid == 0) *k.ticket = 0u;
}

// K2R -- the same DMMA Gram pass when W = AP is NOT stored (R23):
// only P (plus the stored w_{s-1}, and diag(M) per point when it varies) is
// streamed, and each B fragment w_j(point) is recovered in registers from the
// Chebyshev recurrence (PAPER.md:36-42 solved for M^{-1} A p_j)
//   w_0 = m (p_1/theta + sigma p_0),  w_j = m ((p_{j+1} + p_{j-1})/(2 theta) + sigma p_j),
// p_{j+-1} of the fragment row taken from the neighbouring lanes' A fragments
// by two shuffles.  Half the Gram bytes of K2/K2D.
struct K2RParams {
    int64_t N;
    int s, s_pad, nstage, wlp;   // wlp: padded pitch (doubles) of the w_{s-1} / diag(M) rows
    int ngroups;                 // consumer warp groups (a divisor of NCW, <= nstage)
    double inv_theta, inv_2theta, sigma, dm;
    double *part, *out;
    unsigned *ticket;
    int sb;                  // BLK: the basis size s (the pass runs over 2s rows, k.s = 2s)
};

// PAP (the w_{s-1} fold; constant diagonal only): w_{s-1} is
// not stored and not read.  Its fragment row is zero, and the pass forms the
// LOWER block triangle instead, A being symmetric:
//   Ghat_{ij} = p_i^T A p_j = (A p_i)^T p_j = w_i^T p_j,  i <= j,
// from tile (J, I) -- p_j against the recovered w_i, i < j --, so no entry
// needs w_{s-1} except the diagonal p_{s-1}^T A p_{s-1}, left 0 here and
// written afterwards by one stencil pass over p_{s-1} with a reduction (the
// TMA single step K1T in its dot mode; k_pap without TMA).  Same tile count
// and DMMA work as the upper triangle.
// GS (with PAP; R27): no w_j is formed at all.  The tiles hold the
// Euclidean Gram E = P^T P (lower block triangle, B fragment = A fragment),
// and each CTA maps its partial E to its partial Ghat by the same recurrence
// written in Gram space (A P_{:,0:s-1} = P_{:,0:s} T, T tridiagonal):
//   Ghat_{ji} = p_i^T w_j = m ((E_{i,j+1} + E_{i,j-1})/(2 theta) + sigma E_{ij}),
//   (j = 0: m (E_{i,1}/theta + sigma E_{i0})),  j <= i, (j, i) != (s-1, s-1),
// every E entry it reads in the lower triangle (j + 1 <= i, or E_{i,i+1} =
// E_{i+1,i}); c = P^T p_0 is E's column 0.  No recovery FMAs, no neighbour-row
// loads, no c FMAs: the DMMA tiles are the whole per-point work.
// BLK (the block-conjugate mode without the stored W_k, R24): the
// pass runs over the 2s rows A = [P_k | Q'] against B = [W_k | Z']: W_k's rows
// recovered from P_k as above (w_{s-1} from its stored row), Z' = A Q' staged
// from the stored rows s..2s-1 of W (tmDv carries that map); one more box per
// stage, the same tiles, reduction and output block as the stored-W pass.
// IL (with PAP, NB = 2, s even; DESIGN.md §6 K2R): interleaved fragment rows.
// Fragment row r of block J is basis row 2r + J (not 8J + r), so a lane holds
// p_{2r} and p_{2r+1}: w_{2r} takes its p_{2r+1} and w_{2r+1} its p_{2r} from
// the lane's own A fragments, and only p_{2r-1} and p_{2r+2} are loaded -- two
// shared loads per k-step pair fewer (five instead of seven).  The three
// tiles are then even x even, odd x even and odd x odd rows: every unordered
// pair once (the odd x even tile holds both orientations of the mixed pairs,
// p_i^T w_j = p_j^T w_i, R26), and w_{s-1} (s-1 odd) is never a B column there.
template <int NB, int EP, bool VARM, bool PAP = false, bool BLK = false, bool GS = false, bool IL = false>
__global__ void __launch_bounds__(threads_for(NB, VARM), 1)
    k2r(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmWl,
        const __grid_constant__ CUtensorMap tmDv, K2RParams k, const DevState *st)
{
    static_assert(!(PAP && VARM), "the fold needs a constant diagonal");
    static_assert(!GS || PAP, "the Gram-space map is the fold's");
    static_assert(!IL || (PAP && NB == 2 && !GS), "interleaved rows: the fold's two-block pass");
    static_assert(!(BLK && (VARM || PAP)), "the block mode's W-free pass: constant diagonal, w_{s-1} stored");
    PDL_ENTRY(st);
    constexpr int SP = 8 * NB;
    constexpr int NCW = ncw_for(NB, VARM), THREADS = threads_for(NB, VARM);
    // NB <= 2: k-step pairs from 16-B loads (pitch EP = 136, 64 mod 128 B); larger
    // NB (more live fragments): single k-steps from 8-B loads (EP = 132 / 68,
    // 32 mod 128 B) -- measured faster there (cfg 4 s = 32: 0.453 vs 0.486 ms)
    constexpr bool PAIRS = NB <= 2;
    constexpr int KS = EP / 4;
    constexpr int KS2 = EP / 8;   // k-step pairs per stage (EP = 136 or 72: row pitch 64 mod 128 B)
    constexpr int NT = NB * (NB + 1) / 2;
    extern __shared__ __align__(1024) double smem[];
    __shared__ uint64_t full[MAXS], empty[MAXS];
    __shared__ bool is_last;
    const int s = k.s, NS = k.nstage;
    constexpr int SZ = BLK ? SP / 2 : 0;   // BLK: the Z' box (rows s..2s-1 of W)
    const int stage_elems = SP * EP + SZ * EP + k.wlp * (VARM ? 2 : 1);
    const uint32_t stage_bytes = (uint32_t)(SP * EP + SZ * EP + EP * (PAP ? 0 : VARM ? 2 : 1)) * 8u;   // bytes the TMA delivers
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t nchunks = (k.N + EP - 1) / EP;
    const int nit = (int)((nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x);

    if (tid == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NCW / k.ngroups);
        }
        mbar_fence_init();
        tma_prefetch_desc(&tmP);
        if (!PAP) tma_prefetch_desc(&tmWl);
        if (VARM || BLK) tma_prefetch_desc(&tmDv);
    }
    __syncthreads();

    // U accumulator sets: k-steps rotate over them so that U*NT independent
    // DMMA chains hide the tensor-core latency when the tile count is small
#ifndef K2R_U10
#define K2R_U10 1
#endif
    constexpr int U = (NT >= 10) ? K2R_U10 : (NT >= 6) ? 2 : (NT >= 3) ? K2R_U3 : 8;
    constexpr int UP = (U >= 2) ? U / 2 : 1;   // k-step pairs per unrolled block
    double acc[U][NT][2];
    double cac[NB];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[u][t][0] = acc[u][t][1] = 0.0;
#pragma unroll
    for (int i = 0; i < NB; ++i) cac[i] = 0.0;

    if (warp == 0) {
        for (int it = 0; it < nit; ++it) {
            if (lane == 0) {
                const int stg = it % NS;
                if (it >= NS) mbar_wait(&empty[stg], (uint32_t)((it / NS - 1) & 1));
                double *dst = smem + (size_t)stg * stage_elems;
                const int x = (int)((blockIdx.x + (int64_t)it * gridDim.x) * EP);
                mbar_expect_tx(&full[stg], stage_bytes);
                tma_load_2d(dst, &tmP, x, 0, &full[stg]);
                if (BLK) {
                    tma_load_2d(dst + SP * EP, &tmDv, x, 0, &full[stg]);                 // Z' rows
                    tma_load_2d(dst + SP * EP + SZ * EP, &tmWl, x, k.sb - 1, &full[stg]);   // w_{s-1}
                } else if (!PAP) {
                    tma_load_2d(dst + SP * EP, &tmWl, x, s - 1, &full[stg]);
                }
                if (VARM) tma_load_2d(dst + SP * EP + k.wlp, &tmDv, x, 0, &full[stg]);
            }
            __syncwarp();
        }
    } else {
        const int cw = warp - 1;
        const int r = lane >> 2, kk = lane & 3;
        const int ngroups = k.ngroups, wpg = NCW / ngroups;   // as in k2d
        const int grp = cw / wpg, wig = cw - grp * wpg;
        // per-lane recurrence coefficients of fragment row j = J*8 + r (fixed for the kernel):
        //   w = m (up c1 + dn c2 + sigma p_j)  (j <= s-2),  w = w_{s-1} (stored),  0 (j >= s).
        // Constant m (VARM false): m is folded into c1, c2, cs, and row j = s-1
        // reads its "up" operand from the staged w_{s-1} row with c1 = 1,
        // c2 = cs = 0 (exactly w_{s-1}); row 0 reads its "dn" operand from row
        // 0 itself with c2 = 0.  Both are per-lane smem offsets, no selects.
        double c1[NB], c2[NB], cs[NB], use_wl[NB];
        int upd[NB], dnd[NB];
        // IL: lane rows 2r, 2r+1 at offsets (r + J) EP from o = r EP + pt; the
        // loaded neighbours p_{2r-1} (row 0: its own row, c2 = 0) and p_{2r+2}
        // (rows >= s-1 are zero rows: their own row)
        const int ilo0 = (r > 0 ? 2 * r - 1 : 0) * EP, ilo1 = ((2 * r + 1 < s - 1) ? 2 * r + 2 : 2 * r + 1) * EP;
#pragma unroll
        for (int J = 0; J < NB; ++J) {
            const int j = IL ? 2 * r + J : J * 8 + r;
            const bool rec = j < s - 1;
            const double mf = VARM ? 1.0 : k.dm;
            c1[J] = !rec ? 0.0 : (j == 0 ? k.inv_theta : k.inv_2theta) * mf;
            c2[J] = (rec && j > 0) ? k.inv_2theta * mf : 0.0;
            cs[J] = rec ? k.sigma * mf : 0.0;
            use_wl[J] = (j == s - 1) ? 1.0 : 0.0;
            upd[J] = J * 8 * EP + EP;
            dnd[J] = J * 8 * EP - ((j == 0) ? 0 : EP);
            if (!VARM && !PAP && j == s - 1) {
                c1[J] = 1.0;
                upd[J] = (SP - r) * EP;   // the w_{s-1} row: SP*EP + pt = o + (SP - r)*EP
            }
            if (PAP && j == s - 1) upd[J] = 0;   // a zero row (c1 = c2 = cs = 0) read from its own, finite, values
            if (BLK) {   // rows of [W_k | Z']: recovered below s-1, w_{s-1} and Z' staged
                const int sb = k.sb;
                const bool recb = j < sb - 1;
                c1[J] = !recb ? 0.0 : (j == 0 ? k.inv_theta : k.inv_2theta) * k.dm;
                c2[J] = (recb && j > 0) ? k.inv_2theta * k.dm : 0.0;
                cs[J] = recb ? k.sigma * k.dm : 0.0;
                upd[J] = J * 8 * EP + EP;
                dnd[J] = J * 8 * EP - ((j == 0) ? 0 : EP);
                if (j == sb - 1) {
                    c1[J] = 1.0;
                    upd[J] = SP * EP + SZ * EP - r * EP;   // the w_{s-1} slot
                } else if (j >= sb && j < 2 * sb) {
                    c1[J] = 1.0;
                    upd[J] = SP * EP + (j - sb - r) * EP;  // Z' row j - s
                    dnd[J] = J * 8 * EP;                   // (times c2 = 0)
                } else if (j >= 2 * sb) {
                    upd[J] = J * 8 * EP;                   // padding rows: zero (own, finite, values x 0)
                    dnd[J] = J * 8 * EP;
                }
            }
        }
        for (int it = (grp < ngroups ? grp : nit); it < nit; it += ngroups) {
            const int stg = it % NS;
            mbar_wait(&full[stg], (uint32_t)((it / NS) & 1));
            const double *sP = smem + (size_t)stg * stage_elems;
            const double *sWl = sP + SP * EP, *sDv = sWl + k.wlp;
            if constexpr (PAIRS) {
            // k-step pairs: lane (r, kk) loads the points 2kk, 2kk+1 of an 8-point
            // block with one 16-B load per row; k-step A takes the even points,
            // k-step B the odd ones (the dot over points is order-free), into
            // accumulator sets 2u and 2u+1
            for (int kp0 = wig; kp0 < KS2; kp0 += wpg * UP) {
#pragma unroll
              for (int u = 0; u < UP; ++u) {
                const int kp = kp0 + u * wpg;
                if (kp >= KS2) break;
                const int pt = kp * 8 + 2 * kk;
                const int o = r * EP + pt;
                double2 a[NB], b[NB];
#pragma unroll
                for (int i = 0; i < NB; ++i) a[i] = lds2(sP + o + (IL ? (r + i) * EP : i * 8 * EP));   // IL: row 2r + i
                constexpr int SX = 0, SY = (U > 1) ? 1 : 0;
                if constexpr (IL) {
                    const double2 p0 = lds2(sP + pt);
                    const double2 dn0 = lds2(sP + pt + ilo0), up1 = lds2(sP + pt + ilo1);
                    b[0].x = fma(a[1].x, c1[0], fma(dn0.x, c2[0], cs[0] * a[0].x));
                    b[0].y = fma(a[1].y, c1[0], fma(dn0.y, c2[0], cs[0] * a[0].y));
                    b[1].x = fma(up1.x, c1[1], fma(a[0].x, c2[1], cs[1] * a[1].x));
                    b[1].y = fma(up1.y, c1[1], fma(a[0].y, c2[1], cs[1] * a[1].y));
#pragma unroll
                    for (int i = 0; i < NB; ++i) cac[i] = fma(a[i].y, p0.y, fma(a[i].x, p0.x, cac[i]));
                    int t = 0;
#pragma unroll
                    for (int i = 0; i < NB; ++i)
#pragma unroll
                        for (int J = 0; J <= i; ++J, ++t) {
                            dmma(acc[(2 * u + SX) % U][t][0], acc[(2 * u + SX) % U][t][1], a[i].x, b[J].x);
                            dmma(acc[(2 * u + SY) % U][t][0], acc[(2 * u + SY) % U][t][1], a[i].y, b[J].y);
                        }
                    continue;
                }
                if constexpr (GS) {   // E = P^T P: tile (i, J <= i) from the A fragments alone
                    int t = 0;
#pragma unroll
                    for (int i = 0; i < NB; ++i)
#pragma unroll
                        for (int J = 0; J <= i; ++J, ++t) {
                            dmma(acc[(2 * u + SX) % U][t][0], acc[(2 * u + SX) % U][t][1], a[i].x, a[J].x);
                            dmma(acc[(2 * u + SY) % U][t][0], acc[(2 * u + SY) % U][t][1], a[i].y, a[J].y);
                        }
                    continue;
                }
                const double2 p0 = lds2(sP + pt);
#pragma unroll
                for (int J = 0; J < NB; ++J) {
                    const double2 up = lds2(sP + o + upd[J]);
                    const double2 dn = lds2(sP + o + dnd[J]);
                    if (VARM) {
                        const double2 m = lds2(sDv + pt), wl = lds2(sWl + pt);
                        const double wx = m.x * fma(up.x, c1[J], fma(dn.x, c2[J], cs[J] * a[J].x));
                        const double wy = m.y * fma(up.y, c1[J], fma(dn.y, c2[J], cs[J] * a[J].y));
                        b[J].x = (use_wl[J] != 0.0) ? wl.x : wx;   // branch-free select
                        b[J].y = (use_wl[J] != 0.0) ? wl.y : wy;
                    } else {
                        b[J].x = fma(up.x, c1[J], fma(dn.x, c2[J], cs[J] * a[J].x));
                        b[J].y = fma(up.y, c1[J], fma(dn.y, c2[J], cs[J] * a[J].y));
                    }
                }
#pragma unroll
                for (int i = 0; i < NB; ++i) cac[i] = fma(a[i].y, p0.y, fma(a[i].x, p0.x, cac[i]));
                int t = 0;
#pragma unroll
                for (int i = 0; i < NB; ++i)
#pragma unroll
                    for (int J = (PAP ? 0 : i); J < (PAP ? i + 1 : NB); ++J, ++t) {   // PAP: tile (i, J <= i)
                        dmma(acc[(2 * u + SX) % U][t][0], acc[(2 * u + SX) % U][t][1], a[i].x, b[J].x);
                        dmma(acc[(2 * u + SY) % U][t][0], acc[(2 * u + SY) % U][t][1], a[i].y, b[J].y);
                    }
              }
            }
            } else {
            for (int ks0 = wig; ks0 < KS; ks0 += wpg * U) {
#pragma unroll
              for (int u = 0; u < U; ++u) {
                const int ks = ks0 + u * wpg;
                if (ks >= KS) break;
                const int pt = ks * 4 + kk;
                const int o = r * EP + pt;
                double a[NB], b[NB];
#pragma unroll
                for (int i = 0; i < NB; ++i) a[i] = sP[o + i * 8 * EP];
                if constexpr (GS) {
                    int t = 0;
#pragma unroll
                    for (int i = 0; i < NB; ++i)
#pragma unroll
                        for (int J = 0; J <= i; ++J, ++t) dmma(acc[u][t][0], acc[u][t][1], a[i], a[J]);
                    continue;
                }
                const double p0 = sP[pt];
#pragma unroll
                for (int J = 0; J < NB; ++J) {
                    const double up = sP[o + upd[J]];
                    const double dn = sP[o + dnd[J]];
                    if (VARM) {
                        const double m = sDv[pt];
                        const double w = m * fma(up, c1[J], fma(dn, c2[J], cs[J] * a[J]));
                        b[J] = (use_wl[J] != 0.0) ? sWl[pt] : w;   // branch-free select
                    } else {
                        b[J] = fma(up, c1[J], fma(dn, c2[J], cs[J] * a[J]));
                    }
                }
#pragma unroll
                for (int i = 0; i < NB; ++i) cac[i] = fma(a[i], p0, cac[i]);
                int t = 0;
#pragma unroll
                for (int i = 0; i < NB; ++i)
#pragma unroll
                    for (int J = (PAP ? 0 : i); J < (PAP ? i + 1 : NB); ++J, ++t)
                        dmma(acc[u][t][0], acc[u][t][1], a[i], b[J]);
              }
            }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stg]);
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            cac[i] += __shfl_xor_sync(0xffffffffu, cac[i], 1);
            cac[i] += __shfl_xor_sync(0xffffffffu, cac[i], 2);
        }
    }
    __syncthreads();
    double *red = smem;
    if (warp > 0) {
        const int cw = warp - 1;
        constexpr int NTT = NT;
#pragma unroll
        for (int t = 0; t < NTT; ++t) {
#pragma unroll
            for (int u = 1; u < U; ++u) {   // fold the accumulator sets in a fixed order
                acc[0][t][0] += acc[u][t][0];
                acc[0][t][1] += acc[u][t][1];
            }
            red[((cw * NTT + t) * 32 + lane) * 2 + 0] = acc[0][t][0];
            red[((cw * NTT + t) * 32 + lane) * 2 + 1] = acc[0][t][1];
        }
        if (!GS && (lane & 3) == 0)
#pragma unroll
            for (int i = 0; i < NB; ++i) red[NCW * NTT * 64 + cw * SP + (IL ? 2 * (lane >> 2) + i : i * 8 + (lane >> 2))] = cac[i];
    }
    __syncthreads();
    const int nent = s * s + s;
    double *mypart = k.part + (int64_t)blockIdx.x * nent;
    constexpr int NTT = NT;
    if constexpr (GS) {
        // this CTA's E (lower triangle, row-major s x s after the reduction area),
        // then its partial Ghat and c by the Gram-space recurrence
        double *E = red + NCW * NTT * 64;
        for (int q = tid; q < NTT * 64; q += THREADS) {
            const int t = q >> 6, e = q & 63, ln = e >> 1, h = e & 1;
            double v = 0.0;
            for (int w = 0; w < NCW; ++w) v += red[((w * NTT + t) * 32 + ln) * 2 + h];
            int I = 0, J = 0, tt = t;
            for (int aa = 0; aa < NB; ++aa) {
                if (tt <= aa) { I = aa; J = tt; break; }
                tt -= aa + 1;
            }
            const int i = I * 8 + (ln >> 2), j = J * 8 + 2 * (ln & 3) + h;
            if (i < s && j <= i) E[i * s + j] = v;
        }
        __syncthreads();
        const double m2 = k.dm * k.inv_2theta, m1 = k.dm * k.inv_theta, ms = k.dm * k.sigma;
        for (int q = tid; q < s * s; q += THREADS) {
            const int j = q / s, i = q - j * s;   // entry (j, i), j <= i: p_i^T w_j
            if (j > i) continue;
            double v;
            if (j == s - 1) v = 0.0;                                                   // p_{s-1}^T A p_{s-1}: the dot-mode single step
            else if (j == 0) v = fma(i >= 1 ? E[i * s + 1] : E[s], m1, ms * E[i * s]);      // E_{i,1} (= E_{1,0} at i = 0)
            else {
                const double up = (j + 1 <= i) ? E[i * s + j + 1] : E[(j + 1) * s + i];   // E_{i,j+1}
                v = fma(up + E[i * s + j - 1], m2, ms * E[i * s + j]);
            }
            mypart[q] = v;
        }
        for (int i = tid; i < s; i += THREADS) mypart[s * s + i] = E[i * s];   // c_i = p_i^T p_0
    }
    for (int q = tid; q < (GS ? 0 : NTT * 64); q += THREADS) {
        const int t = q >> 6, e = q & 63, ln = e >> 1, h = e & 1;
        double v = 0.0;
        for (int w = 0; w < NCW; ++w) v += red[((w * NTT + t) * 32 + ln) * 2 + h];
        int I = 0, J = 0, tt = t;
        if (!PAP) {   // upper tiles (I, J >= I), row-major
            for (int aa = 0; aa < NB; ++aa) {
                if (tt < NB - aa) { I = aa; J = aa + tt; break; }
                tt -= NB - aa;
            }
        } else {      // lower tiles (I, J <= I), row-major
            for (int aa = 0; aa < NB; ++aa) {
                if (tt <= aa) { I = aa; J = tt; break; }
                tt -= aa + 1;
            }
        }
        if (IL) {   // rows 2r + I, columns 2c + J: even x even, odd x even, odd x odd
            const int i = 2 * (ln >> 2) + I, j = 2 * (2 * (ln & 3) + h) + J;
            if (i >= s || j >= s) continue;
            if (j <= i) mypart[j * s + i] = (i == s - 1 && j == s - 1) ? 0.0 : v;   // v = p_i^T w_j = Ghat_{j,i}
            else if (I != J) mypart[i * s + j] = v;                                  // mixed pair, j > i: Ghat_{i,j}
            continue;
        }
        const int i = I * 8 + (ln >> 2), j = J * 8 + 2 * (ln & 3) + h;
        if (i >= s || j >= s) continue;
        if (!PAP) {
            if (i <= j) mypart[i * s + j] = v;
        } else if (j <= i) {                   // v = p_i^T w_j = Ghat_{j,i}
            mypart[j * s + i] = (i == s - 1 && j == s - 1) ? 0.0 : v;   // the diagonal p_{s-1}^T A p_{s-1}: k_pap
        }
    }
    for (int i = tid; i < (GS ? 0 : s); i += THREADS) {
        double v = 0.0;
        for (int w = 0; w < NCW; ++w) v += red[NCW * NTT * 64 + w * SP + i];
        mypart[s * s + i] = v;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) is_last = atomicAdd(k.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    last_cta_sum(k.part, gridDim.x, s, k.out);
    if (tid == 0) *k.ticket = 0u;
}

// K2S -- the W-free Gram pass for small bases (s <= 8): a plain streaming
// kernel.  With one 8x8 DMMA tile per point the tensor-core pass is bound by
// its per-chunk pipeline, while here every thread streams point pairs with
// 16-B loads (s + 1 rows, + diag(M)), recovers w_j from the recurrence as
// K2R does, and keeps the s(s+1)/2 + s partial sums in registers.  Warp
// shuffles, then a fixed-order sum over the warps, then the last-CTA sum:
// deterministic for a given grid.
__host__ __device__ constexpr int k2s_threads(int S) { return S >= 7 ? 256 : 512; }   // registers

template <int S, bool VARM>
__global__ void __launch_bounds__(k2s_threads(S), 1)
    k2s(const double *__restrict__ P, const double *__restrict__ Wl, const double *__restrict__ Dv, int64_t vstride,
        K2RParams k, const DevState *st)
{
    PDL_ENTRY(st);
    constexpr int K2S_THREADS = k2s_threads(S);
    constexpr int NUP = S * (S + 1) / 2, NACC = NUP + S;
    __shared__ double red[K2S_THREADS / 32][NACC];
    __shared__ bool is_last;
    double g[NACC];
#pragma unroll
    for (int q = 0; q < NACC; ++q) g[q] = 0.0;
    double c1[S], c2[S], cs[S];
#pragma unroll
    for (int j = 0; j < S; ++j) {
        const bool rec = j < S - 1;
        const double mf = VARM ? 1.0 : k.dm;
        c1[j] = !rec ? 0.0 : (j == 0 ? k.inv_theta : k.inv_2theta) * mf;
        c2[j] = (rec && j > 0) ? k.inv_2theta * mf : 0.0;
        cs[j] = rec ? k.sigma * mf : 0.0;
    }
    const int64_t n2 = k.N >> 1, vs2 = vstride >> 1;
    const double2 *P2 = reinterpret_cast<const double2 *>(P);
    const double2 *W2 = reinterpret_cast<const double2 *>(Wl);
    const double2 *D2 = reinterpret_cast<const double2 *>(Dv);
    for (int64_t e = (int64_t)blockIdx.x * K2S_THREADS + threadIdx.x; e < n2; e += (int64_t)gridDim.x * K2S_THREADS) {
        double2 p[S + 1], w[S];
#pragma unroll
        for (int j = 0; j < S; ++j) p[j] = __ldcs(P2 + j * vs2 + e);
        p[S] = make_double2(0.0, 0.0);
        const double2 wl = __ldcs(W2 + e);
        const double2 m = VARM ? __ldcs(D2 + e) : make_double2(1.0, 1.0);
#pragma unroll
        for (int j = 0; j < S; ++j) {
            if (j == S - 1) {
                w[j] = wl;
            } else {
                const double2 up = p[j + 1], dn = (j > 0) ? p[j - 1] : make_double2(0.0, 0.0);
                double wx = fma(up.x, c1[j], fma(dn.x, c2[j], cs[j] * p[j].x));
                double wy = fma(up.y, c1[j], fma(dn.y, c2[j], cs[j] * p[j].y));
                if (VARM) {
                    wx *= m.x;
                    wy *= m.y;
                }
                w[j] = make_double2(wx, wy);
            }
        }
        int t = 0;
#pragma unroll
        for (int i = 0; i < S; ++i)
#pragma unroll
            for (int j = i; j < S; ++j, ++t) g[t] = fma(p[i].y, w[j].y, fma(p[i].x, w[j].x, g[t]));
#pragma unroll
        for (int i = 0; i < S; ++i) g[NUP + i] = fma(p[i].y, p[0].y, fma(p[i].x, p[0].x, g[NUP + i]));
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < NACC; ++q) {
        double v = g[q];
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        if (lane == 0) red[warp][q] = v;
    }
    __syncthreads();
    const int s = S, nent = s * s + s;
    double *mypart = k.part + (int64_t)blockIdx.x * nent;
    for (int q = threadIdx.x; q < NACC; q += K2S_THREADS) {
        double v = 0.0;
        for (int w8 = 0; w8 < K2S_THREADS / 32; ++w8) v += red[w8][q];
        if (q < NUP) {
            int i = 0, rem = q;
            while (rem >= s - i) { rem -= s - i; ++i; }
            mypart[i * s + i + rem] = v;
        } else {
            mypart[s * s + (q - NUP)] = v;
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = atomicAdd(k.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    last_cta_sum(k.part, gridDim.x, s, k.out);
    if (threadIdx.x == 0) *k.ticket = 0u;
}

int ep_for(int s_pad) { return s_pad <= 32 ? 132 : 68; }   // row pitch 32 mod 128 bytes (8-B fragment loads)
#ifndef K2R_EP_MID
#define K2R_EP_MID 132
#endif
#ifndef K2R_EP_PAIRS
#define K2R_EP_PAIRS 184   // 23 k-step pairs per stage; cfg 5: 136 -> 2.04 ms, 184 -> 2.00, 216 -> 2.20
#endif
int ep_for_k2r(int s_pad)   // pairs: 64 mod 128 B (16-B loads); single k-steps: 32 mod 128 B
{
    return s_pad <= 16 ? K2R_EP_PAIRS : s_pad <= 32 ? K2R_EP_MID : 68;
}

// consumer warp groups: each group works on its own stages, so the ring keeps
// nstage - ngroups stages in flight for TMA.  ngroups must divide both the
// consumer warps and nstage: then slot `it % nstage` is always consumed by
// group `it % ngroups`, in order, and a group can never wait on a slot whose
// previous phase (another group's) is still pending -- with shared slots a
// group running a full ring ahead would match the parity of an older phase.
int gcd_int(int a, int b) { return b ? gcd_int(b, a % b) : a; }


// largest g <= want dividing every value in {a, b}
int common_divisor_le(int want, int a, int b)
{
    int g = std::max(1, std::min(want, gcd_int(a, b)));
    while (a % g || b % g) --g;
    return g;
}

int stages_for(int s_pad, int ep)
{
    const size_t stage = (size_t)2 * s_pad * ep * sizeof(double);
    return (int)std::max<size_t>(2, std::min<size_t>(MAXS, (200 * 1024) / stage));
}

}  // namespace

bool k2d_enabled(const Geo &g, int s)
{
    if (g.kn.k2_dmma == 0) return false;   // SSCG_K2_DMMA: "0" never, "1" always, unset: s > 16
    if (g.kn.k2_dmma == 1) return s >= 1;
    return s > 16;
}

bool encode_rows_map(CUtensorMap *m, const double *base, int64_t inner, int rows, int64_t stride, int box_inner,
                     int box_rows);

bool k2d_prepare(const Geo &g, Slab &sl, int s)
{
    const int s_pad = (s + 7) / 8 * 8, ep = ep_for(s_pad);
    const int64_t N = (int64_t)sl.nzl * g.plane;
    const int mx = 210 * 1024;
#define K2D_ATTR(NB, EP) cudaFuncSetAttribute(k2d<NB, EP>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess
    if (K2D_ATTR(1, 132) || K2D_ATTR(2, 132) || K2D_ATTR(3, 132) || K2D_ATTR(4, 132) || K2D_ATTR(5, 68) ||
        K2D_ATTR(6, 68) || K2D_ATTR(7, 68) || K2D_ATTR(8, 68))
        return false;
#undef K2D_ATTR
    return encode_rows_map(&sl.tmPd, sl.P + g.plane, N, s, g.vstride, ep, s_pad) &&
           encode_rows_map(&sl.tmWd, sl.W + g.plane, N, s, g.vstride, ep, s_pad);
}

void launch_k2d(const Geo &g, const Slab &sl, int s, const DevState *st, double *out_blk, cudaStream_t stream)
{
    const int s_pad = (s + 7) / 8 * 8, nb = s_pad / 8, ep = ep_for(s_pad);
    K2DParams k;
    k.N = (int64_t)sl.nzl * g.plane;
    k.s = s;
    k.s_pad = s_pad;
    k.nstage = stages_for(s_pad, ep);
    k.ngroups = common_divisor_le(g.kn.k2_groups ? g.kn.k2_groups : k.nstage, k.nstage, ncw_for(nb));
    k.part = sl.part;
    k.out = out_blk;
    k.ticket = sl.ticket;
    const int64_t nchunks = (k.N + ep - 1) / ep;
    const int gx = (int)std::min<int64_t>(k2_grid(), nchunks);
    const int nt = nb * (nb + 1) / 2;
    const size_t ring = (size_t)k.nstage * 2 * s_pad * ep * sizeof(double);
    const size_t red = (size_t)(ncw_for(nb) * nt * 64 + ncw_for(nb) * s_pad) * sizeof(double);   // cross-warp reduction
    const size_t sm = std::max(ring, red);
    switch (nb) {
    case 1: launch_pdl(g.kn.pdl, k2d<1, 132>, dim3(gx), dim3(threads_for(1)), sm, stream, sl.tmPd, sl.tmWd, k, st); break;
    case 2: launch_pdl(g.kn.pdl, k2d<2, 132>, dim3(gx), dim3(threads_for(2)), sm, stream, sl.tmPd, sl.tmWd, k, st); break;
    case 3: launch_pdl(g.kn.pdl, k2d<3, 132>, dim3(gx), dim3(threads_for(3)), sm, stream, sl.tmPd, sl.tmWd, k, st); break;
    case 4: launch_pdl(g.kn.pdl, k2d<4, 132>, dim3(gx), dim3(threads_for(4)), sm, stream, sl.tmPd, sl.tmWd, k, st); break;
    case 5: launch_pdl(g.kn.pdl, k2d<5, 68>, dim3(gx), dim3(threads_for(5)), sm, stream, sl.tmPd, sl.tmWd, k, st); break;
    case 6: launch_pdl(g.kn.pdl, k2d<6, 68>, dim3(gx), dim3(threads_for(6)), sm, stream, sl.tmPd, sl.tmWd, k, st); break;
    case 7: launch_pdl(g.kn.pdl, k2d<7, 68>, dim3(gx), dim3(threads_for(7)), sm, stream, sl.tmPd, sl.tmWd, k, st); break;
    default: launch_pdl(g.kn.pdl, k2d<8, 68>, dim3(gx), dim3(threads_for(8)), sm, stream, sl.tmPd, sl.tmWd, k, st); break;
    }
}

}  // namespace sscg

namespace sscg {

// BLK: the box pitch (k-step pairs for up to 16 rows: 72 = 64 mod 128 B; single
// k-steps above: 68 = 32 mod 128 B)
static int ep_for_k2rb(int sp) { return sp <= 16 ? 72 : 68; }

bool k2r_prepare(const Geo &g, Slab &sl, int s, int nvec)
{
    const int s_pad = (s + 7) / 8 * 8, ep = ep_for_k2r(s_pad);
    const int64_t N = (int64_t)sl.nzl * g.plane;
    const int mx = 226 * 1024;
#define K2R_ATTR(NB, EP, V) cudaFuncSetAttribute(k2r<NB, EP, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess
    if (K2R_ATTR(1, K2R_EP_PAIRS, false) || K2R_ATTR(2, K2R_EP_PAIRS, false) || K2R_ATTR(3, K2R_EP_MID, false) || K2R_ATTR(4, K2R_EP_MID, false) ||
        K2R_ATTR(5, 68, false) || K2R_ATTR(6, 68, false) || K2R_ATTR(7, 68, false) || K2R_ATTR(8, 68, false) ||
        K2R_ATTR(1, K2R_EP_PAIRS, true) || K2R_ATTR(2, K2R_EP_PAIRS, true) || K2R_ATTR(3, K2R_EP_MID, true) || K2R_ATTR(4, K2R_EP_MID, true) ||
        K2R_ATTR(5, 68, true) || K2R_ATTR(6, 68, true) || K2R_ATTR(7, 68, true) || K2R_ATTR(8, 68, true))
        return false;
#undef K2R_ATTR
#define K2R_ATTR_F(NB, EP) (cudaFuncSetAttribute(k2r<NB, EP, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess || \
                            cudaFuncSetAttribute(k2r<NB, EP, false, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess || \
                            cudaFuncSetAttribute(k2r<2, K2R_EP_PAIRS, false, true, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess)
    if (K2R_ATTR_F(1, K2R_EP_PAIRS) || K2R_ATTR_F(2, K2R_EP_PAIRS) || K2R_ATTR_F(3, K2R_EP_MID) || K2R_ATTR_F(4, K2R_EP_MID))
        return false;
#undef K2R_ATTR_F
    // the block-conjugate mode's W-free pass over [P_k | Q'] x [W_k | Z'] (2s <= 32 rows)
    sl.has_k2rb = false;
    if (nvec >= 2 * s && 2 * s <= 32) {
#define K2R_ATTR_B(NB, EP) cudaFuncSetAttribute(k2r<NB, EP, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess
        if (K2R_ATTR_B(1, 72) || K2R_ATTR_B(2, 72) || K2R_ATTR_B(3, 68) || K2R_ATTR_B(4, 68)) return false;
#undef K2R_ATTR_B
        const int spb = (2 * s + 7) / 8 * 8, epb = ep_for_k2rb(spb);
        if (!encode_rows_map(&sl.tmPb, sl.P + g.plane, N, 2 * s, g.vstride, epb, spb) ||
            !encode_rows_map(&sl.tmZb, sl.W + (int64_t)s * g.vstride + g.plane, N, s, g.vstride, epb, spb / 2) ||
            !encode_rows_map(&sl.tmWlb, sl.W + g.plane, N, s, g.vstride, epb, 1))
            return false;
        sl.has_k2rb = true;
    }
    // P rows (own map: K2D's pitch differs), the single row w_{s-1} of W, and diag(M) (one row) when it varies
    if (!encode_rows_map(&sl.tmPr, sl.P + g.plane, N, s, g.vstride, ep, s_pad)) return false;
    if (!encode_rows_map(&sl.tmWl, sl.W + g.plane, N, s, g.vstride, ep, 1)) return false;
    if (sl.dvec && !encode_rows_map(&sl.tmDv, sl.dvec + g.plane, N, 1, g.vstride, ep, 1)) return false;
    return true;
}

namespace {
// w_j of one slab recovered from the recurrence into `out` (padded interior),
// the same formula as the K2R fragments (parity hooks read W through this)
__global__ void k_wrec(const double *P, int64_t vstride, int64_t N, int j, double inv_theta, double inv_2theta,
                       double sigma, double dm, const double *dvec, double *out)
{
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x) {
        const double m = dvec ? dvec[e] : dm;
        const double pj = P[j * vstride + e], up = P[(j + 1) * vstride + e];
        out[e] = (j == 0) ? m * (up * inv_theta + sigma * pj)
                          : m * ((up + P[(j - 1) * vstride + e]) * inv_2theta + sigma * pj);
    }
}
}  // namespace

void launch_wrec(const Geo &g, const Slab &sl, int j, double theta, double sigma, double *out, cudaStream_t stream)
{
    const int64_t N = (int64_t)sl.nzl * g.plane;
    const int blocks = (int)std::min<int64_t>((N + 255) / 256, 148 * 16);
    k_wrec<<<blocks, 256, 0, stream>>>(sl.P + g.plane, g.vstride, N, j, 1.0 / theta, 1.0 / (2.0 * theta), sigma,
                                       g.center, sl.dvec ? sl.dvec + g.plane : nullptr, out + g.plane);
}

void launch_k2r(const Geo &g, const Slab &sl, int s, double theta, double sigma, const DevState *st, double *out_blk,
                cudaStream_t stream, bool fold)
{
    const int s_pad = (s + 7) / 8 * 8, nb = s_pad / 8, ep = ep_for_k2r(s_pad);
    const bool varm = sl.dvec != nullptr;
    fold = fold && !varm && nb <= 4;   // (the capi asks for it only then: uses_wlfold)
    K2RParams k;
    k.N = (int64_t)sl.nzl * g.plane;
    if (g.kn.k2s && s >= 2 && s <= 8 && !fold) {
        k.s = s;
        k.inv_theta = 1.0 / theta;
        k.inv_2theta = 1.0 / (2.0 * theta);
        k.sigma = sigma;
        k.dm = g.center;
        k.part = sl.part;
        k.out = out_blk;
        k.ticket = sl.ticket;
        const double *P = sl.P + g.plane, *Wl = sl.W + (int64_t)(s - 1) * g.vstride + g.plane;
        const double *Dv = varm ? sl.dvec + g.plane : nullptr;
        const int nth = k2s_threads(s);
#ifndef K2S_BLOCKS_PER_SM
#define K2S_BLOCKS_PER_SM 1   // measured: 2, 4, 8 slower (the last-CTA sum grows)
#endif
        // the partial buffer holds 8 blocks per SM
        const int gx = (int)std::max<int64_t>(
            1, std::min<int64_t>((int64_t)k2_grid() * std::min(8, K2S_BLOCKS_PER_SM), (k.N / 2 + nth - 1) / nth));
#define K2S_LAUNCH(S)                                                                                            \
        if (varm) launch_pdl(g.kn.pdl, k2s<S, true>, dim3(gx), dim3(nth), 0, stream, P, Wl, Dv, g.vstride, k, st);                            \
        else launch_pdl(g.kn.pdl, k2s<S, false>, dim3(gx), dim3(nth), 0, stream, P, Wl, Dv, g.vstride, k, st);
        switch (s) {
        case 2: K2S_LAUNCH(2) break;
        case 3: K2S_LAUNCH(3) break;
        case 4: K2S_LAUNCH(4) break;
        case 5: K2S_LAUNCH(5) break;
        case 6: K2S_LAUNCH(6) break;
        case 7: K2S_LAUNCH(7) break;
        default: K2S_LAUNCH(8) break;
        }
#undef K2S_LAUNCH
        return;
    }
    k.s = s;
    k.s_pad = s_pad;
    k.wlp = (ep * 8 + 127) / 128 * 128 / 8;
    const size_t stage = (size_t)(s_pad * ep + k.wlp * (varm ? 2 : 1)) * sizeof(double);
    const int smem_kb = g.kn.k2_smem_kb;
    {
        // 4 groups by default (each with nstage/4 slots), nstage a multiple of the groups
        const int nsmax = (int)std::max<size_t>(1, std::min<size_t>(MAXS, ((size_t)smem_kb * 1024) / stage));
        const int gr = common_divisor_le(g.kn.k2_groups ? g.kn.k2_groups : 4, ncw_for(nb, varm), ncw_for(nb, varm));
        k.ngroups = std::min(gr, nsmax);
        while (ncw_for(nb, varm) % k.ngroups) --k.ngroups;
        k.nstage = std::max(k.ngroups, nsmax / k.ngroups * k.ngroups);
    }
    k.inv_theta = 1.0 / theta;
    k.inv_2theta = 1.0 / (2.0 * theta);
    k.sigma = sigma;
    k.dm = g.center;
    k.part = sl.part;
    k.out = out_blk;
    k.ticket = sl.ticket;
    const int64_t nchunks = (k.N + ep - 1) / ep;
    const int gx = (int)std::min<int64_t>(k2_grid(), nchunks);
    const int nt = nb * (nb + 1) / 2;
    const size_t red = (size_t)(ncw_for(nb, varm) * nt * 64 + std::max(ncw_for(nb, varm) * s_pad, s * s)) * sizeof(double);
    const size_t sm = std::max((size_t)k.nstage * stage, red);
    const CUtensorMap &dv = varm ? sl.tmDv : sl.tmWl;
    if (fold) {
#define K2R_LAUNCH_F(NB, EP)                                                                                 \
        if (g.kn.gram_space) launch_pdl(g.kn.pdl, k2r<NB, EP, false, true, false, true>, dim3(gx), dim3(threads_for(NB, false)), sm, stream, sl.tmPr, sl.tmWl, dv, k, st); \
        else if (NB == 2 && g.kn.k2_il && s % 2 == 0) launch_pdl(g.kn.pdl, k2r<2, EP, false, true, false, false, true>, dim3(gx), dim3(threads_for(2, false)), sm, stream, sl.tmPr, sl.tmWl, dv, k, st); \
        else launch_pdl(g.kn.pdl, k2r<NB, EP, false, true>, dim3(gx), dim3(threads_for(NB, false)), sm, stream, sl.tmPr, sl.tmWl, dv, k, st);
        switch (nb) {
        case 1: K2R_LAUNCH_F(1, K2R_EP_PAIRS) break;
        case 2: K2R_LAUNCH_F(2, K2R_EP_PAIRS) break;
        case 3: K2R_LAUNCH_F(3, K2R_EP_MID) break;
        default: K2R_LAUNCH_F(4, K2R_EP_MID) break;
        }
#undef K2R_LAUNCH_F
        return;
    }
#define K2R_LAUNCH(NB, EP)                                                                                   \
    if (varm) launch_pdl(g.kn.pdl, k2r<NB, EP, true>, dim3(gx), dim3(threads_for(NB, true)), sm, stream, sl.tmPr, sl.tmWl, dv, k, st);          \
    else launch_pdl(g.kn.pdl, k2r<NB, EP, false>, dim3(gx), dim3(threads_for(NB, false)), sm, stream, sl.tmPr, sl.tmWl, dv, k, st);
    switch (nb) {
    case 1: K2R_LAUNCH(1, K2R_EP_PAIRS) break;
    case 2: K2R_LAUNCH(2, K2R_EP_PAIRS) break;
    case 3: K2R_LAUNCH(3, K2R_EP_MID) break;
    case 4: K2R_LAUNCH(4, K2R_EP_MID) break;
    case 5: K2R_LAUNCH(5, 68) break;
    case 6: K2R_LAUNCH(6, 68) break;
    case 7: K2R_LAUNCH(7, 68) break;
    default: K2R_LAUNCH(8, 68) break;
    }
#undef K2R_LAUNCH
}

// the block-conjugate mode's Gram pass without the stored W_k (BLK, above):
// 2s rows [P_k | Q'] x [W_k | Z'] into the (2s) x (2s + 1) block
void launch_k2r_block(const Geo &g, const Slab &sl, int s, double theta, double sigma, const DevState *st,
                      double *out_blk, cudaStream_t stream)
{
    const int sp = (2 * s + 7) / 8 * 8, nb = sp / 8, ep = ep_for_k2rb(sp);
    K2RParams k{};
    k.N = (int64_t)sl.nzl * g.plane;
    k.s = 2 * s;
    k.sb = s;
    k.s_pad = sp;
    k.wlp = (ep * 8 + 127) / 128 * 128 / 8;
    const size_t stage = (size_t)(sp * ep + (sp / 2) * ep + k.wlp) * sizeof(double);
    {
        const int nsmax = (int)std::max<size_t>(1, std::min<size_t>(MAXS, ((size_t)g.kn.k2_smem_kb * 1024) / stage));
        const int gr = common_divisor_le(g.kn.k2_groups ? g.kn.k2_groups : 4, ncw_for(nb), ncw_for(nb));
        k.ngroups = std::min(gr, nsmax);
        while (ncw_for(nb) % k.ngroups) --k.ngroups;
        k.nstage = std::max(k.ngroups, nsmax / k.ngroups * k.ngroups);
    }
    k.inv_theta = 1.0 / theta;
    k.inv_2theta = 1.0 / (2.0 * theta);
    k.sigma = sigma;
    k.dm = g.center;
    k.part = sl.part;
    k.out = out_blk;
    k.ticket = sl.ticket;
    const int64_t nchunks = (k.N + ep - 1) / ep;
    const int gx = (int)std::min<int64_t>(k2_grid(), nchunks);
    const int nt = nb * (nb + 1) / 2;
    const size_t red = (size_t)(ncw_for(nb) * nt * 64 + ncw_for(nb) * sp) * sizeof(double);
    const size_t sm = std::max((size_t)k.nstage * stage, red);
    switch (nb) {
    case 1: launch_pdl(g.kn.pdl, k2r<1, 72, false, false, true>, dim3(gx), dim3(threads_for(1)), sm, stream, sl.tmPb, sl.tmWlb, sl.tmZb, k, st); break;
    case 2: launch_pdl(g.kn.pdl, k2r<2, 72, false, false, true>, dim3(gx), dim3(threads_for(2)), sm, stream, sl.tmPb, sl.tmWlb, sl.tmZb, k, st); break;
    case 3: launch_pdl(g.kn.pdl, k2r<3, 68, false, false, true>, dim3(gx), dim3(threads_for(3)), sm, stream, sl.tmPb, sl.tmWlb, sl.tmZb, k, st); break;
    default: launch_pdl(g.kn.pdl, k2r<4, 68, false, false, true>, dim3(gx), dim3(threads_for(4)), sm, stream, sl.tmPb, sl.tmWlb, sl.tmZb, k, st); break;
    }
}

namespace {
// k_pap (the w_{s-1} fold without TMA; the TMA path runs the K1T single step
// in its dot mode): Ghat_{s-1,s-1} = p_{s-1}^T A p_{s-1} over one slab, A the
// 7-point stencil with a constant centre (zero outside the grid in x and y;
// the ghost planes carry the z-neighbours), each A p formed in the order of
// the single step it replaces: c p - (p_{z-1} + p_{y-1} + p_{x-1} + p_{x+1} +
// p_{y+1} + p_{z+1}).  A block owns a 64 x 16 tile of columns and marches a
// z-chunk: warp = row, lane = point pair; p(z-1), p(z) ride in registers, so
// per plane only p(z+1) streams from HBM and the in-plane neighbours are L1
// hits (a grid-stride pass with all six neighbour loads ran 0.27 ms at 448^3:
// L2-bound; this one 0.22 ms over tile heights 4..32 and 4..16 blocks per SM).
// Per-block partials in a fixed order, then the last block sums them in index
// order (deterministic) into the slab's Gram block entry.
constexpr int PAP_TX = 64, PAP_TY = 16, PAP_THREADS = 32 * PAP_TY;

__global__ void __launch_bounds__(PAP_THREADS) k_pap(const double *p, int nx, int ny, int nzl, int64_t plane, int zc,
                                                     int tiles_x, int nitems, double center, double *part,
                                                     unsigned *ticket, double *entry, const DevState *st)
{
    PDL_ENTRY(st);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ntiles = tiles_x * ((ny + PAP_TY - 1) / PAP_TY);
    double acc = 0.0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {   // items: tile x z-chunk
        const int tile = item % ntiles, chunk = item / ntiles;
        const int x = (tile % tiles_x) * PAP_TX + 2 * lane, y = (tile / tiles_x) * PAP_TY + warp;
        const int zb = 1 + chunk * zc, ze = min(nzl + 1, zb + zc);
        if (x >= nx || y >= ny || zb >= ze) continue;
        // p points at plane 0 (the lower ghost plane) of p_{s-1}
        const double *col = p + (int64_t)y * nx + x;
        double2 dn = __ldg(reinterpret_cast<const double2 *>(col + (int64_t)(zb - 1) * plane));
        double2 c = __ldg(reinterpret_cast<const double2 *>(col + (int64_t)zb * plane));
        const bool hl = x > 0, hr = x + 2 < nx, hy0 = y > 0, hy1 = y + 1 < ny;
#pragma unroll 4
        for (int z = zb; z < ze; ++z) {
            const double *pc = col + (int64_t)z * plane;
            const double2 up = __ldg(reinterpret_cast<const double2 *>(pc + plane));
            const double l = hl ? __ldg(pc - 1) : 0.0, rr = hr ? __ldg(pc + 2) : 0.0;
            const double2 z0 = make_double2(0.0, 0.0);
            const double2 ylo = hy0 ? __ldg(reinterpret_cast<const double2 *>(pc - nx)) : z0;
            const double2 yhi = hy1 ? __ldg(reinterpret_cast<const double2 *>(pc + nx)) : z0;
            const double ax = center * c.x - (dn.x + ylo.x + l + c.y + yhi.x + up.x);
            const double ay = center * c.y - (dn.y + ylo.y + c.x + rr + yhi.y + up.y);
            acc = fma(c.x, ax, acc);
            acc = fma(c.y, ay, acc);
            dn = c;
            c = up;
        }
    }
    __shared__ double red[PAP_THREADS / 32];
    __shared__ bool is_last;
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < PAP_THREADS / 32; ++w) v += red[w];
        part[blockIdx.x] = v;
        __threadfence();
        is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    if (threadIdx.x < 32) {   // lane m sums partials m, m+32, ... in order, then a fixed xor tree
        double v = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) v += __ldcg(part + b);
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) {
            *entry = v;
            *ticket = 0u;
        }
    }
}
}  // namespace

// items: tiles x z-chunks, the chunk length chosen for about 8 blocks per SM
// (one wave); the grid (one partial per block) at most k2_grid() * 8 blocks,
// which the partial buffer always holds
void launch_pap(const Geo &g, const Slab &sl, int s, const DevState *st, double *out_blk, cudaStream_t stream)
{
    const int tiles_x = (g.nx + PAP_TX - 1) / PAP_TX, tiles = tiles_x * ((g.ny + PAP_TY - 1) / PAP_TY);
    const int64_t want = (int64_t)k2_grid() * 8;
    int nch = (int)std::max<int64_t>(1, std::min<int64_t>(sl.nzl, want / tiles));
    const int zc = (sl.nzl + nch - 1) / nch;
    nch = (sl.nzl + zc - 1) / zc;
    const int nitems = tiles * nch, grid = (int)std::min<int64_t>(nitems, want);
    launch_pdl(g.kn.pdl, k_pap, dim3((unsigned)grid), dim3(PAP_THREADS), 0, stream,
               (const double *)(sl.P + (int64_t)(s - 1) * g.vstride), g.nx, g.ny, sl.nzl, g.plane, zc, tiles_x,
               nitems, g.center, sl.part, sl.ticket, out_blk + (int64_t)(s - 1) * s + (s - 1), st);
}

}  // namespace sscg
