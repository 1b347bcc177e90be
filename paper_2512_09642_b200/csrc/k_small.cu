// KS -- one whole outer iteration in ONE launch of ONE thread-block cluster
// (8 CTAs x 512 threads), for problems whose working set fits the cluster's
// shared memory (BASELINE cfg 1: 2D 64 x 64, s = 8; "a latency
// measurement").  At that size every kernel of the multi-kernel schedule is a
// partial wave whose launch and fill/drain dominate (11 launches, 33 us per
// outer iteration, profiles/r02f_launches_cfg1_*); here the steps are
// separated by cluster barriers instead of kernel boundaries:
//   basis  j = 0..s-1   w_j = A p_j, p_{j+1} = c_j (D^{-1} w_j - sigma p_j) [- p_{j-1}]
//                        on P and W held in the cluster's
//                       distributed shared memory
//   Gram               Ghat = P^T W (i <= j), c = P^T p_0 by
//                       FP64 DMMA per warp, fixed-order sums over warps and CTAs
//   K4 (CTA 0, warp 0)  stopping test, Ruhe scaling, nu FGS sweeps -- the same
//                       k4_small.cuh body as the one-warp K4 kernel (the other
//                       warps meanwhile copy P and W to global memory)
//   update              x += P alpha, r_{k+1} = p_0 - W alpha into p_0
// 5-point 2D and 7-point 3D constant stencils, Chebyshev basis, s <= 8, at most
// 8192 points, one slab, no communicator, FGS solver.  Measured (tools/
// ks_timing.py with a KS_TIMING build): basis 4.3 us (8 barriers), Gram 2.0,
// K4 6.3, update 2.1 -- 18.6 us per outer iteration under graph replay.
#include <cooperative_groups.h>
#include <cstdio>

#include <algorithm>

#include "sscg_internal.cuh"
#include "k4_small.cuh"

namespace sscg {
namespace {

namespace cg = cooperative_groups;

// KS_TIMING (variant builds only): CTA 0 prints the %globaltimer ns at each phase boundary
#ifdef KS_TIMING
__device__ __forceinline__ unsigned long long gtime()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define KS_T(i) if (rank == 0 && threadIdx.x == 0) tt[i] = gtime();
#else
#define KS_T(i)
#endif

constexpr int KS_CL = 8;          // CTAs per cluster (portable size); the steps are separated by cluster barriers
constexpr int KS_THREADS = 512;
constexpr int KS_PPT = 2;         // points per thread (at most)
constexpr int KS_MAXPTS = KS_CL * KS_THREADS * KS_PPT;   // 8192

struct KSArgs {
    double *P, *W;         // interior start (plane 1) of vector 0; vectors vstride apart
    int64_t vstride;
    int nx, ny, nzl, pitch;
    int64_t plane;
    double center, dinv_c, theta, sigma;
    double *const *xpp;    // device cell with the caller's x
};

// One cluster of KS_CL CTAs.  CTA r owns the points [r*ppc, (r+1)*ppc) of the
// slab (ppc = ceil(npts / KS_CL)); thread t of it the points r*ppc + t +
// KS_THREADS*u.  Each CTA keeps P and W of its own points in shared memory
// (dense, [S][ppc] each), so the basis steps, the Gram pass and the update
// read only shared memory; a stencil neighbour owned by another CTA is read
// through distributed shared memory (pointers resolved once per point).  The
// cluster barriers between the basis steps then order only shared-memory
// traffic; P and W are copied to global memory once (the parity hooks read
// them there), p_0 = r_{k+1} and x are written back by the update.
template <int S, int KIND>
__global__ void __launch_bounds__(KS_THREADS, 1) k_small(KSArgs a, K4Args k4, DevState *st)
{
    PDL_ENTRY(st);
    constexpr int NW = KS_THREADS / 32;
    extern __shared__ __align__(16) double loc[];   // P [S][ppc] | W [S][ppc]
    __shared__ double red[NW][72];                  // per-warp 8 x 8 Ghat tile + 8 entries of c
    __shared__ double part[72];                     // this CTA's Gram partials (read by CTA 0)
    __shared__ double scratch[S * S + S + 64];      // CTA 0: the block, K4's staging area
    __shared__ double alsh[S];                      // CTA 0: alpha (read by every CTA)
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
#ifdef KS_TIMING
    unsigned long long tt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
    KS_T(0)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nx = a.nx, ny = a.ny;
    const int npts = nx * ny * a.nzl, nxy = nx * ny;
    const int ppc = (npts + KS_CL - 1) / KS_CL;
    double *Pl = loc, *Wl = loc + (size_t)S * ppc;
    const int64_t vs = a.vstride, pl = a.plane;
    constexpr int NB = (KIND == 1) ? 6 : 4;
    int off[KS_PPT], ge[KS_PPT];   // padded offset and global point index (-1: none)
    const double *nbp[KS_PPT][NB]; // neighbour in slot 0 of its owner's P (nullptr: Dirichlet)
#pragma unroll
    for (int u = 0; u < KS_PPT; ++u) {
        const int le = tid + KS_THREADS * u, e = rank * ppc + le;
        off[u] = -1;
        ge[u] = -1;
#pragma unroll
        for (int q = 0; q < NB; ++q) nbp[u][q] = nullptr;
        if (le < ppc && e < npts) {
            const int xx = e % nx, y = (e / nx) % ny, z = e / nxy;
            off[u] = (int)((int64_t)z * pl + (int64_t)y * a.pitch + xx);
            ge[u] = e;
            const int nbe[6] = {e - 1, e + 1, e - nx, e + nx, e - nxy, e + nxy};
            const bool ok[6] = {xx > 0, xx + 1 < nx, y > 0, y + 1 < ny, z > 0, z + 1 < a.nzl};
#pragma unroll
            for (int q = 0; q < NB; ++q)
                if (ok[q]) {
                    const int r = nbe[q] / ppc;
                    nbp[u][q] = cluster.map_shared_rank(Pl, r) + (nbe[q] - r * ppc);
                }
            Pl[le] = a.P[off[u]];   // p_0
        }
    }
    cluster.sync();
    KS_T(1)
    // ---- basis: s steps of the three-term recurrence, all operands in (distributed) shared memory ----
#pragma unroll 1
    for (int j = 0; j < S; ++j) {
        const double cf = (j == 0) ? a.theta : 2.0 * a.theta;
        const int oj = j * ppc;
#pragma unroll
        for (int u = 0; u < KS_PPT; ++u) {
            if (off[u] < 0) continue;
            const int le = tid + KS_THREADS * u;
            const double c = Pl[oj + le];
            double nb = 0.0;
            // the neighbour order of the other basis kernels: z, y, x
            if (KIND == 1) {
                if (nbp[u][4]) nb += nbp[u][4][oj];
                if (nbp[u][5]) nb += nbp[u][5][oj];
            }
            if (nbp[u][2]) nb += nbp[u][2][oj];
            if (nbp[u][3]) nb += nbp[u][3][oj];
            if (nbp[u][0]) nb += nbp[u][0][oj];
            if (nbp[u][1]) nb += nbp[u][1][oj];
            const double Ap = a.center * c - nb;
            Wl[oj + le] = Ap;
            if (j < S - 1) {
                double v = cf * (a.dinv_c * Ap - a.sigma * c);
                if (j > 0) v -= Pl[oj - ppc + le];
                Pl[oj + ppc + le] = v;
            }
        }
        cluster.sync();
    }
    KS_T(2)
    // ---- Gram block on FP64 tensor cores: each warp runs DMMA k-steps of 4 of
    // its points -- A = the basis rows P^T (8 x 4), B = W (4 x 8) for Ghat and
    // B = P for c = P^T p_0 (column 0) -- then a fixed-order sum over the warps ----
    double g0 = 0.0, g1 = 0.0, h0 = 0.0, h1 = 0.0;
    {
        const int fi = lane >> 2, fk = lane & 3;   // A: row i, col k;  B: row k, col j = fi
#pragma unroll
        for (int u = 0; u < KS_PPT; ++u) {
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int le = u * KS_THREADS + warp * 32 + ks * 4 + fk;
                const bool v = le < ppc && rank * ppc + le < npts && fi < S;
                const double av = v ? Pl[fi * ppc + le] : 0.0;
                const double bw = v ? Wl[fi * ppc + le] : 0.0;
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(g0), "+d"(g1) : "d"(av), "d"(bw));
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(h0), "+d"(h1) : "d"(av), "d"(av));
            }
        }
    }
    {
        // D fragment: lane holds (row lane/4, cols 2*(lane%4) + {0, 1})
        const int r = lane >> 2, c0 = 2 * (lane & 3);
        red[warp][r * 8 + c0] = g0;
        red[warp][r * 8 + c0 + 1] = g1;
        if (c0 == 0) red[warp][64 + r] = h0;   // (P^T P)_{r,0} = p_r^T p_0
    }
    __syncthreads();
    for (int q = tid; q < 72; q += KS_THREADS) {
        double v = 0.0;
        for (int w8 = 0; w8 < NW; ++w8) v += red[w8][q];
        part[q] = v;
    }
    cluster.sync();
    KS_T(3)
    if (rank == 0 && warp == 0) {
        // the block (CTA partials summed in rank order) into K4's staging area:
        // Ghat_ij for i <= j (mirrored), c_i
        for (int q = lane; q < 72; q += 32) {
            const int i = (q < 64) ? q >> 3 : q - 64, jj = (q < 64) ? q & 7 : 0;
            if (i >= S || jj >= S || (q < 64 && i > jj)) continue;
            double v = 0.0;
            for (int r = 0; r < KS_CL; ++r) v += cluster.map_shared_rank(part, r)[q];
            if (q < 64) {
                scratch[i * S + jj] = v;
                scratch[jj * S + i] = v;
            } else {
                scratch[S * S + i] = v;
            }
        }
        __syncwarp();
        // ---- K4: stopping test, scaling, nu FGS sweeps ----
        k4_fgs_small<(S + 3) / 4, true>(k4, st, scratch);
        __syncwarp();
        if (lane < S) alsh[lane] = __ldcg(k4.alpha + lane);
    } else {
        // meanwhile every other warp copies its points' basis to global memory
        // (the parity hooks read P and W there; p_0 is rewritten by the update)
        const int nth = (rank == 0) ? KS_THREADS - 32 : KS_THREADS, t0 = (rank == 0) ? tid - 32 : tid;
        for (int q = t0; q < S * ppc; q += nth) {
            const int j = q / ppc, le = q - j * ppc, e = rank * ppc + le;
            if (e >= npts) continue;
            const int xx = e % nx, y = (e / nx) % ny, z = e / nxy;
            const int64_t o = (int64_t)z * pl + (int64_t)y * a.pitch + xx + (int64_t)j * vs;
            a.P[o] = Pl[q];
            a.W[o] = Wl[q];
        }
    }
    cluster.sync();
    KS_T(4)
    if (*(volatile int *)&st->done) return;
    // ---- update: x += P alpha, r_{k+1} = p_0 - W alpha (into p_0) ----
    double al[S];
    const double *al0 = cluster.map_shared_rank(alsh, 0);
#pragma unroll
    for (int j = 0; j < S; ++j) al[j] = al0[j];
    double *x = *a.xpp;
#pragma unroll
    for (int u = 0; u < KS_PPT; ++u) {
        if (off[u] < 0) continue;
        const int le = tid + KS_THREADS * u;
        double ax = 0.0, aw = 0.0;
#pragma unroll
        for (int j = 0; j < S; ++j) {
            ax = fma(al[j], Pl[j * ppc + le], ax);
            aw = fma(al[j], Wl[j * ppc + le], aw);
        }
        x[ge[u]] = x[ge[u]] + ax;
        a.P[off[u]] = Pl[le] - aw;
    }
    // no CTA may exit while another can still read its shared memory (alpha, partials)
    cluster.sync();
    KS_T(5)
#ifdef KS_TIMING
    if (rank == 0 && threadIdx.x == 0)
        printf("KS ns: init %llu basis %llu gram %llu k4 %llu update %llu\n", tt[1] - tt[0], tt[2] - tt[1],
               tt[3] - tt[2], tt[4] - tt[3], tt[5] - tt[4]);
#endif
}

template <int S, int K>
cudaError_t ks_launch(bool pdl, const KSArgs &a, const K4Args &k4, DevState *st, size_t smem, cudaStream_t strm)
{
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(KS_CL);
    cfg.blockDim = dim3(KS_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = strm;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = KS_CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, k_small<S, K>, a, k4, st);
}

}  // namespace

bool ks_supported(const Geo &g, int s, int64_t npts)
{
    return (g.kind == 0 || g.kind == 1) && s >= 2 && s <= 8 && npts <= KS_MAXPTS;
}

bool ks_prepare()
{
    const int mx = 2 * 8 * ((KS_MAXPTS + KS_CL - 1) / KS_CL) * (int)sizeof(double);   // P and W, S <= 8
#define KS_ATTR(S, K) cudaFuncSetAttribute(k_small<S, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) == cudaSuccess
    return KS_ATTR(2, 0) && KS_ATTR(3, 0) && KS_ATTR(4, 0) && KS_ATTR(5, 0) && KS_ATTR(6, 0) && KS_ATTR(7, 0) &&
           KS_ATTR(8, 0) && KS_ATTR(2, 1) && KS_ATTR(3, 1) && KS_ATTR(4, 1) && KS_ATTR(5, 1) && KS_ATTR(6, 1) &&
           KS_ATTR(7, 1) && KS_ATTR(8, 1);
#undef KS_ATTR
}

void launch_ks(const Geo &g, const Slab &sl, int s, double theta, double sigma, double *const *xpp, double *blk,
               const K4Args &k4, DevState *st, cudaStream_t stream)
{
    (void)blk;
    KSArgs a;
    a.P = sl.P + g.plane;
    a.W = sl.W + g.plane;
    a.vstride = g.vstride;
    a.nx = g.nx;
    a.ny = g.ny;
    a.nzl = sl.nzl;
    a.pitch = g.pitch;
    a.plane = g.plane;
    a.center = g.center;
    a.dinv_c = g.dinv_c;
    a.theta = theta;
    a.sigma = sigma;
    a.xpp = xpp;
    const int64_t npts = (int64_t)g.nx * g.ny * sl.nzl;
    const size_t ring = (size_t)2 * s * ((npts + KS_CL - 1) / KS_CL) * sizeof(double);
#define KS_LAUNCH(S)                                                     \
    if (g.kind == 0) ks_launch<S, 0>(g.kn.pdl, a, k4, st, ring, stream); \
    else ks_launch<S, 1>(g.kn.pdl, a, k4, st, ring, stream);
    switch (s) {
    case 2: KS_LAUNCH(2) break;
    case 3: KS_LAUNCH(3) break;
    case 4: KS_LAUNCH(4) break;
    case 5: KS_LAUNCH(5) break;
    case 6: KS_LAUNCH(6) break;
    case 7: KS_LAUNCH(7) break;
    default: KS_LAUNCH(8) break;
    }
#undef KS_LAUNCH
}

}  // namespace sscg
