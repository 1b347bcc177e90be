// AMG coarse-grid Forward Gauss-Seidel (PAPER.md:225-246
// §6 "AMG Coarse-Grid Extension", §8; R25).
//
// One coarse level of unsmoothed aggregation: P piecewise constant on
// bx x by x bz blocks of fine cells, A_c = P^T A_f P.  For the 5-point,
// 7-point and variable-coefficient 7-point operators A_c couples only
// face-adjacent aggregates, so a coarse row has at most 7 entries.
//
//   streaming  (the paper's matrix-free variant): A_c is never stored; each
//              visit of row I recomputes its entries from A_f -- entry (I, J)
//              is the sum over the cells a of aggregate I of (A_f p_J)_a,
//              p_J = P e_J: a face sum of -k_face for a neighbour, the sum of
//              the cells' diagonals minus the couplings inside the aggregate
//              for the diagonal.
//   assembled  the same entries formed once at create (7 n_c doubles).
//
// Forward (lexicographic) Gauss-Seidel needs, for row c, the new values of
// its lower neighbours (z-1, y-1, x-1) and the previous sweep's values of its
// upper ones.  With the wavefront index t = I + J + K every lower neighbour
// lies on t - 1 and every upper one on t + 1, so all rows of a wavefront are
// independent, and sweep m can run wavefront t while sweep m-1 runs t + 2:
// step tau processes the wavefronts t = tau - 2m of every sweep m at once, a
// CTA barrier between steps -- T + 2(nu - 1) steps for nu sweeps instead of
// nu T.  Rows read only wavefronts t +- 1, which no other sweep writes in the
// same step, so the result is exactly the sequential sweep order.  r_c and y
// live in shared memory of one CTA (the coarsest level is small: n_c ~ 5000
// in the paper); arithmetic in the oracle's order without FMA contraction, so
// results are bitwise equal to it.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <vector>

#include "../../include/sscg.h"
#include "sscg_internal.cuh"

namespace sscg {
sscg_status api_fail(sscg_status st, const char *fmt, ...);
}
using sscg::api_fail;

namespace {

struct CG {
    int kind, nx, ny, nz, bx, by, bz, ncx, ncy, ncz;
    const double *kx, *ky, *kz;   // VARCOEF7 faces (layout of sscg.h), else null
};

constexpr int NT = 1024;   // FGS threads (one CTA); 512 for the variable-coefficient streaming mode
constexpr int nt_for(int mode) { return mode == 2 ? 512 : NT; }

// face coefficients around fine cell (i, j, k); 1 for the constant stencils
__device__ __forceinline__ double kxm(const CG &g, int i, int j, int k)
{
    return g.kx ? g.kx[((int64_t)k * g.ny + j) * (g.nx + 1) + i] : 1.0;
}
__device__ __forceinline__ double kxp(const CG &g, int i, int j, int k) { return kxm(g, i + 1, j, k); }
__device__ __forceinline__ double kym(const CG &g, int i, int j, int k)
{
    return g.ky ? g.ky[((int64_t)k * (g.ny + 1) + j) * g.nx + i] : 1.0;
}
__device__ __forceinline__ double kyp(const CG &g, int i, int j, int k) { return kym(g, i, j + 1, k); }
__device__ __forceinline__ double kzm(const CG &g, int i, int j, int k)
{
    return g.kz ? g.kz[((int64_t)k * g.ny + j) * g.nx + i] : 1.0;
}
__device__ __forceinline__ double kzp(const CG &g, int i, int j, int k) { return kzm(g, i, j, k + 1); }

// the fine diagonal: 4 / 6, or the six faces summed in the order z-, y-, x-, x+, y+, z+
__device__ __forceinline__ double fine_diag(const CG &g, int i, int j, int k)
{
    if (g.kind == SSCG_OP_STENCIL5_2D) return 4.0;
    if (g.kind == SSCG_OP_STENCIL7) return 6.0;
    double d = __dadd_rn(kzm(g, i, j, k), kym(g, i, j, k));
    d = __dadd_rn(d, kxm(g, i, j, k));
    d = __dadd_rn(d, kxp(g, i, j, k));
    d = __dadd_rn(d, kyp(g, i, j, k));
    return __dadd_rn(d, kzp(g, i, j, k));
}

// the entries of coarse row (I, J, K): e[0..6] for the neighbours z-1, y-1,
// x-1, itself, x+1, y+1, z+1 (0 where absent).  Each entry is the sum, over
// the aggregate's cells in ascending fine index, of (A_f p_nbr)_a formed as
// the fine operator's row is (diagonal first, then the couplings in the order
// z-, y-, x-, x+, y+, z+; terms of cells outside the neighbour vanish exactly)
__device__ void coarse_row(const CG &g, int I, int J, int K, double e[7])
{
    const int x0 = I * g.bx, x1 = min(x0 + g.bx, g.nx);
    const int y0 = J * g.by, y1 = min(y0 + g.by, g.ny);
    const int z0 = K * g.bz, z1 = min(z0 + g.bz, g.nz);
    double d = 0.0;
    for (int k = z0; k < z1; ++k)
        for (int j = y0; j < y1; ++j)
            for (int i = x0; i < x1; ++i) {
                double t = fine_diag(g, i, j, k);
                if (k - 1 >= z0) t = __dsub_rn(t, kzm(g, i, j, k));
                if (j - 1 >= y0) t = __dsub_rn(t, kym(g, i, j, k));
                if (i - 1 >= x0) t = __dsub_rn(t, kxm(g, i, j, k));
                if (i + 1 < x1) t = __dsub_rn(t, kxp(g, i, j, k));
                if (j + 1 < y1) t = __dsub_rn(t, kyp(g, i, j, k));
                if (k + 1 < z1) t = __dsub_rn(t, kzp(g, i, j, k));
                d = __dadd_rn(d, t);
            }
    e[3] = d;
    double a = 0.0;
    if (K > 0)
        for (int j = y0; j < y1; ++j)
            for (int i = x0; i < x1; ++i) a = __dsub_rn(a, kzm(g, i, j, z0));
    e[0] = a;
    a = 0.0;
    if (J > 0)
        for (int k = z0; k < z1; ++k)
            for (int i = x0; i < x1; ++i) a = __dsub_rn(a, kym(g, i, y0, k));
    e[1] = a;
    a = 0.0;
    if (I > 0)
        for (int k = z0; k < z1; ++k)
            for (int j = y0; j < y1; ++j) a = __dsub_rn(a, kxm(g, x0, j, k));
    e[2] = a;
    a = 0.0;
    if (I + 1 < g.ncx)
        for (int k = z0; k < z1; ++k)
            for (int j = y0; j < y1; ++j) a = __dsub_rn(a, kxp(g, x1 - 1, j, k));
    e[4] = a;
    a = 0.0;
    if (J + 1 < g.ncy)
        for (int k = z0; k < z1; ++k)
            for (int i = x0; i < x1; ++i) a = __dsub_rn(a, kyp(g, i, y1 - 1, k));
    e[5] = a;
    a = 0.0;
    if (K + 1 < g.ncz)
        for (int j = y0; j < y1; ++j)
            for (int i = x0; i < x1; ++i) a = __dsub_rn(a, kzp(g, i, j, z1 - 1));
    e[6] = a;
}

// coarse_row for a full 2 x 2 x 2 aggregate of the variable-coefficient
// operator, the streaming mode's common case: the 36 distinct faces it touches
// are loaded first (independent L2 loads, one round trip instead of a chain of
// ~96), then combined in exactly coarse_row's order -- the same doubles
__device__ void coarse_row_vc222(const CG &g, int I, int J, int K, double e[7])
{
    const int x0 = 2 * I, y0 = 2 * J, z0 = 2 * K;
    double fx[2][2][3], fy[2][3][2], fz[3][2][2];   // fx[k][j][i]: kx(x0+i, y0+j, z0+k), i = 0..2; etc.
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int i = 0; i < 3; ++i) fx[k][j][i] = __ldg(g.kx + ((int64_t)(z0 + k) * g.ny + y0 + j) * (g.nx + 1) + x0 + i);
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int i = 0; i < 2; ++i) fy[k][j][i] = __ldg(g.ky + ((int64_t)(z0 + k) * (g.ny + 1) + y0 + j) * g.nx + x0 + i);
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int i = 0; i < 2; ++i) fz[k][j][i] = __ldg(g.kz + ((int64_t)(z0 + k) * g.ny + y0 + j) * g.nx + x0 + i);
    double d = 0.0;
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                // fine_diag: z-, y-, x-, x+, y+, z+
                double t = __dadd_rn(fz[k][j][i], fy[k][j][i]);
                t = __dadd_rn(t, fx[k][j][i]);
                t = __dadd_rn(t, fx[k][j][i + 1]);
                t = __dadd_rn(t, fy[k][j + 1][i]);
                t = __dadd_rn(t, fz[k + 1][j][i]);
                // couplings inside the aggregate, same order
                if (k == 1) t = __dsub_rn(t, fz[k][j][i]);
                if (j == 1) t = __dsub_rn(t, fy[k][j][i]);
                if (i == 1) t = __dsub_rn(t, fx[k][j][i]);
                if (i == 0) t = __dsub_rn(t, fx[k][j][i + 1]);
                if (j == 0) t = __dsub_rn(t, fy[k][j + 1][i]);
                if (k == 0) t = __dsub_rn(t, fz[k + 1][j][i]);
                d = __dadd_rn(d, t);
            }
    e[3] = d;
    double a;
    a = 0.0;
    if (K > 0)
        for (int j = 0; j < 2; ++j)
            for (int i = 0; i < 2; ++i) a = __dsub_rn(a, fz[0][j][i]);
    e[0] = a;
    a = 0.0;
    if (J > 0)
        for (int k = 0; k < 2; ++k)
            for (int i = 0; i < 2; ++i) a = __dsub_rn(a, fy[k][0][i]);
    e[1] = a;
    a = 0.0;
    if (I > 0)
        for (int k = 0; k < 2; ++k)
            for (int j = 0; j < 2; ++j) a = __dsub_rn(a, fx[k][j][0]);
    e[2] = a;
    a = 0.0;
    if (I + 1 < g.ncx)
        for (int k = 0; k < 2; ++k)
            for (int j = 0; j < 2; ++j) a = __dsub_rn(a, fx[k][j][2]);
    e[4] = a;
    a = 0.0;
    if (J + 1 < g.ncy)
        for (int k = 0; k < 2; ++k)
            for (int i = 0; i < 2; ++i) a = __dsub_rn(a, fy[k][2][i]);
    e[5] = a;
    a = 0.0;
    if (K + 1 < g.ncz)
        for (int j = 0; j < 2; ++j)
            for (int i = 0; i < 2; ++i) a = __dsub_rn(a, fz[2][j][i]);
    e[6] = a;
}

__global__ void k_coarse_entries(CG g, double *out)
{
    const int nc = g.ncx * g.ncy * g.ncz;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
        const int I = c % g.ncx, J = (c / g.ncx) % g.ncy, K = c / (g.ncx * g.ncy);
        double e[7];
        coarse_row(g, I, J, K, e);
#pragma unroll
        for (int d = 0; d < 7; ++d) out[(int64_t)d * nc + c] = e[d];
    }
}

// r_c = P^T r_f: one coarse point per thread, its cells in ascending fine index
__global__ void k_coarse_restrict(CG g, const double *rf, double *rc)
{
    const int nc = g.ncx * g.ncy * g.ncz;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
        const int I = c % g.ncx, J = (c / g.ncx) % g.ncy, K = c / (g.ncx * g.ncy);
        const int x0 = I * g.bx, x1 = min(x0 + g.bx, g.nx);
        const int y0 = J * g.by, y1 = min(y0 + g.by, g.ny);
        const int z0 = K * g.bz, z1 = min(z0 + g.bz, g.nz);
        double a = 0.0;
        for (int k = z0; k < z1; ++k)
            for (int j = y0; j < y1; ++j)
                for (int i = x0; i < x1; ++i) a = __dadd_rn(a, rf[((int64_t)k * g.ny + j) * g.nx + i]);
        rc[c] = a;
    }
}

// x_f += P y: one fine cell per thread
__global__ void k_coarse_prolong(CG g, const double *y, double *xf)
{
    const int64_t nf = (int64_t)g.nx * g.ny * g.nz;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nf; q += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(q % g.nx), j = (int)((q / g.nx) % g.ny), k = (int)(q / ((int64_t)g.nx * g.ny));
        const int c = i / g.bx + g.ncx * (j / g.by + g.ncy * (k / g.bz));
        xf[q] = __dadd_rn(xf[q], y[c]);
    }
}

// nu pipelined Gauss-Seidel sweeps (see the file comment).
//
// The items of a step are the wavefronts t = tau - 2m of the active sweeps m,
// all of one parity; the host lists the coarse points parity-major (even t
// ascending, then odd t ascending), so a step's items are ONE contiguous list
// range [wlo[t_lo], whi[t_hi]), thread tid taking items tid, tid + NT, ...
// Per item a packed word meta = c | flags << 24 (flags: the neighbour exists
// at z-1, y-1, x-1, x+1, y+1, z+1) replaces the index arithmetic.  Entries:
//   MODE 0 (assembled): A7L[q * 8 + d] in list order, the next step's entries
//          loaded into registers before the barrier that ends this step, so
//          no L2 latency sits on the step's critical path;
//   MODE 1 (streaming, 5-/7-point): the entries in closed form from the
//          aggregate's extents -- face areas and 6 / 4 x cells - 2 x internal
//          couplings; every term is a small integer, so any summation order
//          gives the oracle's doubles exactly;
//   MODE 2 (streaming, variable coefficients): coarse_row from the faces at
//          every visit (the oracle's per-cell order).
// Within a step all reads (r, neighbour y) precede all writes of the thread's
// items, and no item of a step reads another's output (neighbours lie on
// t +- 1), so the result is the sequential sweep order, bitwise.
// MODE 0: items per thread whose entries are prefetched (3 spilled at the
// 64-register limit of 1024 threads: 0.31 ms per 20 sweeps at n_c = 4913 vs
// 0.21 with 2)
#ifndef COARSE_PF
#define COARSE_PF 2
#endif
constexpr int PF = COARSE_PF;

// Shared memory holds y and r_c in a row-padded layout, s(c) = I + px (J + ncy K)
// with px = ncx rounded up to even: the items of a wavefront, consecutive in
// ascending c, are (ncx - 1) apart in c -- with ncx = 17 every lane of a warp
// hit the same bank (a 32-way conflict on every y load) -- and px - 1 odd
// apart in s; meta carries s(c).
template <int MODE, int NT = nt_for(MODE)>
__global__ void __launch_bounds__(NT, 1)
    k_coarse_fgs(CG g, const double *__restrict__ A7L, const double *rc, double *y, int nu, const int *meta_g,
                 const int *wlo_g, const int *whi_g, int T, int exl, int eyl, int ezl, double center)
{
    extern __shared__ __align__(16) double sm[];
    const int nc = g.ncx * g.ncy * g.ncz, px = (g.ncx + 1) & ~1, ns = px * g.ncy * g.ncz, sxy = px * g.ncy;
    double *ys = sm, *rs = sm + ns;
    int *meta = reinterpret_cast<int *>(rs + ns), *wlo = meta + nc, *whi = wlo + T;
    const int tid = threadIdx.x;
    auto sidx = [&](int c) { const int I = c % g.ncx, r = c / g.ncx; return I + px * r; };
    for (int i = tid; i < nc; i += NT) {
        ys[sidx(i)] = y[i];
        rs[sidx(i)] = rc[i];
        meta[i] = meta_g[i];
    }
    for (int i = tid; i < T; i += NT) {
        wlo[i] = wlo_g[i];
        whi[i] = whi_g[i];
    }
    __syncthreads();
    const int steps = nu > 0 ? T + 2 * (nu - 1) : 0;
    auto range = [&](int tau, int &q0, int &q1) {
        const int a = tau - (T - 1);
        const int m_lo = a > 0 ? (a + 1) / 2 : 0, m_hi = min(nu - 1, tau / 2);
        if (tau >= steps || m_lo > m_hi) {
            q0 = q1 = 0;
            return;
        }
        q0 = wlo[tau - 2 * m_hi];
        q1 = whi[tau - 2 * m_lo];
    };
    auto entries = [&](int q, int m, double e[7]) {
        if (MODE == 0) {
            const double2 *p = reinterpret_cast<const double2 *>(A7L + (int64_t)q * 8);
            const double2 a0 = __ldg(p), a1 = __ldg(p + 1), a2 = __ldg(p + 2), a3 = __ldg(p + 3);
            e[0] = a0.x; e[1] = a0.y; e[2] = a1.x; e[3] = a1.y; e[4] = a2.x; e[5] = a2.y; e[6] = a3.x;
        } else if (MODE == 1) {
            const int f = m >> 24;
            const int ex = (f & 8) ? g.bx : exl, ey = (f & 16) ? g.by : eyl, ez = (f & 32) ? g.bz : ezl;
            const double axy = (double)(ex * ey), axz = (double)(ex * ez), ayz = (double)(ey * ez);
            e[0] = (f & 1) ? -axy : 0.0;
            e[1] = (f & 2) ? -axz : 0.0;
            e[2] = (f & 4) ? -ayz : 0.0;
            e[4] = (f & 8) ? -ayz : 0.0;
            e[5] = (f & 16) ? -axz : 0.0;
            e[6] = (f & 32) ? -axy : 0.0;
            e[3] = center * (double)(ex * ey * ez) -
                   2.0 * (double)((ex - 1) * ey * ez + ex * (ey - 1) * ez + ex * ey * (ez - 1));
        } else {
            const int sc = m & 0xFFFFFF;   // s(c) = I + px (J + ncy K)
            const int I = sc % px, J = (sc / px) % g.ncy, K = sc / sxy;
            if (g.bx == 2 && g.by == 2 && g.bz == 2 && 2 * I + 2 <= g.nx && 2 * J + 2 <= g.ny && 2 * K + 2 <= g.nz)
                coarse_row_vc222(g, I, J, K, e);   // a full aggregate: all faces loaded at once
            else
                coarse_row(g, I, J, K, e);
        }
    };
    // y_c = (r_c - sum_{j != c} a_cj y_j) / a_cc, j ascending (the oracle's order, no FMA)
    auto relax = [&](int m, const double e[7]) -> double {
        const int c = m & 0xFFFFFF, f = m >> 24;
        double s = rs[c];
        if (f & 1) s = __dsub_rn(s, __dmul_rn(e[0], ys[c - sxy]));
        if (f & 2) s = __dsub_rn(s, __dmul_rn(e[1], ys[c - px]));
        if (f & 4) s = __dsub_rn(s, __dmul_rn(e[2], ys[c - 1]));
        if (f & 8) s = __dsub_rn(s, __dmul_rn(e[4], ys[c + 1]));
        if (f & 16) s = __dsub_rn(s, __dmul_rn(e[5], ys[c + px]));
        if (f & 32) s = __dsub_rn(s, __dmul_rn(e[6], ys[c + sxy]));
        return __ddiv_rn(s, e[3]);
    };
    // MODE 0: pe[k] = the entries of this thread's k-th item of the current step;
    // as soon as item k is relaxed, pe[k] is refilled with the next step's k-th
    // item (the loads depend on nothing), so the rest of the step and the
    // barrier cover their L2 latency
    double pe[PF][7];
    int q0, q1, n0, n1;
    range(0, q0, q1);
    if (MODE == 0) {
#pragma unroll
        for (int k = 0; k < PF; ++k) {
            const int q = q0 + tid + k * NT;
            if (q < q1) entries(q, 0, pe[k]);
        }
    }
    for (int tau = 0; tau < steps; ++tau) {
        range(tau + 1, n0, n1);
        double v[PF];
        int mk[PF];
#pragma unroll
        for (int k = 0; k < PF; ++k) {   // reads of the first PF items
            const int q = q0 + tid + k * NT;
            mk[k] = (q < q1) ? meta[q] : -1;
            if (mk[k] >= 0) {
                double e[7];
                if (MODE == 0) {
#pragma unroll
                    for (int d = 0; d < 7; ++d) e[d] = pe[k][d];
                } else {
                    entries(q, mk[k], e);
                }
                v[k] = relax(mk[k], e);
            }
            if (MODE == 0 && n0 + tid + k * NT < n1) entries(n0 + tid + k * NT, 0, pe[k]);
        }
        // items beyond PF per thread (n_c above ~2 PF NT): read and written in turn
        // (no item of a step reads another's output, so the order is free)
        for (int q = q0 + tid + PF * NT; q < q1; q += NT) {
            double e[7];
            const int m = meta[q];
            entries(q, m, e);
            ys[m & 0xFFFFFF] = relax(m, e);
        }
#pragma unroll
        for (int k = 0; k < PF; ++k)
            if (mk[k] >= 0) ys[mk[k] & 0xFFFFFF] = v[k];
        q0 = n0;
        q1 = n1;
        __syncthreads();
    }
    for (int i = tid; i < nc; i += NT) y[i] = ys[sidx(i)];
}

// assembled entries in list order: A7L[q * 8 + d]
__global__ void k_coarse_entries_list(CG g, const int *meta, int nc, double *out)
{
    const int px = (g.ncx + 1) & ~1;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nc; q += gridDim.x * blockDim.x) {
        const int sc = meta[q] & 0xFFFFFF;
        const int I = sc % px, J = (sc / px) % g.ncy, K = sc / (px * g.ncy);
        double e[7];
        coarse_row(g, I, J, K, e);
#pragma unroll
        for (int d = 0; d < 7; ++d) out[(int64_t)q * 8 + d] = e[d];
        out[(int64_t)q * 8 + 7] = 0.0;
    }
}

size_t fgs_smem(int nc, int ns, int T) { return (size_t)ns * 16 + (size_t)nc * 4 + (size_t)2 * T * 4; }

}  // namespace

struct sscg_coarse {
    CG g{};
    int mode = 0, nc = 0, T = 0;
    int exl = 0, eyl = 0, ezl = 0;   // extents of the last aggregate of each axis
    double *A7L = nullptr;           // assembled: entries in list order, 8 doubles per point
    int *meta = nullptr, *wlo = nullptr, *whi = nullptr;   // the parity-major point list (k_coarse_fgs)
};

#define CCU(call)                                                                                   \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return api_fail(e_ == cudaErrorMemoryAllocation ? SSCG_ERR_OOM : SSCG_ERR_CUDA, "%s: %s", #call, \
                            cudaGetErrorString(e_));                                                \
    } while (0)

static unsigned grid_for(int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8); }

extern "C" void sscg_coarse_destroy(sscg_coarse *h)
{
    if (!h) return;
    cudaFree(h->A7L);
    cudaFree(h->meta);
    cudaFree(h->wlo);
    cudaFree(h->whi);
    delete h;
}

extern "C" sscg_status sscg_coarse_create(const sscg_operator *A, int32_t bx, int32_t by, int32_t bz, int32_t mode,
                                          sscg_coarse **out)
{
    if (!A || !out) return api_fail(SSCG_ERR_INVALID, "sscg_coarse_create: null argument");
    *out = nullptr;
    if (A->kind != SSCG_OP_STENCIL5_2D && A->kind != SSCG_OP_STENCIL7 && A->kind != SSCG_OP_VARCOEF7)
        return api_fail(SSCG_ERR_UNSUPPORTED, "sscg_coarse_create: operator kind %d (5-point, 7-point and "
                        "variable-coefficient 7-point only)", (int)A->kind);
    if (bx < 1 || by < 1 || bz < 1 || A->nx < 1 || A->ny < 1 || A->nz < 1)
        return api_fail(SSCG_ERR_INVALID, "sscg_coarse_create: bad grid or aggregate size");
    if (A->kind == SSCG_OP_STENCIL5_2D && (A->nz != 1 || bz != 1))
        return api_fail(SSCG_ERR_INVALID, "sscg_coarse_create: the 2D operator needs nz = bz = 1");
    if (A->kind == SSCG_OP_VARCOEF7 && (!A->kx || !A->ky || !A->kz))
        return api_fail(SSCG_ERR_INVALID, "sscg_coarse_create: face arrays missing");
    if (mode != SSCG_COARSE_STREAMING && mode != SSCG_COARSE_ASSEMBLED)
        return api_fail(SSCG_ERR_INVALID, "sscg_coarse_create: mode %d", (int)mode);
    if (A->nx > (1 << 20) || A->ny > (1 << 20) || A->nz > (1 << 20))
        return api_fail(SSCG_ERR_INVALID, "sscg_coarse_create: grid too large");
    CG g{};
    g.kind = A->kind;
    g.nx = (int)A->nx; g.ny = (int)A->ny; g.nz = (int)A->nz;
    g.bx = bx; g.by = by; g.bz = bz;
    g.ncx = (g.nx + bx - 1) / bx; g.ncy = (g.ny + by - 1) / by; g.ncz = (g.nz + bz - 1) / bz;
    if (A->kind == SSCG_OP_VARCOEF7) {
        g.kx = A->kx; g.ky = A->ky; g.kz = A->kz;
    }
    const int64_t nc = (int64_t)g.ncx * g.ncy * g.ncz;
    if (nc > SSCG_COARSE_MAX_N)
        return api_fail(SSCG_ERR_UNSUPPORTED, "sscg_coarse_create: n_c = %lld > %d (one CTA's shared memory)",
                        (long long)nc, SSCG_COARSE_MAX_N);
    auto *h = new sscg_coarse;
    h->g = g;
    h->mode = mode;
    h->nc = (int)nc;
    h->T = g.ncx + g.ncy + g.ncz - 2;   // wavefronts t = I + J + K in [0, T)
    h->exl = g.nx - (g.ncx - 1) * bx;
    h->eyl = g.ny - (g.ncy - 1) * by;
    h->ezl = g.nz - (g.ncz - 1) * bz;
    // the point list, parity-major: wavefronts t = 0, 2, 4, ... then 1, 3, ...,
    // each in ascending index; meta = c | neighbour flags << 24
    const int T = h->T;
    std::vector<int> cnt(T, 0), wlo(T), whi(T), meta(nc);
    for (int64_t c = 0; c < nc; ++c) {
        const int I = (int)(c % g.ncx), J = (int)((c / g.ncx) % g.ncy), K = (int)(c / ((int64_t)g.ncx * g.ncy));
        cnt[I + J + K] += 1;
    }
    int pos = 0;
    for (int p = 0; p < 2; ++p)
        for (int t = p; t < T; t += 2) {
            wlo[t] = pos;
            pos += cnt[t];
            whi[t] = pos;
        }
    std::vector<int> fill(wlo);
    for (int64_t c = 0; c < nc; ++c) {
        const int I = (int)(c % g.ncx), J = (int)((c / g.ncx) % g.ncy), K = (int)(c / ((int64_t)g.ncx * g.ncy));
        const int flags = (K > 0) | (J > 0) << 1 | (I > 0) << 2 | (I + 1 < g.ncx) << 3 | (J + 1 < g.ncy) << 4 |
                          (K + 1 < g.ncz) << 5;
        meta[fill[I + J + K]++] = (I + ((g.ncx + 1) & ~1) * (J + g.ncy * K)) | flags << 24;   // s(c), see k_coarse_fgs
    }
    auto bail = [&](sscg_status st) {
        sscg_coarse_destroy(h);
        return st;
    };
    cudaError_t e = cudaMalloc(&h->meta, nc * sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&h->wlo, T * sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&h->whi, T * sizeof(int));
    if (e == cudaSuccess) e = cudaMemcpy(h->meta, meta.data(), nc * sizeof(int), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->wlo, wlo.data(), T * sizeof(int), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->whi, whi.data(), T * sizeof(int), cudaMemcpyHostToDevice);
    const int smem = (int)fgs_smem(h->nc, ((h->g.ncx + 1) & ~1) * h->g.ncy * h->g.ncz, h->T);
    if (smem > 226 * 1024)
        return bail(api_fail(SSCG_ERR_UNSUPPORTED, "sscg_coarse_create: %d B of shared memory for n_c = %lld "
                             "(row-padded y and r)", smem, (long long)nc));
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_coarse_fgs<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_coarse_fgs<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_coarse_fgs<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess && mode == SSCG_COARSE_ASSEMBLED) {
        e = cudaMalloc(&h->A7L, 8 * nc * sizeof(double));
        if (e == cudaSuccess) {
            k_coarse_entries_list<<<grid_for(nc), 256>>>(g, h->meta, (int)nc, h->A7L);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
    }
    if (e != cudaSuccess)
        return bail(api_fail(e == cudaErrorMemoryAllocation ? SSCG_ERR_OOM : SSCG_ERR_CUDA, "sscg_coarse_create: %s",
                             cudaGetErrorString(e)));
    *out = h;
    return SSCG_OK;
}

extern "C" sscg_status sscg_coarse_restrict(sscg_coarse *h, const double *rf, double *rc, void *stream)
{
    if (!h || !rf || !rc) return api_fail(SSCG_ERR_INVALID, "sscg_coarse_restrict: null argument");
    k_coarse_restrict<<<grid_for(h->nc), 256, 0, (cudaStream_t)stream>>>(h->g, rf, rc);
    CCU(cudaGetLastError());
    return SSCG_OK;
}

extern "C" sscg_status sscg_coarse_prolong_add(sscg_coarse *h, const double *y, double *xf, void *stream)
{
    if (!h || !y || !xf) return api_fail(SSCG_ERR_INVALID, "sscg_coarse_prolong_add: null argument");
    const int64_t nf = (int64_t)h->g.nx * h->g.ny * h->g.nz;
    k_coarse_prolong<<<grid_for(nf), 256, 0, (cudaStream_t)stream>>>(h->g, y, xf);
    CCU(cudaGetLastError());
    return SSCG_OK;
}

extern "C" sscg_status sscg_coarse_fgs(sscg_coarse *h, const double *rc, double *y, int32_t nu, void *stream)
{
    if (!h || !rc || !y) return api_fail(SSCG_ERR_INVALID, "sscg_coarse_fgs: null argument");
    if (nu < 0) return api_fail(SSCG_ERR_INVALID, "sscg_coarse_fgs: nu = %d", (int)nu);
    if (nu == 0) return SSCG_OK;
    const size_t smem = fgs_smem(h->nc, ((h->g.ncx + 1) & ~1) * h->g.ncy * h->g.ncz, h->T);
    const double center = h->g.kind == SSCG_OP_STENCIL5_2D ? 4.0 : 6.0;
    cudaStream_t st = (cudaStream_t)stream;
    if (h->mode == SSCG_COARSE_ASSEMBLED)
        k_coarse_fgs<0><<<1, NT, smem, st>>>(h->g, h->A7L, rc, y, nu, h->meta, h->wlo, h->whi, h->T, h->exl, h->eyl,
                                             h->ezl, center);
    else if (h->g.kind != SSCG_OP_VARCOEF7)   // streaming, constant stencils: closed-form entries
        k_coarse_fgs<1><<<1, NT, smem, st>>>(h->g, nullptr, rc, y, nu, h->meta, h->wlo, h->whi, h->T, h->exl, h->eyl,
                                             h->ezl, center);
    else
        k_coarse_fgs<2><<<1, nt_for(2), smem, st>>>(h->g, nullptr, rc, y, nu, h->meta, h->wlo, h->whi, h->T, h->exl, h->eyl,
                                             h->ezl, center);
    CCU(cudaGetLastError());
    return SSCG_OK;
}

extern "C" sscg_status sscg_coarse_entries(sscg_coarse *h, double *out, void *stream)
{
    if (!h || !out) return api_fail(SSCG_ERR_INVALID, "sscg_coarse_entries: null argument");
    k_coarse_entries<<<grid_for(h->nc), 256, 0, (cudaStream_t)stream>>>(h->g, out);   // (the routine the assembly ran)
    CCU(cudaGetLastError());
    return SSCG_OK;
}

extern "C" sscg_status sscg_coarse_query(const sscg_coarse *h, int32_t what, int64_t *out)
{
    if (!h || !out) return api_fail(SSCG_ERR_INVALID, "sscg_coarse_query: null argument");
    switch (what) {
    case SSCG_COARSE_QUERY_N: *out = h->nc; break;
    case SSCG_COARSE_QUERY_NCX: *out = h->g.ncx; break;
    case SSCG_COARSE_QUERY_NCY: *out = h->g.ncy; break;
    case SSCG_COARSE_QUERY_NCZ: *out = h->g.ncz; break;
    case SSCG_COARSE_QUERY_WAVEFRONTS: *out = h->T; break;
    case SSCG_COARSE_QUERY_MATRIX_BYTES: *out = h->A7L ? 8 * (int64_t)h->nc * 8 : 0; break;
    default: return api_fail(SSCG_ERR_INVALID, "sscg_coarse_query: unknown key %d", (int)what);
    }
    return SSCG_OK;
}
