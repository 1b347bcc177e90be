// K4 -- Ruhe scaling + nu Forward Gauss-Seidel sweeps on the s x s Gram
//       system, stopping test and history (single warp).
// K5 -- fused solution/residual update x += P alpha, r -= (AP) alpha
//       (r is stored in place of p_0).
#include <cstdio>

#include "sscg_internal.cuh"
#include "k4_small.cuh"

namespace sscg {
namespace {

constexpr int SMAX = 64;

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// s > 32 (up to 64): one warp, lane l owns rows l and l + 32; the scaled G
// lives in shared memory (column-major), coordinate by coordinate in residual
// form (see k4_small.cuh for the method and the s <= 32 kernel).
__global__ void __launch_bounds__(32) k4_fgs_big(K4Args a, DevState *st)
{
    PDL_ENTRY(st);
    __shared__ double Gc[SMAX * SMAX];   // column-major: Gc[j*s + i] = G_ij
    __shared__ double dsh[SMAX];
    const int s = a.s, lane = threadIdx.x;
    const int k = st->k;
    const int nent = s * s + s;
    const bool rec = k < st->hist_cap, recg = k < st->gram_cap;
    if (recg)
        for (int q = lane; q < nent; q += 32) a.h_gram[(int64_t)k * nent + q] = a.blk[q];
    const double *Gh = a.blk, *c = Gh + s * s;

    const double rn = sqrt(a.rn2 ? *a.rn2 : c[0]);
    const double r0 = (k == 0) ? rn : st->r0norm;
    if (lane == 0) {
        if (k == 0) st->r0norm = rn;
        if (rec) a.h_relres[k] = (r0 > 0.0) ? rn / r0 : 0.0;
    }
    if (!isfinite(rn)) {
        if (lane == 0) { st->nonfinite = 1; st->done = 1; st->outer = k; }
        return;
    }
    if (rn <= st->rtol * r0) {
        if (lane == 0) { st->converged = 1; st->done = 1; st->outer = k; }
        return;
    }
    if (k >= st->max_outer) {
        if (lane == 0) { st->done = 1; st->outer = k; }
        return;
    }
    // Ruhe scaling
    const int i0 = lane, i1 = lane + 32;
    const bool v0 = i0 < s, v1 = i1 < s;
    double d0 = 0.0, d1 = 0.0;
    bool ok = true;
    if (v0) { const double gd = Gh[i0 * s + i0]; ok &= (gd > 0.0) && isfinite(gd); d0 = 1.0 / sqrt(gd); }
    if (v1) { const double gd = Gh[i1 * s + i1]; ok &= (gd > 0.0) && isfinite(gd); d1 = 1.0 / sqrt(gd); }
    if (!__all_sync(0xffffffffu, ok)) {
        if (lane == 0) { st->breakdown = 1; st->done = 1; st->outer = k; }
        return;
    }
    if (v0) dsh[i0] = d0;
    if (v1) dsh[i1] = d1;
    __syncwarp();
    const double ct0 = v0 ? d0 * c[i0] : 0.0;
    const double ct1 = v1 ? d1 * c[i1] : 0.0;
    double rho0 = ct0, rho1 = ct1, al0 = 0.0, al1 = 0.0;
    for (int q = lane; q < s * s; q += 32) {
        const int i = q / s, j = q - i * s;
        Gc[j * s + i] = (i == j) ? 1.0 : (dsh[i] * Gh[q]) * dsh[j];
    }
    __syncwarp();
    for (int sw = 0; sw < a.nu; ++sw) {
        for (int j = 0; j < s; ++j) {
            const bool hi = j >= 32;
            const int owner = j & 31;
            const double dj = __shfl_sync(0xffffffffu, hi ? rho1 : rho0, owner);
            const double g0 = v0 ? Gc[j * s + i0] : 0.0;
            const double g1 = v1 ? Gc[j * s + i1] : 0.0;
            rho0 = fma(-g0, dj, rho0);
            rho1 = fma(-g1, dj, rho1);
            al0 += (!hi && lane == owner) ? dj : 0.0;
            al1 += (hi && lane == owner) ? dj : 0.0;
        }
    }
    double res0 = ct0, res1 = ct1;
    for (int j = 0; j < s; ++j) {
        const double aj = __shfl_sync(0xffffffffu, (j < 32) ? al0 : al1, j & 31);
        if (v0) res0 = fma(-Gc[j * s + i0], aj, res0);
        if (v1) res1 = fma(-Gc[j * s + i1], aj, res1);
    }
    // ||L||_F^2 = sum_{i > j} G_ij^2 (the quantity FGS convergence depends on)
    double ll = 0.0;
    for (int j = 0; j < s; ++j) {
        if (v0 && j < i0) { const double gij = Gc[j * s + i0]; ll = fma(gij, gij, ll); }
        if (v1 && j < i1) { const double gij = Gc[j * s + i1]; ll = fma(gij, gij, ll); }
    }
    ll = warp_sum(ll);
    // delta = ||c~ - G a~|| / ||c~||  (PAPER.md:259-262 inexactness monitor)
    const double rr = warp_sum(res0 * res0 + res1 * res1);
    const double cc = warp_sum(ct0 * ct0 + ct1 * ct1);
    if (v0) a.alpha[i0] = d0 * al0;
    if (v1) a.alpha[i1] = d1 * al1;
    if (recg) {
        if (v0) { a.h_d[(int64_t)k * s + i0] = d0; a.h_at[(int64_t)k * s + i0] = al0; a.h_al[(int64_t)k * s + i0] = d0 * al0; }
        if (v1) { a.h_d[(int64_t)k * s + i1] = d1; a.h_at[(int64_t)k * s + i1] = al1; a.h_al[(int64_t)k * s + i1] = d1 * al1; }
    }
    if (rec && lane == 0) {
        a.h_delta[k] = sqrt(rr) / sqrt(cc);
        a.h_lnorm[k] = sqrt(ll);
    }
    if (lane == 0) {
        st->outer = k + 1;
        st->k = k + 1;
    }
}

// K4C -- the exact Gram solve the paper's FGS replaces:
// the same stopping test and Ruhe scaling as K4, then a dense Cholesky
// factorisation G = R^T R of the scaled Gram matrix (left-looking, row k of R
// by the lanes in parallel) and two triangular solves, all in shared memory
// (s <= 64) by one warp.  O(s^3) work -- SURVEY §8(f) NEXT-2, selected with
// SSCG_OPT_GRAM_SOLVER = SSCG_GRAM_CHOLESKY.  A non-positive pivot is a Gram
// breakdown (R19).
__global__ void __launch_bounds__(32) k4_chol(K4Args a, DevState *st)
{
    PDL_ENTRY(st);
    // R overwrites the upper triangle of G in place (row k of R is written
    // after row k of G was last read)
    __shared__ double R[SMAX * SMAX], dsh[SMAX], ct[SMAX], y[SMAX], al[SMAX];
    const int s = a.s, lane = threadIdx.x;
    const int k = st->k;
    const double *Gh = a.blk, *c = a.blk + s * s;
    const int nent = s * s + s;
    const bool rec = k < st->hist_cap, recg = k < st->gram_cap;
    if (recg)
        for (int q = lane; q < nent; q += 32) a.h_gram[(int64_t)k * nent + q] = a.blk[q];
    const double rn = sqrt(a.rn2 ? *a.rn2 : c[0]);
    const double r0 = (k == 0) ? rn : st->r0norm;
    if (lane == 0) {
        if (k == 0) st->r0norm = rn;
        if (rec) a.h_relres[k] = (r0 > 0.0) ? rn / r0 : 0.0;
    }
    if (!isfinite(rn)) {
        if (lane == 0) { st->nonfinite = 1; st->done = 1; st->outer = k; }
        return;
    }
    if (rn <= st->rtol * r0) {
        if (lane == 0) { st->converged = 1; st->done = 1; st->outer = k; }
        return;
    }
    if (k >= st->max_outer) {
        if (lane == 0) { st->done = 1; st->outer = k; }
        return;
    }
    bool ok = true;
    for (int i = lane; i < s; i += 32) {
        const double gd = Gh[i * s + i];
        ok &= (gd > 0.0) && isfinite(gd);
        dsh[i] = 1.0 / sqrt(gd);
    }
    if (!__all_sync(0xffffffffu, ok)) {
        if (lane == 0) { st->breakdown = 1; st->done = 1; st->outer = k; }
        return;
    }
    __syncwarp();
    for (int q = lane; q < s * s; q += 32) {
        const int i = q / s, j = q - i * s;
        R[q] = (i == j) ? 1.0 : (dsh[i] * Gh[q]) * dsh[j];
    }
    for (int i = lane; i < s; i += 32) ct[i] = dsh[i] * c[i];
    __syncwarp();
    // R_kk = sqrt(G_kk - sum_{m<k} R_mk^2);  R_kj = (G_kj - sum_{m<k} R_mk R_mj) / R_kk
    for (int kk = 0; kk < s; ++kk) {
        double piv = R[kk * s + kk];
        for (int m = 0; m < kk; ++m) piv -= R[m * s + kk] * R[m * s + kk];
        if (!(piv > 0.0)) {
            if (lane == 0) { st->breakdown = 1; st->done = 1; st->outer = k; }
            return;
        }
        const double rkk = sqrt(piv);
        for (int j = kk + 1 + lane; j < s; j += 32) {
            double b = R[kk * s + j];
            for (int m = 0; m < kk; ++m) b -= R[m * s + kk] * R[m * s + j];
            R[kk * s + j] = b / rkk;
        }
        if (lane == 0) R[kk * s + kk] = rkk;
        __syncwarp();
    }
    // R^T y = c~ (forward), R a~ = y (backward): one lane, s^2/2 FMAs each
    if (lane == 0) {
        for (int i = 0; i < s; ++i) {
            double t = ct[i];
            for (int m = 0; m < i; ++m) t -= R[m * s + i] * y[m];
            y[i] = t / R[i * s + i];
        }
        for (int i = s - 1; i >= 0; --i) {
            double t = y[i];
            for (int m = i + 1; m < s; ++m) t -= R[i * s + m] * al[m];
            al[i] = t / R[i * s + i];
        }
    }
    __syncwarp();
    double rr = 0.0, cc = 0.0;
    for (int i = lane; i < s; i += 32) {
        double ri = ct[i];
        for (int j = 0; j < s; ++j) ri -= ((i == j) ? 1.0 : (dsh[i] * Gh[i * s + j]) * dsh[j]) * al[j];
        rr += ri * ri;
        cc += ct[i] * ct[i];
        a.alpha[i] = dsh[i] * al[i];
        if (recg) {
            a.h_d[(int64_t)k * s + i] = dsh[i];
            a.h_at[(int64_t)k * s + i] = al[i];
            a.h_al[(int64_t)k * s + i] = dsh[i] * al[i];
        }
    }
    double ll = 0.0;
    for (int i = lane; i < s; i += 32)
        for (int j = 0; j < i; ++j) {
            const double gij = (dsh[i] * Gh[i * s + j]) * dsh[j];
            ll = fma(gij, gij, ll);
        }
    rr = warp_sum(rr);
    cc = warp_sum(cc);
    ll = warp_sum(ll);
    if (lane == 0) {
        if (rec) {
            a.h_delta[k] = sqrt(rr) / sqrt(cc);
            a.h_lnorm[k] = sqrt(ll);
        }
        st->outer = k + 1;
        st->k = k + 1;
    }
}

// Diagnostics (SSCG_OPT_DIAGNOSTICS): kappa(G) of the
// Ruhe-scaled Gram matrix of the outer iteration K4 just completed
// ("kappa(G) = O(s^2) ... conditioning"), from its eigenvalues
// by cyclic Jacobi rotations on one warp (each rotation's row/column update
// spread over the lanes).  Off the hot path: launched only when enabled.
__global__ void __launch_bounds__(32) k_kappa(const double *blk, int s, const DevState *st, double *h_kappa)
{
    PDL_ENTRY(st);
    const int k = st->k - 1;
    if (k < 0 || k >= st->hist_cap) return;
    __shared__ double A[SMAX * SMAX], d[SMAX];
    const int lane = threadIdx.x;
    for (int i = lane; i < s; i += 32) d[i] = 1.0 / sqrt(blk[i * s + i]);
    __syncwarp();
    for (int q = lane; q < s * s; q += 32) {
        const int i = q / s, j = q - i * s;
        A[q] = (i == j) ? 1.0 : (d[i] * blk[q]) * d[j];
    }
    __syncwarp();
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0, dia = 0.0;
        for (int q = lane; q < s * s; q += 32) {
            const int i = q / s, j = q - i * s;
            if (i < j) off += A[q] * A[q];
            else if (i == j) dia += A[q] * A[q];
        }
        for (int o = 16; o > 0; o >>= 1) {
            off += __shfl_xor_sync(0xffffffffu, off, o);
            dia += __shfl_xor_sync(0xffffffffu, dia, o);
        }
        if (off <= 1e-32 * dia) break;
        for (int p = 0; p < s - 1; ++p)
            for (int q = p + 1; q < s; ++q) {
                const double apq = A[p * s + q];
                if (apq == 0.0) continue;
                const double app = A[p * s + p], aqq = A[q * s + q];
                const double th = (aqq - app) / (2.0 * apq);
                const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
                __syncwarp();
                for (int r = lane; r < s; r += 32) {
                    if (r == p || r == q) continue;
                    const double arp = A[r * s + p], arq = A[r * s + q];
                    const double np = c * arp - sn * arq, nq = sn * arp + c * arq;
                    A[r * s + p] = np; A[p * s + r] = np;
                    A[r * s + q] = nq; A[q * s + r] = nq;
                }
                __syncwarp();
                if (lane == 0) {
                    A[p * s + p] = app - t * apq;
                    A[q * s + q] = aqq + t * apq;
                    A[p * s + q] = 0.0;
                    A[q * s + p] = 0.0;
                }
                __syncwarp();
            }
    }
    double lo = 1e300, hi = -1e300;
    for (int i = lane; i < s; i += 32) {
        lo = fmin(lo, A[i * s + i]);
        hi = fmax(hi, A[i * s + i]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) h_kappa[k] = (lo > 0.0) ? hi / lo : INFINITY;
}

struct K5Params {
    const double *P;   // interior start of p_0 (= r_k)
    const double *W;   // interior start of w_0
    int64_t vstride;
    int64_t N;         // interior doubles (nzl * plane)
    int s;
    const double *alpha;
    int rec;              // 1: r -= W alpha formed from the basis recurrence (k5 REC)
    double theta, sigma, dm;   // Chebyshev parameters and the constant Jacobi diagonal M
    const double *dvec;        // or the diagonal M per point (padded layout, interior start), else null
    double *const *xpp;   // device cell holding the caller's x (process layout):
    int64_t xoff;         //   this launch updates (*xpp)[xoff ...]; read per launch so one
                          //   captured graph serves every x (sscg_solve / sscg_iterate)
    int nx, pitch;
    // w_{s-1} folded (DESIGN.md §6 "w_{s-1} fold"): not stored by the basis
    // kernels; formed here as A p_{s-1} (7-point, constant centre) from
    // p_{s-1} and its six neighbours (ghost planes current)
    int ny;
    int64_t plane;
    double inv_nx, inv_ny, center;
};

// flat path: pitch == nx and x 16-B aligned; 2 points per thread per step.
// S > 0: the basis size is a compile-time constant, so all 2S loads of a
// point are issued before the first FMA (S = 0: runtime s).
// REC: the Chebyshev recurrence gives, for a constant
// Jacobi diagonal M = m I,
//   w_0 = m (p_1/theta + sigma p_0),  w_j = m ((p_{j+1} + p_{j-1})/(2 theta) + sigma p_j)  (1 <= j <= s-2)
// so  W alpha = m sum_k gamma_k p_k + alpha_{s-1} w_{s-1}  with gamma from alpha
// (R21).  The update then streams P, w_{s-1} and x (s+2 vectors in,
// 2 out) instead of P, W and x (2s+1 in): the per-point rounding is of the
// same order as forming W alpha from the stored W (whose SpMV entries carry
// the same m |p| cancellation), unlike the Gram dots, which keep W.
//
// FOLD (REC only): w_{s-1} = A p_{s-1} is not read but formed per point pair
// from p_{s-1} (x+-1 from the neighbouring pairs, y+-1 and z+-1 from the rows /
// planes around it, zero outside the grid in x and y; the ghost planes carry
// the z neighbours), in the order of the single step it replaces: centre
// term minus (z-1, y-1, x-1, x+1, y+1, z+1).  p_{s-1} is then loaded with
// the default cache policy, since the neighbouring points re-read it from L2.
template <int S, bool REC, bool FOLD>
__global__ void __launch_bounds__(256) k5_update_vec(K5Params k, const DevState *st)
{
    PDL_ENTRY(st);
    __shared__ double al[SMAX], ga[SMAX];
    for (int j = threadIdx.x; j < k.s; j += blockDim.x) al[j] = k.alpha[j];
    __syncthreads();
    if (REC) {
        for (int j = threadIdx.x; j < k.s; j += blockDim.x) {
            const int s1 = k.s - 1;
            double g = (j < s1) ? k.sigma * al[j] : 0.0;
            if (j == 1) g += al[0] / k.theta;
            if (j - 1 >= 1 && j - 1 <= s1 - 1) g += al[j - 1] / (2.0 * k.theta);
            if (j + 1 >= 1 && j + 1 <= s1 - 1) g += al[j + 1] / (2.0 * k.theta);
            ga[j] = k.dvec ? g : k.dm * g;
        }
        __syncthreads();
    }
    const int s = S > 0 ? S : k.s;
    const int64_t n2 = k.N >> 1;
    const double2 *P2 = reinterpret_cast<const double2 *>(k.P);
    const double2 *W2 = reinterpret_cast<const double2 *>(k.W);
    double *xs = *k.xpp + k.xoff;
    const bool xal = (reinterpret_cast<uintptr_t>(xs) & 15) == 0;   // else two 8-B accesses
    double2 *x2 = reinterpret_cast<double2 *>(xs);
    double2 *r2 = reinterpret_cast<double2 *>(const_cast<double *>(k.P));
    const int64_t vs2 = k.vstride >> 1;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += (int64_t)gridDim.x * blockDim.x) {
        double2 ax = make_double2(0.0, 0.0), aw = make_double2(0.0, 0.0);
        const double2 p0 = __ldcs(P2 + e);
        if (REC) {
#pragma unroll
            for (int j = 0; j < s; ++j) {
                const double2 pj = (j == 0) ? p0 : (FOLD && j == s - 1) ? __ldg(P2 + j * vs2 + e) : __ldcs(P2 + j * vs2 + e);
                ax.x = fma(al[j], pj.x, ax.x); ax.y = fma(al[j], pj.y, ax.y);
                aw.x = fma(ga[j], pj.x, aw.x); aw.y = fma(ga[j], pj.y, aw.y);
            }
            if (k.dvec) {   // variable diagonal: M sum gamma_k p_k pointwise
                const double2 m = __ldcs(reinterpret_cast<const double2 *>(k.dvec) + e);
                aw.x *= m.x;
                aw.y *= m.y;
            }
            double2 wl;
            if (FOLD) {
                const double2 *q2 = P2 + (s - 1) * vs2;
                const double *q = reinterpret_cast<const double *>(q2);
                const double2 c = __ldg(q2 + e);
                // all neighbour loads are in bounds (the ghost planes bracket the
                // launch range), issued before the coordinates mask them
                const int64_t py = k.pitch >> 1, pz = k.plane >> 1;
                double l = __ldg(q + 2 * e - 1), rr = __ldg(q + 2 * e + 2);
                double2 ylo = __ldg(q2 + e - py), yhi = __ldg(q2 + e + py);
                const double2 dn = __ldg(q2 + e - pz), up = __ldg(q2 + e + pz);
                // grid coordinates of the pair's first point (rows of the
                // launch range start on a plane boundary; exact in FP64)
                const double fe = (double)(2 * e);
                const double row = floor((fe + 0.5) * k.inv_nx);
                const int x = (int)(fe - row * (double)k.nx);
                const int y = (int)(row - floor((row + 0.5) * k.inv_ny) * (double)k.ny);
                if (x == 0) l = 0.0;
                if (x + 2 >= k.nx) rr = 0.0;
                if (y == 0) ylo = make_double2(0.0, 0.0);
                if (y + 1 >= k.ny) yhi = make_double2(0.0, 0.0);
                wl.x = k.center * c.x - (dn.x + ylo.x + l + c.y + yhi.x + up.x);
                wl.y = k.center * c.y - (dn.y + ylo.y + c.x + rr + yhi.y + up.y);
            } else {
                wl = __ldcs(W2 + (s - 1) * vs2 + e);
            }
            aw.x = fma(al[s - 1], wl.x, aw.x); aw.y = fma(al[s - 1], wl.y, aw.y);
        } else {
#pragma unroll
            for (int j = 0; j < s; ++j) {
                const double2 pj = (j == 0) ? p0 : __ldcs(P2 + j * vs2 + e);
                const double2 wj = __ldcs(W2 + j * vs2 + e);
                ax.x = fma(al[j], pj.x, ax.x); ax.y = fma(al[j], pj.y, ax.y);
                aw.x = fma(al[j], wj.x, aw.x); aw.y = fma(al[j], wj.y, aw.y);
            }
        }
        if (xal) {
            double2 xv = __ldcs(x2 + e);
            xv.x += ax.x; xv.y += ax.y;
            __stcs(x2 + e, xv);
        } else {
            xs[2 * e] += ax.x;
            xs[2 * e + 1] += ax.y;
        }
        __stcs(r2 + e, make_double2(p0.x - aw.x, p0.y - aw.y));
    }
}

// generic path (odd nx / unaligned x): scalar, skips the pad column.
__global__ void __launch_bounds__(256) k5_update_gen(K5Params k, const DevState *st)
{
    PDL_ENTRY(st);
    __shared__ double al[SMAX];
    for (int j = threadIdx.x; j < k.s; j += blockDim.x) al[j] = k.alpha[j];
    __syncthreads();
    double *r = const_cast<double *>(k.P);
    double *xs = *k.xpp + k.xoff;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < k.N; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e / k.pitch;
        const int xx = (int)(e - row * k.pitch);
        if (xx >= k.nx) continue;
        double ax = 0.0, aw = 0.0;
        const double p0 = k.P[e];
        for (int j = 0; j < k.s; ++j) {
            const double pj = (j == 0) ? p0 : k.P[j * k.vstride + e];
            ax = fma(al[j], pj, ax);
            aw = fma(al[j], k.W[j * k.vstride + e], aw);
        }
        const int64_t xi = row * k.nx + xx;
        xs[xi] += ax;
        r[e] = p0 - aw;
    }
}

}  // namespace

// s <= 32: the one-warp FGS of k4_small.cuh (the same body the Gram pass runs
// when it is fused there)
__global__ void __launch_bounds__(32) k4_fgs_warp(K4Args a, DevState *st)
{
    PDL_ENTRY(st);
    __shared__ double scratch[32 * 32 + 32 + 32];
#ifdef K4_TIMING   // variant builds only: the kernel's own duration at the clocks of the real schedule
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#endif
    k4_fgs_dispatch(a, st, scratch);
#ifdef K4_TIMING
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) printf("K4 ns %llu (s %d nu %d)\n", t1 - t0, a.s, a.nu);
#endif
}

void launch_k4(const K4Args &a, DevState *st, cudaStream_t s)
{
    if (a.solver == 1) launch_pdl(a.pdl, k4_chol, dim3(1), dim3(32), 0, s, a, st);
    else if (a.s <= 32) launch_pdl(a.pdl, k4_fgs_warp, dim3(1), dim3(32), 0, s, a, st);
    else launch_pdl(a.pdl, k4_fgs_big, dim3(1), dim3(32), 0, s, a, st);
}

// Diagnostics: ||P_k||_F^2 of the basis of this outer iteration (before K5
// overwrites p_0) as per-block partials, their fixed-order sum, and the
// inexactness budget term delta_k ||A|| ||P_k||_F of PAPER.md:259-266
// (Thm "Inexact Convergence"; ||P_k|| taken as the Frobenius norm, SPEC.md:353,
// ||A|| as the Gershgorin bound max_i sum_j |A_ij|).
__global__ void __launch_bounds__(256) k_pnorm(const double *P, int64_t vstride, int64_t N, int s, double *part,
                                               const DevState *st)
{
    PDL_ENTRY(st);
    __shared__ double red[8];
    double acc = 0.0;
    for (int j = 0; j < s; ++j)
        for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x) {
            const double v = P[j * vstride + e];
            acc = fma(v, v, acc);
        }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[w];
        part[blockIdx.x] = v;
    }
}

__global__ void k_psum(const double *part, int n, double *sum, const DevState *st)
{
    PDL_ENTRY(st);
    double v = 0.0;
    for (int b = threadIdx.x; b < n; b += 32) v += part[b];
    v = warp_sum(v);
    if (threadIdx.x == 0) *sum = v;
}

__global__ void k_budget(const double *sum, double anorm, const DevState *st, const double *h_delta, double *h_pnorm,
                         double *h_budget)
{
    PDL_ENTRY(st);
    const int k = st->k - 1;
    if (k < 0 || k >= st->hist_cap) return;
    const double pf = sqrt(*sum);
    h_pnorm[k] = pf;
    h_budget[k] = h_delta[k] * anorm * pf;
}

// Gershgorin bound of ||A||_2: max over rows of sum_j |A_ij| (per-block maxima)
__global__ void __launch_bounds__(256) k_anorm(Geo g, const double *kx, const double *ky, const double *kz, int nzl,
                                               double *bmax)
{
    __shared__ double red[8];
    double mx = 0.0;
    if (g.kind == 4) {
        for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < g.n; r += (int64_t)gridDim.x * blockDim.x) {
            double a = 0.0;
            for (int64_t q = g.rowptr[r]; q < g.rowptr[r + 1]; ++q) a += fabs(g.val[q]);
            mx = fmax(mx, a);
        }
    } else if (g.kind == 3) {
        const int64_t nxy = (int64_t)g.nx * g.ny, tot = nxy * nzl;
        for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
            const int64_t zl = e / nxy, rem = e - zl * nxy, y = rem / g.nx, x = rem - y * g.nx;
            const double d = kx[(zl * g.ny + y) * (g.nx + 1) + x] + kx[(zl * g.ny + y) * (g.nx + 1) + x + 1] +
                             ky[(zl * (g.ny + 1) + y) * g.nx + x] + ky[(zl * (g.ny + 1) + y + 1) * g.nx + x] +
                             kz[(zl * g.ny + y) * g.nx + x] + kz[((zl + 1) * g.ny + y) * g.nx + x];
            mx = fmax(mx, 2.0 * d);   // A_ii + sum of the (positive) off-diagonal faces
        }
    } else {
        mx = 2.0 * g.center;          // graph-Laplacian stencils: centre + |off-diagonals|
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, red[w]);
        bmax[blockIdx.x] = v;
    }
}

void launch_pnorm(const Geo &g, const Slab &sl, int s, double *part, int nblk, const DevState *st, cudaStream_t stream)
{
    k_pnorm<<<nblk, 256, 0, stream>>>(sl.P + g.plane, g.vstride, (int64_t)sl.nzl * g.plane, s, part, st);
}

void launch_budget(const double *part, int nparts, double *sum, double anorm, bool allreduce_needed,
                   const DevState *st, const double *h_delta, double *h_pnorm, double *h_budget, cudaStream_t stream,
                   int phase)
{
    if (phase == 0) k_psum<<<1, 32, 0, stream>>>(part, nparts, sum, st);
    else k_budget<<<1, 1, 0, stream>>>(sum, anorm, st, h_delta, h_pnorm, h_budget);
    (void)allreduce_needed;
}

void launch_anorm(const Geo &g, const Slab &sl, double *bmax, int nblk, cudaStream_t stream)
{
    k_anorm<<<nblk, 256, 0, stream>>>(g, sl.kx, sl.ky, sl.kz, sl.nzl, bmax);
}

void launch_kappa(const double *blk, int s, const DevState *st, double *h_kappa, cudaStream_t stream)
{
    k_kappa<<<1, 32, 0, stream>>>(blk, s, st, h_kappa);
}

void launch_k5(const Geo &g, const Slab &sl, int s, const double *alpha, double *const *xpp, int64_t xoff,
               const DevState *st, cudaStream_t stream, int zb, int ze, double theta, double sigma, bool rec,
               bool fold)
{
    if (ze < 0) ze = sl.nzl + 1;
    if (ze <= zb) return;
    K5Params k;
    k.P = sl.P + (int64_t)zb * g.plane;
    k.W = sl.W + (int64_t)zb * g.plane;
    k.vstride = g.vstride;
    k.N = (int64_t)(ze - zb) * g.plane;
    k.rec = rec && s >= 2;
    k.theta = theta;
    k.sigma = sigma;
    k.dm = g.center;
    k.dvec = sl.dvec ? sl.dvec + (int64_t)zb * g.plane : nullptr;
    k.xpp = xpp;
    k.xoff = xoff + (int64_t)(zb - 1) * g.nx * g.ny;
    k.s = s;
    k.alpha = alpha;
    k.nx = g.nx;
    k.pitch = g.pitch;
    k.ny = g.ny;
    k.plane = g.plane;
    k.inv_nx = 1.0 / g.nx;
    k.inv_ny = 1.0 / g.ny;
    k.center = g.center;
    const bool vec = (g.pitch == g.nx) && (k.N % 2 == 0) && (k.xoff % 2 == 0);
    const int64_t work = vec ? k.N / 2 : k.N;
    int64_t blocks = (work + 255) / 256;
#ifndef K5_BLOCKS_PER_SM
#define K5_BLOCKS_PER_SM 256   // measured at cfg 5: 8 -> 2.22 ms, 64 -> 2.13, 256 -> 2.09, 4096 -> 2.11
#endif
    const int64_t cap = (int64_t)k2_grid() * K5_BLOCKS_PER_SM;
    if (blocks > cap) blocks = cap;
    // fold => rec and pitch == nx with nx even (uses_wlfold), so the flat path applies
    if (vec && k.rec && fold) {
        switch (s) {
        case 16: launch_pdl(g.kn.pdl, k5_update_vec<16, true, true>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        case 24: launch_pdl(g.kn.pdl, k5_update_vec<24, true, true>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        case 32: launch_pdl(g.kn.pdl, k5_update_vec<32, true, true>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        default: launch_pdl(g.kn.pdl, k5_update_vec<0, true, true>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        }
    } else if (vec && k.rec) {
        switch (s) {
        case 4: launch_pdl(g.kn.pdl, k5_update_vec<4, true, false>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        case 8: launch_pdl(g.kn.pdl, k5_update_vec<8, true, false>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        case 16: launch_pdl(g.kn.pdl, k5_update_vec<16, true, false>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        case 24: launch_pdl(g.kn.pdl, k5_update_vec<24, true, false>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        case 32: launch_pdl(g.kn.pdl, k5_update_vec<32, true, false>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        default: launch_pdl(g.kn.pdl, k5_update_vec<0, true, false>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        }
    } else if (vec) {
        switch (s) {
        case 4: launch_pdl(g.kn.pdl, k5_update_vec<4, false, false>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        case 8: launch_pdl(g.kn.pdl, k5_update_vec<8, false, false>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        case 16: launch_pdl(g.kn.pdl, k5_update_vec<16, false, false>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        case 24: launch_pdl(g.kn.pdl, k5_update_vec<24, false, false>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        case 32: launch_pdl(g.kn.pdl, k5_update_vec<32, false, false>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        default: launch_pdl(g.kn.pdl, k5_update_vec<0, false, false>, dim3((unsigned)blocks), dim3(256), 0, stream, k, st); break;
        }
    }
    else launch_pdl(g.kn.pdl, k5_update_gen, dim3((unsigned)blocks), dim3(256), 0, stream, k, st);
}

}  // namespace sscg
