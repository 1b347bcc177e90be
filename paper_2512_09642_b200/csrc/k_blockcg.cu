// Block-conjugate s-step CG (DESIGN.md
// R24) on the same boundary as the restart form.  The previous
// search block Q' and Z' = A Q' are kept in the upper halves of P and W
// (vectors s..2s-1), so the stored-W Gram pass over the 2s vectors [P_k | Q']
// and [W_k | Z'] gives, in ONE pass and ONE allreduce of the 2s x (2s+1)
// block: Ghat = P_k^T A P_k, c = P_k^T r_k (the restart system), the cross
// block C^T = P_k^T Z', e = Q'^T r_k and G' = Q'^T Z'.  Then
//   K4B (k_bcg_prep, one warp): B = G'^{-1} C (Cholesky of G'),
//        G_k = Ghat - C^T B,  c_k = c - B^T e   (= Q_k^T A Q_k, Q_k^T r_k)
//   K4  (unchanged FGS / Cholesky kernel) on (G_k, c_k); the stopping test
//        reads ||r_k||^2 = c_0 of the raw block
//   K5B (k5_block): Q_k = P_k - Q' B, Z_k = W_k - Z' B (in place of Q', Z'),
//        x += Q_k alpha, r_{k+1} = p_0 - Z_k alpha (into p_0)
// At the first outer iteration of a solve (k = 0) there is no previous block:
// B = 0, G_k = Ghat, c_k = c -- the restart step.
#include <algorithm>

#include "sscg_internal.cuh"

namespace sscg {
namespace {

constexpr int SB = 32;   // largest s of the block-conjugate mode (2s <= 64 Gram rows)

// big: [(2s) x (2s) row-major | c2 (2s)] from the Gram pass over [P | Q'],
// [W | Z'];  out: blk2 = [G_k (s x s) | c_k (s)],  Bm = B (s x s, row-major)
__global__ void __launch_bounds__(32) k_bcg_prep(const double *big, int s, double *blk2, double *Bm, DevState *st)
{
    PDL_ENTRY(st);
    __shared__ double R[SB * SB], Cm[SB * SB], Bs[SB * SB], e[SB];
    const int lane = threadIdx.x, S2 = 2 * s, k = st->k;
    const double *c2 = big + S2 * S2;
    if (k == 0) {   // no previous block: the restart system, B = 0
        for (int q = lane; q < s * s; q += 32) {
            const int i = q / s, j = q - i * s;
            blk2[q] = big[i * S2 + j];
            Bm[q] = 0.0;
        }
        for (int i = lane; i < s; i += 32) blk2[s * s + i] = c2[i];
        return;
    }
    // C_ij = z'_i^T p_j = entry (j, s + i) of the big block; G' = rows/cols s..2s-1; e = c2[s..]
    for (int q = lane; q < s * s; q += 32) {
        const int i = q / s, j = q - i * s;
        Cm[q] = big[j * S2 + s + i];
        R[q] = big[(s + i) * S2 + s + j];
    }
    for (int i = lane; i < s; i += 32) e[i] = c2[s + i];
    __syncwarp();
    // G' = R^T R (upper R in place; row kk of R after its last use as G')
    for (int kk = 0; kk < s; ++kk) {
        double piv = R[kk * s + kk];
        for (int m = 0; m < kk; ++m) piv -= R[m * s + kk] * R[m * s + kk];
        if (!(piv > 0.0) || !isfinite(piv)) {
            if (lane == 0) { st->breakdown = 1; st->done = 1; st->outer = k; }
            return;
        }
        const double rkk = sqrt(piv);
        for (int j = kk + 1 + lane; j < s; j += 32) {
            double b = R[kk * s + j];
            for (int m = 0; m < kk; ++m) b -= R[m * s + kk] * R[m * s + j];
            R[kk * s + j] = b / rkk;
        }
        __syncwarp();
        if (lane == 0) R[kk * s + kk] = rkk;
        __syncwarp();
    }
    // B = G'^{-1} C: lane j solves R^T y = C[:, j], R b = y
    for (int j = lane; j < s; j += 32) {
        for (int i = 0; i < s; ++i) {
            double a = Cm[i * s + j];
            for (int m = 0; m < i; ++m) a -= R[m * s + i] * Bs[m * s + j];
            Bs[i * s + j] = a / R[i * s + i];
        }
        for (int i = s - 1; i >= 0; --i) {
            double a = Bs[i * s + j];
            for (int m = i + 1; m < s; ++m) a -= R[i * s + m] * Bs[m * s + j];
            Bs[i * s + j] = a / R[i * s + i];
        }
    }
    __syncwarp();
    // G_k = Ghat - C^T B (i <= j, mirrored), c_k = c - B^T e; lane i owns row i
    for (int i = lane; i < s; i += 32) {
        for (int j = i; j < s; ++j) {
            double v = 0.0;
            for (int m = 0; m < s; ++m) v += Cm[m * s + i] * Bs[m * s + j];
            const double gij = big[i * S2 + j] - v;
            blk2[i * s + j] = gij;
            blk2[j * s + i] = gij;
        }
        double v = 0.0;
        for (int m = 0; m < s; ++m) v += Bs[m * s + i] * e[m];
        blk2[s * s + i] = c2[i] - v;
    }
    for (int q = lane; q < s * s; q += 32) Bm[q] = Bs[q];
}

struct K5BParams {
    double *P, *W;        // interior start of p_0 / w_0 of this launch's planes (Q' = P + s*vstride, ...)
    int64_t vstride, N;   // N: doubles of the launch's planes (incl. pad columns)
    int s, nx, pitch;
    const double *alpha, *B;
    double *const *xpp;   // device cell with the caller's x (process layout)
    int64_t xoff;
    double inv_theta, inv_2theta, sigma, dm;   // REC: W_k recovered from P_k (constant diagonal m)
};

// one phase of the update at one point: y_j = v_j - sum_m o_m B_mj for the s
// columns j (v = P_k or W_k, o = Q' or Z' of the point, already in registers),
// y_j stored over o_j's slot, returns sum_j alpha_j y_j.  Columns in groups of
// four whose loads are issued together; the restrict pointers tell the
// compiler the basis loads and the block stores never overlap (they are
// different vectors), so loads are not held behind earlier stores.
template <int S>
__device__ __forceinline__ double bcg_phase(const double *__restrict__ v, double *__restrict__ y, int64_t vs,
                                            int s, const double (&o)[S], const double *Bsh, const double *al)
{
    double acc = 0.0;
#pragma unroll 1
    for (int j0 = 0; j0 < s; j0 += 4) {
        double vj[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) vj[u] = (j0 + u < s) ? v[(int64_t)(j0 + u) * vs] : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = j0 + u;
            double sp = 0.0;
#pragma unroll
            for (int m = 0; m < S; ++m) sp = fma(o[m], Bsh[m * S + j], sp);
            const double yj = vj[u] - sp;
            if (j < s) {
                y[(int64_t)j * vs] = yj;
                acc = fma(al[j], yj, acc);
            }
        }
    }
    return acc;
}

// one point per thread (grid-stride): Q' (Z') of the point is loaded before
// Q_k (Z_k) overwrites it.  REC (the W-free block mode): W_k is not stored but
// recovered per point from the P_k values the first phase loads, in K2R's
// arithmetic (w_0 = m(p_1/theta + sigma p_0), w_j = m((p_{j+1} + p_{j-1})/(2 theta)
// + sigma p_j), w_{s-1} from its stored row) -- the W_k the Gram pass used.
template <int S, bool REC>
__global__ void __launch_bounds__(256) k5_block(K5BParams k, const DevState *st)
{
    PDL_ENTRY(st);
    __shared__ double Bsh[S * (S + 4)], al[S + 4];   // padded: groups of four columns past s read zeros
    const int s = k.s;
    for (int q = threadIdx.x; q < S * (S + 4); q += blockDim.x) {
        const int i = q / S, j = q % S;
        Bsh[q] = (i < s && j < s) ? k.B[i * s + j] : 0.0;
    }
    for (int q = threadIdx.x; q < S + 4; q += blockDim.x) al[q] = (q < s) ? k.alpha[q] : 0.0;
    __syncthreads();
    double *x = *k.xpp + k.xoff;
    const int64_t vs = k.vstride;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < k.N; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e / k.pitch;
        const int xx = (int)(e - row * k.pitch);
        if (xx >= k.nx) continue;   // pad column
        double o[S];
        // x += Q_k alpha with Q_k = P_k - Q' B
#pragma unroll
        for (int i = 0; i < S; ++i) o[i] = (i < s) ? k.P[(int64_t)(s + i) * vs + e] : 0.0;
        const double p0 = k.P[e];
        double ax, aw;
        if constexpr (REC) {
            // both phases in one pass over groups of four columns: Q' and Z' of the
            // point in registers first (their slots are overwritten), each P_k row
            // loaded once (one row of lookahead for w_j's p_{j+1})
            double o2[S];
#pragma unroll
            for (int i = 0; i < S; ++i) o2[i] = (i < s) ? k.W[(int64_t)(s + i) * vs + e] : 0.0;
            const double wl = k.W[(int64_t)(s - 1) * vs + e];
            const double c1a = k.inv_theta * k.dm, c1b = k.inv_2theta * k.dm, cs = k.sigma * k.dm;
            const double *pp = k.P + e;
            double *qy = k.P + (int64_t)s * vs + e, *zy = k.W + (int64_t)s * vs + e;
            double pprev = 0.0, pnext = pp[0];   // p_{j0-1}, p_{j0}
            ax = 0.0;
            aw = 0.0;
#pragma unroll 1
            for (int j0 = 0; j0 < s; j0 += 4) {
                double pv[5];
                pv[0] = pnext;
#pragma unroll
                for (int u = 1; u < 5; ++u) pv[u] = (j0 + u < s) ? pp[(int64_t)(j0 + u) * vs] : 0.0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j0 + u;
                    if (j >= s) break;
                    const double pj = pv[u], dn = (u == 0) ? pprev : pv[u - 1];
                    // w_j as K2R forms it (w_{s-1} stored)
                    const double wj = (j == s - 1) ? wl
                                                   : fma(pv[u + 1], j == 0 ? c1a : c1b, fma(j > 0 ? dn : pj, j > 0 ? c1b : 0.0, cs * pj));
                    double sq = 0.0, sz = 0.0;
#pragma unroll
                    for (int m = 0; m < S; ++m) {
                        sq = fma(o[m], Bsh[m * S + j], sq);
                        sz = fma(o2[m], Bsh[m * S + j], sz);
                    }
                    const double qj = pj - sq, zj = wj - sz;
                    qy[(int64_t)j * vs] = qj;
                    zy[(int64_t)j * vs] = zj;
                    ax = fma(al[j], qj, ax);
                    aw = fma(al[j], zj, aw);
                }
                pprev = pv[3];
                pnext = pv[4];
            }
        } else {
            ax = bcg_phase<S>(k.P + e, k.P + (int64_t)s * vs + e, vs, s, o, Bsh, al);
            // r_{k+1} = p_0 - Z_k alpha with Z_k = W_k - Z' B
#pragma unroll
            for (int i = 0; i < S; ++i) o[i] = (i < s) ? k.W[(int64_t)(s + i) * vs + e] : 0.0;
            aw = bcg_phase<S>(k.W + e, k.W + (int64_t)s * vs + e, vs, s, o, Bsh, al);
        }
        const int64_t xi = row * k.nx + xx;
        x[xi] = x[xi] + ax;
        k.P[e] = p0 - aw;
    }
}

}  // namespace

void launch_bcg_prep(const double *big, int s, double *blk2, double *Bm, DevState *st, bool pdl, cudaStream_t strm)
{
    launch_pdl(pdl, k_bcg_prep, dim3(1), dim3(32), 0, strm, big, s, blk2, Bm, st);
}

void launch_k5_block(const Geo &g, const Slab &sl, int s, const double *alpha, const double *B, double *const *xpp,
                     int64_t xoff, const DevState *st, cudaStream_t stream, int zb, int ze, bool rec, double theta,
                     double sigma)
{
    if (ze < 0) ze = sl.nzl + 1;
    if (ze <= zb) return;
    K5BParams k;
    k.P = sl.P + (int64_t)zb * g.plane;
    k.W = sl.W + (int64_t)zb * g.plane;
    k.vstride = g.vstride;
    k.N = (int64_t)(ze - zb) * g.plane;
    k.s = s;
    k.nx = g.nx;
    k.pitch = g.pitch;
    k.alpha = alpha;
    k.B = B;
    k.xpp = xpp;
    k.xoff = xoff + (int64_t)(zb - 1) * g.nx * g.ny;
    k.inv_theta = 1.0 / theta;
    k.inv_2theta = 1.0 / (2.0 * theta);
    k.sigma = sigma;
    k.dm = g.center;
    const unsigned blocks = (unsigned)std::min<int64_t>((k.N + 255) / 256, (int64_t)k2_grid() * 16);
    if (rec) {
        if (s <= 8) launch_pdl(g.kn.pdl, k5_block<8, true>, dim3(blocks), dim3(256), 0, stream, k, st);
        else launch_pdl(g.kn.pdl, k5_block<16, true>, dim3(blocks), dim3(256), 0, stream, k, st);
        return;
    }
    if (s <= 8) launch_pdl(g.kn.pdl, k5_block<8, false>, dim3(blocks), dim3(256), 0, stream, k, st);
    else if (s <= 16) launch_pdl(g.kn.pdl, k5_block<16, false>, dim3(blocks), dim3(256), 0, stream, k, st);
    else launch_pdl(g.kn.pdl, k5_block<32, false>, dim3(blocks), dim3(256), 0, stream, k, st);
}

}  // namespace sscg
