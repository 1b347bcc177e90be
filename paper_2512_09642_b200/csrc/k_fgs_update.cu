// K4 -- Ruhe scaling + nu Forward Gauss-Seidel sweeps on the s x s Gram
//       system, stopping test and history (single warp).
// K5 -- fused solution/residual update x += P alpha, r -= (AP) alpha
//       (r is stored in place of p_0).
#include "sscg_internal.cuh"

namespace sscg {
namespace {

constexpr int SMAX = 64;

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One warp; lane l owns rows i = l and i = l + 32.
//   d_i = Ghat_ii^{-1/2};  G = S Ghat S with G_ii := 1;  c~ = S c
//   FGS sweep (I + L) a^(l+1) = c~ - L^T a^(l) in residual form: with
//   rho = c~ - G a (unit diagonal), coordinate j takes a_j += rho_j and every
//   other row updates rho_i -= G_ij rho_j (rho_j becomes 0) -- the same
//   forward substitution a_j = c~_j - sum_{i != j} G_ji a_i,
//   evaluated with one shuffle + one FMA per coordinate instead of a dot.
__global__ void __launch_bounds__(32) k4_fgs(K4Args a, DevState *st)
{
    if (st->done) return;
    __shared__ double Gc[SMAX * SMAX];   // column-major: Gc[j*s + i] = G_ij
    const int s = a.s, lane = threadIdx.x;
    const int k = st->k;
    const double *Gh = a.blk, *c = a.blk + s * s;
    const int nent = s * s + s;
    const bool rec = k < st->hist_cap;
    if (rec)
        for (int q = lane; q < nent; q += 32) a.h_gram[(int64_t)k * nent + q] = a.blk[q];

    const double rn = sqrt(c[0]);
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
    double d0 = 0.0, d1 = 0.0;
    bool ok = true;
    if (i0 < s) { const double gdiag = Gh[i0 * s + i0]; ok &= (gdiag > 0.0) && isfinite(gdiag); d0 = 1.0 / sqrt(gdiag); }
    if (i1 < s) { const double gdiag = Gh[i1 * s + i1]; ok &= (gdiag > 0.0) && isfinite(gdiag); d1 = 1.0 / sqrt(gdiag); }
    if (!__all_sync(0xffffffffu, ok)) {
        if (lane == 0) { st->breakdown = 1; st->done = 1; st->outer = k; }
        return;
    }
    __shared__ double dsh[SMAX];
    if (i0 < s) dsh[i0] = d0;
    if (i1 < s) dsh[i1] = d1;
    __syncwarp();
    for (int q = lane; q < s * s; q += 32) {
        const int i = q / s, j = q - i * s;
        Gc[j * s + i] = (i == j) ? 1.0 : (dsh[i] * Gh[q]) * dsh[j];
    }
    const double ct0 = (i0 < s) ? d0 * c[i0] : 0.0;
    const double ct1 = (i1 < s) ? d1 * c[i1] : 0.0;
    __syncwarp();

    double rho0 = ct0, rho1 = ct1, al0 = 0.0, al1 = 0.0;
    for (int sw = 0; sw < a.nu; ++sw) {
        for (int j = 0; j < s; ++j) {
            const int owner = j & 31;
            const double src = (j < 32) ? rho0 : rho1;
            const double dj = __shfl_sync(0xffffffffu, src, owner);
            if (j < 32) {
                if (lane == owner) { al0 += dj; rho0 = 0.0; }
                else if (i0 < s) rho0 = fma(-Gc[j * s + i0], dj, rho0);
                if (i1 < s) rho1 = fma(-Gc[j * s + i1], dj, rho1);
            } else {
                if (i0 < s) rho0 = fma(-Gc[j * s + i0], dj, rho0);
                if (lane == owner) { al1 += dj; rho1 = 0.0; }
                else if (i1 < s) rho1 = fma(-Gc[j * s + i1], dj, rho1);
            }
        }
    }
    // explicit residual of the Gram system: delta = ||c~ - G a~|| / ||c~||
    double res0 = ct0, res1 = ct1;
    for (int j = 0; j < s; ++j) {
        const double aj = __shfl_sync(0xffffffffu, (j < 32) ? al0 : al1, j & 31);
        if (i0 < s) res0 = fma(-Gc[j * s + i0], aj, res0);
        if (i1 < s) res1 = fma(-Gc[j * s + i1], aj, res1);
    }
    const double rr = warp_sum(res0 * res0 + res1 * res1);
    const double cc = warp_sum(ct0 * ct0 + ct1 * ct1);
    if (i0 < s) a.alpha[i0] = d0 * al0;
    if (i1 < s) a.alpha[i1] = d1 * al1;
    if (rec) {
        if (i0 < s) { a.h_d[(int64_t)k * s + i0] = d0; a.h_at[(int64_t)k * s + i0] = al0; a.h_al[(int64_t)k * s + i0] = d0 * al0; }
        if (i1 < s) { a.h_d[(int64_t)k * s + i1] = d1; a.h_at[(int64_t)k * s + i1] = al1; a.h_al[(int64_t)k * s + i1] = d1 * al1; }
        if (lane == 0) a.h_delta[k] = sqrt(rr) / sqrt(cc);
    }
    if (lane == 0) {
        st->outer = k + 1;
        st->k = k + 1;
    }
}

struct K5Params {
    const double *P;   // interior start of p_0 (= r_k)
    const double *W;   // interior start of w_0
    int64_t vstride;
    int64_t N;         // interior doubles (nzl * plane)
    int s;
    const double *alpha;
    double *x;         // process-layout x of this slab
    int nx, pitch;
};

// flat path: pitch == nx and x 16-B aligned; 2 points per thread per step.
__global__ void __launch_bounds__(256) k5_update_vec(K5Params k, const DevState *st)
{
    if (st->done) return;
    __shared__ double al[SMAX];
    for (int j = threadIdx.x; j < k.s; j += blockDim.x) al[j] = k.alpha[j];
    __syncthreads();
    const int64_t n2 = k.N >> 1;
    const double2 *P2 = reinterpret_cast<const double2 *>(k.P);
    const double2 *W2 = reinterpret_cast<const double2 *>(k.W);
    double2 *x2 = reinterpret_cast<double2 *>(k.x);
    double2 *r2 = reinterpret_cast<double2 *>(const_cast<double *>(k.P));
    const int64_t vs2 = k.vstride >> 1;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n2; e += (int64_t)gridDim.x * blockDim.x) {
        double2 ax = make_double2(0.0, 0.0), aw = make_double2(0.0, 0.0);
        const double2 p0 = __ldcs(P2 + e);
        for (int j = 0; j < k.s; ++j) {
            const double2 pj = (j == 0) ? p0 : __ldcs(P2 + j * vs2 + e);
            const double2 wj = __ldcs(W2 + j * vs2 + e);
            ax.x = fma(al[j], pj.x, ax.x); ax.y = fma(al[j], pj.y, ax.y);
            aw.x = fma(al[j], wj.x, aw.x); aw.y = fma(al[j], wj.y, aw.y);
        }
        double2 xv = x2[e];
        xv.x += ax.x; xv.y += ax.y;
        x2[e] = xv;
        r2[e] = make_double2(p0.x - aw.x, p0.y - aw.y);
    }
}

// generic path (odd nx / unaligned x): scalar, skips the pad column.
__global__ void __launch_bounds__(256) k5_update_gen(K5Params k, const DevState *st)
{
    if (st->done) return;
    __shared__ double al[SMAX];
    for (int j = threadIdx.x; j < k.s; j += blockDim.x) al[j] = k.alpha[j];
    __syncthreads();
    double *r = const_cast<double *>(k.P);
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
        k.x[xi] += ax;
        r[e] = p0 - aw;
    }
}

}  // namespace

void launch_k4(const K4Args &a, DevState *st, cudaStream_t s) { k4_fgs<<<1, 32, 0, s>>>(a, st); }

void launch_k5(const Geo &g, const Slab &sl, int s, const double *alpha, double *x_slab, const DevState *st,
               cudaStream_t stream)
{
    K5Params k;
    k.P = sl.P + g.plane;
    k.W = sl.W + g.plane;
    k.vstride = g.vstride;
    k.N = (int64_t)sl.nzl * g.plane;
    k.s = s;
    k.alpha = alpha;
    k.x = x_slab;
    k.nx = g.nx;
    k.pitch = g.pitch;
    const bool vec = (g.pitch == g.nx) && ((reinterpret_cast<uintptr_t>(x_slab) & 15) == 0) && (k.N % 2 == 0);
    const int64_t work = vec ? k.N / 2 : k.N;
    int64_t blocks = (work + 255) / 256;
    const int64_t cap = (int64_t)k2_grid() * 8;
    if (blocks > cap) blocks = cap;
    if (vec) k5_update_vec<<<(unsigned)blocks, 256, 0, stream>>>(k, st);
    else k5_update_gen<<<(unsigned)blocks, 256, 0, stream>>>(k, st);
}

}  // namespace sscg
