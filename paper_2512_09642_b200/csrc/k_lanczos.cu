// Spectral bounds of M^{-1}A by Lanczos (PAPER.md:311
// "bounds ... estimated with Lanczos", BASELINE cfg 3/4: 50 steps, widened
// 5 %).  Lanczos runs on the symmetric D^{-1/2} A D^{-1/2} (same spectrum as
// M^{-1}A, D = M) from v_0 = b/||b|| without reorthogonalisation.  It is
// carried out in the scaled variable y = D^{-1/2} v, so the operator step is
// the plain stencil/CSR SpMV of K1 (mode 0) on y:
//   a_k = y_k^T A y_k                      (= v_k^T D^{-1/2}AD^{-1/2} v_k)
//   z   = D^{-1} A y_k - a_k y_k - b_{k-1} y_{k-1}   (= D^{-1/2} u_k)
//   b_k = (z^T D z)^{1/2},  y_{k+1} = z / b_k
// Two reductions per step (fixed-order per-CTA partials, last-CTA ordered
// sum; summed over slabs in order and over ranks by one ncclAllReduce each).
// The extreme eigenvalues of the tridiagonal T_m = tridiag(b, a, b) are found
// on the device by bisection on the Sturm sign count of T_m - x I.
#include <cmath>

#include "sscg_internal.cuh"

namespace sscg {
namespace {

constexpr int LZ_THREADS = 256;

__global__ void k_lz_diag(Geo g, const double *kx, const double *ky, const double *kz, const double *dinv, double *D,
                          int nzl)
{
    const int64_t nxy = (int64_t)g.nx * g.ny, tot = nxy * nzl;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t zl = e / nxy, rem = e - zl * nxy;
        const int64_t y = rem / g.nx, x = rem - y * g.nx;
        const int64_t i = (zl + 1) * g.plane + y * g.pitch + x;
        double d;
        if (dinv) {
            d = 1.0 / dinv[i];
        } else if (g.kind == 3) {   // A_ii = sum of the six faces (R12)
            // same summation order as the basis kernels: kz-, ky-, kx-, kx+, ky+, kz+
            d = kz[(zl * g.ny + y) * g.nx + x] + ky[(zl * (g.ny + 1) + y) * g.nx + x] +
                kx[(zl * g.ny + y) * (g.nx + 1) + x] + kx[(zl * g.ny + y) * (g.nx + 1) + x + 1] +
                ky[(zl * (g.ny + 1) + y + 1) * g.nx + x] + kz[((zl + 1) * g.ny + y) * g.nx + x];
        } else {
            d = g.center;
        }
        D[i] = d;
    }
}

// y (padded) = v0 (process layout) / (||v0|| sqrt(D))
__global__ void k_lz_init(Geo g, const double *v0, const double *D, const double *nrm2, double *y, int nzl)
{
    const double inv = 1.0 / sqrt(*nrm2);
    const int64_t nxy = (int64_t)g.nx * g.ny, tot = nxy * nzl;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t zl = e / nxy, rem = e - zl * nxy;
        const int64_t yy = rem / g.nx, x = rem - yy * g.nx;
        const int64_t i = (zl + 1) * g.plane + yy * g.pitch + x;
        y[i] = (v0[e] * inv) / sqrt(D[i]);
    }
}

// sum over the interior doubles of x.y (mode 0) or D x.x (mode 1); pad
// columns hold zeros.  Deterministic: fixed per-CTA tree, last CTA sums the
// partials in index order.
__global__ void __launch_bounds__(LZ_THREADS) k_lz_dot(const double *x, const double *y, const double *D, int64_t N,
                                                       int mode, double *part, unsigned *ticket, double *out,
                                                       const int *stop)
{
    if (stop && *stop) return;
    __shared__ double red[LZ_THREADS / 32];
    __shared__ bool last;
    double acc = 0.0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x)
        acc = (mode == 0) ? fma(x[e], y[e], acc) : fma(D[e] * x[e], x[e], acc);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < LZ_THREADS / 32; ++w) v += red[w];
        part[blockIdx.x] = v;
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    double v = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) v += __ldcg(part + b);
    *out = v;
    *ticket = 0u;
}

// fixed-order sum of per-slab scalars
__global__ void k_lz_sum(const double *vals, int n, double *out, const int *stop)
{
    if (*stop) return;
    double v = 0.0;
    for (int i = 0; i < n; ++i) v += vals[i];
    *out = v;
}

// z = w / D - a y - bprev yp   over the interior doubles (pad columns: D = 0, z = 0)
__global__ void k_lz_update(const double *w, const double *D, const double *y, const double *yp, double *z, int64_t N,
                            const double *a, const double *bprev, const int *stop)
{
    if (*stop) return;
    const double av = *a, bv = *bprev;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x)
        z[e] = (D[e] != 0.0) ? (w[e] / D[e] - av * y[e]) - bv * yp[e] : 0.0;
}

// record a_k, b_k; b_k = 0 (an invariant subspace) stops the iteration
__global__ void k_lz_record(const double *a, const double *b2, double *alpha, double *beta, double *bprev, int k,
                            int *stop, int *m)
{
    if (*stop) return;
    const double b = sqrt(*b2);
    alpha[k] = *a;
    beta[k] = b;
    *bprev = b;
    *m = k + 1;
    if (!(b > 0.0)) *stop = 1;
}

__global__ void k_lz_scale(double *z, int64_t N, const double *bprev, const int *stop)
{
    if (*stop) return;
    const double inv = 1.0 / *bprev;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x)
        z[e] *= inv;
}

// number of eigenvalues of T_m below x: signs of the pivots of the LDL^T
// factorisation of T_m - x I (a zero pivot is nudged to a tiny negative value)
__device__ int below(const double *a, const double *b, int m, double x)
{
    int cnt = 0;
    double piv = 1.0;
    for (int i = 0; i < m; ++i) {
        const double off = (i > 0) ? b[i - 1] * b[i - 1] / piv : 0.0;
        piv = (a[i] - x) - off;
        if (piv == 0.0) piv = -1e-300;
        cnt += piv < 0.0;
    }
    return cnt;
}

// thread 0: smallest, thread 1: largest eigenvalue of T_m, bisection inside
// the Gershgorin interval to full precision; widened by (1 -+ margin)
__global__ void k_lz_extremes(const double *alpha, const double *beta, const int *mptr, double margin, double *out)
{
    const int t = threadIdx.x;
    if (t > 1) return;
    const int m = *mptr;
    double lo = 1e300, hi = -1e300;
    for (int i = 0; i < m; ++i) {
        const double r = (i > 0 ? fabs(beta[i - 1]) : 0.0) + (i + 1 < m ? fabs(beta[i]) : 0.0);
        lo = fmin(lo, alpha[i] - r);
        hi = fmax(hi, alpha[i] + r);
    }
    const int want = (t == 0) ? 0 : m - 1;   // eigenvalue index (ascending)
    for (int it = 0; it < 2000; ++it) {
        const double mid = lo + 0.5 * (hi - lo);
        if (mid <= lo || mid >= hi) break;
        if (below(alpha, beta, m, mid) > want) hi = mid;
        else lo = mid;
    }
    const double ev = lo + 0.5 * (hi - lo);
    out[t] = (t == 0) ? ev * (1.0 - margin) : ev * (1.0 + margin);
}

}  // namespace

int lz_grid() { return k2_grid() * 4; }

void lz_diag(const Geo &g, const Slab &sl, double *D, cudaStream_t s)
{
    const int64_t tot = (int64_t)g.nx * g.ny * sl.nzl;
    k_lz_diag<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 16), 256, 0, s>>>(g, sl.kx, sl.ky, sl.kz, sl.dinv,
                                                                                      D, sl.nzl);
}

void lz_init(const Geo &g, const Slab &sl, const double *v0, const double *D, const double *nrm2, double *y,
             cudaStream_t s)
{
    const int64_t tot = (int64_t)g.nx * g.ny * sl.nzl;
    k_lz_init<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 16), 256, 0, s>>>(g, v0, D, nrm2, y, sl.nzl);
}

void lz_dot(const double *x, const double *y, const double *D, int64_t N, int mode, double *part, unsigned *ticket,
            double *out, const int *stop, cudaStream_t s)
{
    k_lz_dot<<<lz_grid(), LZ_THREADS, 0, s>>>(x, y, D, N, mode, part, ticket, out, stop);
}

void lz_sum(const double *vals, int n, double *out, const int *stop, cudaStream_t s)
{
    k_lz_sum<<<1, 1, 0, s>>>(vals, n, out, stop);
}

void lz_update(const double *w, const double *D, const double *y, const double *yp, double *z, int64_t N,
               const double *a, const double *bprev, const int *stop, cudaStream_t s)
{
    k_lz_update<<<lz_grid(), 256, 0, s>>>(w, D, y, yp, z, N, a, bprev, stop);
}

void lz_record(const double *a, const double *b2, double *alpha, double *beta, double *bprev, int k, int *stop, int *m,
               cudaStream_t s)
{
    k_lz_record<<<1, 1, 0, s>>>(a, b2, alpha, beta, bprev, k, stop, m);
}

void lz_scale(double *z, int64_t N, const double *bprev, const int *stop, cudaStream_t s)
{
    k_lz_scale<<<lz_grid(), 256, 0, s>>>(z, N, bprev, stop);
}

void lz_extremes(const double *alpha, const double *beta, const int *m, double margin, double *out, cudaStream_t s)
{
    k_lz_extremes<<<1, 32, 0, s>>>(alpha, beta, m, margin, out);
}

}  // namespace sscg
