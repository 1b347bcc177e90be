// K1 -- fused stencil/CSR SpMV + Jacobi + Chebyshev three-term recurrence.
//
// For basis step j (§2 Def. Chebyshev Polynomial Basis):
//   w_j     = A p_j
//   p_{j+1} = coef * (M^{-1} w_j - sigma p_j) [- p_{j-1}]
// with coef = theta at j = 0 and 2 theta (minus p_{j-1}) for j >= 1; at
// j = s-1 only w_j is produced (W = AP feeds the Gram pass).  One launch per
// step streams p_j (read once from HBM: z-neighbours come from a register
// sliding window, x/y neighbours from L1), p_{j-1}, and writes w_j, p_{j+1}:
// 4 vectors = 32 B per grid point (the roofline unit of DESIGN.md §K1).
//
// Layout (sscg_internal.cuh Slab/Geo): plane = ny*pitch doubles, one halo
// plane below and above the slab (zero at global Dirichlet boundaries,
// exchanged between slabs).  x/y Dirichlet ghosts are handled by predicates.
#include "sscg_internal.cuh"

namespace sscg {
namespace {

constexpr int BX = 32, BY = 8;

__device__ __forceinline__ double ld(const double *p) { return __ldg(p); }

// Column-marching kernel: thread (x, y) walks planes [z_lo, z_hi) keeping
// p(z-1), p(z), p(z+1) of its own column in registers.
template <int KIND>
__global__ void __launch_bounds__(BX *BY) k1_stencil(Geo g, K1Args a, const DevState *st, int zc)
{
    if (st && st->done) return;
    const int x = blockIdx.x * BX + threadIdx.x;
    const int y = blockIdx.y * BY + threadIdx.y;
    const int z_lo = a.zb + blockIdx.z * zc;
    const int z_hi = min(a.ze, z_lo + zc);
    if (x >= g.nx || y >= g.ny || z_lo >= z_hi) return;
    const int64_t pl = g.plane;
    const int pitch = g.pitch;
    const bool xm = x > 0, xp = x + 1 < g.nx, ym = y > 0, yp = y + 1 < g.ny;
    const double *p = a.p;
    int64_t i = (int64_t)z_lo * pl + (int64_t)y * pitch + x;

    double c_m, c_0, c_p;         // own column: z-1, z, z+1 (7-pt / var-coef)
    double b_m = 0, b_0 = 0, b_p; // 3x3 box sums of planes z-1, z, z+1 (27-pt)
    double kz_lo = 0;             // var-coef: face below the current cell

    auto box2 = [&](int64_t j) -> double {
        // 3x3 in-plane box sum (27-pt separable form: A p = 27 p - box3(p))
        double r = ld(p + j);
        if (xm) r += ld(p + j - 1);
        if (xp) r += ld(p + j + 1);
        if (ym) {
            r += ld(p + j - pitch);
            if (xm) r += ld(p + j - pitch - 1);
            if (xp) r += ld(p + j - pitch + 1);
        }
        if (yp) {
            r += ld(p + j + pitch);
            if (xm) r += ld(p + j + pitch - 1);
            if (xp) r += ld(p + j + pitch + 1);
        }
        return r;
    };

    if (KIND == 2) {
        b_m = box2(i - pl);
        b_0 = box2(i);
        c_0 = ld(p + i);
    } else {
        c_m = ld(p + i - pl);
        c_0 = ld(p + i);
    }
    const int64_t kxs = (int64_t)g.ny * (g.nx + 1), kys = (int64_t)(g.ny + 1) * g.nx,
                  kzs = (int64_t)g.ny * g.nx;
    if (KIND == 3) kz_lo = ld(a.kz + (int64_t)(z_lo - 1) * kzs + (int64_t)y * g.nx + x);

    const int64_t bplane = (int64_t)g.nx * g.ny;
    for (int z = z_lo; z < z_hi; ++z, i += pl) {
        double Ap, dinv;
        if (KIND == 2) {
            b_p = box2(i + pl);
            c_p = ld(p + i + pl);
            Ap = 27.0 * c_0 - (b_m + b_0 + b_p);
            b_m = b_0; b_0 = b_p;
            dinv = a.dinv ? ld(a.dinv + i) : a.dinv_c;
        } else if (KIND == 3) {
            c_p = ld(p + i + pl);
            const int zl = z - 1;
            const double kzm = kz_lo;
            const double kym = ld(a.ky + zl * kys + (int64_t)y * g.nx + x);
            const double kxm = ld(a.kx + zl * kxs + (int64_t)y * (g.nx + 1) + x);
            const double kxp = ld(a.kx + zl * kxs + (int64_t)y * (g.nx + 1) + x + 1);
            const double kyp = ld(a.ky + zl * kys + (int64_t)(y + 1) * g.nx + x);
            const double kzp = ld(a.kz + (int64_t)(zl + 1) * kzs + (int64_t)y * g.nx + x);
            kz_lo = kzp;
            const double D = kzm + kym + kxm + kxp + kyp + kzp;
            double nb = kzm * c_m + kzp * c_p;
            if (ym) nb += kym * ld(p + i - pitch);
            if (xm) nb += kxm * ld(p + i - 1);
            if (xp) nb += kxp * ld(p + i + 1);
            if (yp) nb += kyp * ld(p + i + pitch);
            Ap = D * c_0 - nb;
            dinv = a.dinv ? ld(a.dinv + i) : 1.0 / D;
            c_m = c_0;
        } else {
            double nb = 0.0;
            if (KIND == 1) {
                c_p = ld(p + i + pl);
                nb = c_m + c_p;
                c_m = c_0;
            } else {
                c_p = 0.0;   // 2D: no z neighbours
            }
            if (ym) nb += ld(p + i - pitch);
            if (xm) nb += ld(p + i - 1);
            if (xp) nb += ld(p + i + 1);
            if (yp) nb += ld(p + i + pitch);
            Ap = g.center * c_0 - nb;
            dinv = a.dinv ? ld(a.dinv + i) : a.dinv_c;
        }
        if (a.mode == 3) {
            const int64_t bi = (int64_t)(z - 1) * bplane + (int64_t)y * g.nx + x;
            a.w[i] = ld(a.b + bi) - Ap;
        } else {
            a.w[i] = Ap;
            if (a.mode >= 1) {
                const double t = dinv * Ap - a.sigma * c_0;
                double v = a.coef * t;
                if (a.mode == 2) v -= ld(a.pm + i);
                a.pn[i] = v;
            }
        }
        c_0 = c_p;
    }
}

// CSR: one thread per row (single slab; the vector's interior starts one
// "plane" (= n doubles) in, like the stencil layout).
__global__ void __launch_bounds__(256) k1_csr(Geo g, K1Args a, const DevState *st)
{
    if (st && st->done) return;
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= g.n) return;
    const double *p = a.p + g.plane;
    const int64_t i = g.plane + r;
    double Ap = 0.0;
    for (int64_t q = g.rowptr[r]; q < g.rowptr[r + 1]; ++q) Ap += ld(g.val + q) * ld(p + g.colind[q]);
    if (a.mode == 3) {
        a.w[i] = ld(a.b + r) - Ap;
        return;
    }
    a.w[i] = Ap;
    if (a.mode >= 1) {
        const double t = (a.dinv ? ld(a.dinv + i) : a.dinv_c) * Ap - a.sigma * ld(a.p + i);
        double v = a.coef * t;
        if (a.mode == 2) v -= ld(a.pm + i);
        a.pn[i] = v;
    }
}

__global__ void k_pack(Geo g, const double *src, double *dst, int nzl, const DevState *st)
{
    if (st && st->done) return;
    const int64_t nxy = (int64_t)g.nx * g.ny, tot = nxy * nzl;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t zl = e / nxy, rem = e - zl * nxy;
        const int64_t y = rem / g.nx, x = rem - y * g.nx;
        dst[(zl + 1) * g.plane + y * g.pitch + x] = src[e];
    }
}

__global__ void k_unpack(Geo g, const double *src, double *dst, int nzl)
{
    const int64_t nxy = (int64_t)g.nx * g.ny, tot = nxy * nzl;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t zl = e / nxy, rem = e - zl * nxy;
        const int64_t y = rem / g.nx, x = rem - y * g.nx;
        dst[e] = src[(zl + 1) * g.plane + y * g.pitch + x];
    }
}

}  // namespace

void launch_k1(const Geo &g, const K1Args &a, const DevState *st, cudaStream_t s)
{
    if (g.kind == 4) {
        const int64_t blocks = (g.n + 255) / 256;
        k1_csr<<<(unsigned)blocks, 256, 0, s>>>(g, a, st);
        return;
    }
    const int nplanes = a.ze - a.zb;
    if (nplanes <= 0) return;
    // z-chunk: enough CTAs to fill 148 SMs several times, long enough runs
    // that the 2-plane warm-up of the sliding window is amortised.
    const int64_t tiles = (int64_t)((g.nx + BX - 1) / BX) * ((g.ny + BY - 1) / BY);
    int zc = nplanes;
    const int64_t target = 148 * 8;
    while (zc > 16 && tiles * ((nplanes + zc - 1) / zc) < target) zc = (zc + 1) / 2;
    dim3 grid((g.nx + BX - 1) / BX, (g.ny + BY - 1) / BY, (nplanes + zc - 1) / zc);
    dim3 block(BX, BY);
    switch (g.kind) {
    case 0: k1_stencil<0><<<grid, block, 0, s>>>(g, a, st, zc); break;
    case 1: k1_stencil<1><<<grid, block, 0, s>>>(g, a, st, zc); break;
    case 2: k1_stencil<2><<<grid, block, 0, s>>>(g, a, st, zc); break;
    case 3: k1_stencil<3><<<grid, block, 0, s>>>(g, a, st, zc); break;
    }
}

void launch_pack(const Geo &g, const double *src, double *dst, int nzl, const DevState *st,
                 cudaStream_t s)
{
    if (g.kind == 4) {
        cudaMemcpyAsync(dst + g.plane, src, (size_t)g.n * sizeof(double), cudaMemcpyDeviceToDevice, s);
        return;
    }
    const int64_t tot = (int64_t)g.nx * g.ny * nzl;
    const int64_t blocks = std::min<int64_t>((tot + 255) / 256, 148 * 16);
    k_pack<<<(unsigned)blocks, 256, 0, s>>>(g, src, dst, nzl, st);
}

void launch_unpack(const Geo &g, const double *src, double *dst, int nzl, cudaStream_t s)
{
    if (g.kind == 4) {
        cudaMemcpyAsync(dst, src + g.plane, (size_t)g.n * sizeof(double), cudaMemcpyDeviceToDevice, s);
        return;
    }
    const int64_t tot = (int64_t)g.nx * g.ny * nzl;
    const int64_t blocks = std::min<int64_t>((tot + 255) / 256, 148 * 16);
    k_unpack<<<(unsigned)blocks, 256, 0, s>>>(g, src, dst, nzl);
}

}  // namespace sscg
