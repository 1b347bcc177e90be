// K1 -- fused stencil/CSR SpMV + Jacobi + Chebyshev three-term recurrence.
//
// For basis step j (§2 Def. Chebyshev Polynomial Basis):
//   w_j     = A p_j
//   p_{j+1} = coef * (M^{-1} w_j - sigma p_j) [- p_{j-1}]
// with coef = theta at j = 0 and 2 theta (minus p_{j-1}) for j >= 1; at
// j = s-1 only w_j is produced (W = AP feeds the Gram pass).  One launch per
// step streams p_j once from HBM (z-neighbours come from a register sliding
// window, x/y neighbours from L1/L2), p_{j-1}, and writes w_j, p_{j+1}:
// 4 vectors = 32 B per grid point (the K1 roofline unit).
//
// Work decomposition: 32 x 8 column tiles x z-chunks of ZC planes, walked by
// a persistent grid (resident CTAs only, grid-stride over work items, chunk
// major so that neighbouring tiles and the chunk boundary planes are read
// while still in L2).  Each thread prefetches the next plane's p_j and
// p_{j-1} values one iteration ahead (two HBM loads in flight per thread on
// top of the current plane's).
//
// Layout (sscg_internal.cuh Slab/Geo): plane = ny*pitch doubles, one halo
// plane below and above the slab (zero at global Dirichlet boundaries,
// exchanged between slabs).  x/y Dirichlet ghosts are handled by predicates.
#include <algorithm>

#include "sscg_internal.cuh"

namespace sscg {
namespace {

constexpr int BX = 32, BY = 8, CTAS_PER_SM = 8;

__device__ __forceinline__ double ld(const double *p) { return __ldg(p); }

struct K1Work {
    int tiles_x, tiles_y, zc, nchunks, nch1;
    int64_t nitems;
};

template <int KIND>
__global__ void __launch_bounds__(BX *BY, (KIND == 0 || KIND == 1) ? 8 : 5)
    k1_stencil(Geo g, K1Args a, const DevState *st, K1Work wk)
{
    PDL_ENTRY(st);
    const double *__restrict__ p = a.p;
    const double *__restrict__ pm = a.pm;
    double *__restrict__ w = a.w;
    double *__restrict__ pn = a.pn;
    const int64_t pl = g.plane;
    const int pitch = g.pitch;
    const int ntiles = wk.tiles_x * wk.tiles_y;
    const int64_t kxs = (int64_t)g.ny * (g.nx + 1), kys = (int64_t)(g.ny + 1) * g.nx, kzs = (int64_t)g.ny * g.nx;
    const int64_t bplane = (int64_t)g.nx * g.ny;

    for (int64_t item = blockIdx.x; item < wk.nitems; item += gridDim.x) {
        const int chunk = (int)(item / ntiles);
        const int tile = (int)(item - (int64_t)chunk * ntiles);
        const int ty = tile / wk.tiles_x, tx = tile - ty * wk.tiles_x;
        const int x = tx * BX + threadIdx.x;
        const int y = ty * BY + threadIdx.y;
        int z_lo, z_hi;   // chunk -> planes: range 1 [zb, ze), then range 2 [zb2, ze2)
        if (chunk < wk.nch1) {
            z_lo = a.zb + chunk * wk.zc;
            z_hi = min(a.ze, z_lo + wk.zc);
        } else {
            z_lo = a.zb2 + (chunk - wk.nch1) * wk.zc;
            z_hi = min(a.ze2, z_lo + wk.zc);
        }
        if (x >= g.nx || y >= g.ny) continue;
        const bool xm = x > 0, xp = x + 1 < g.nx, ym = y > 0, yp = y + 1 < g.ny;
        int64_t i = (int64_t)z_lo * pl + (int64_t)y * pitch + x;

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

        double c_m = 0.0, c_0, c_p, b_m = 0.0, b_0 = 0.0, b_p = 0.0, kz_lo = 0.0;
        c_0 = ld(p + i);
        if (KIND == 2) {
            b_m = box2(i - pl);
            b_0 = box2(i);
            b_p = box2(i + pl);
            c_p = ld(p + i + pl);
        } else if (KIND == 0) {
            c_p = 0.0;
        } else {
            c_m = ld(p + i - pl);
            c_p = ld(p + i + pl);
        }
        if (KIND == 3) kz_lo = ld(a.kz + (int64_t)(z_lo - 1) * kzs + (int64_t)y * g.nx + x);
        double pm0 = (a.mode == 2) ? __ldcs(pm + i) : 0.0;

        for (int z = z_lo; z < z_hi; ++z, i += pl) {
            // prefetch the next plane (one iteration ahead)
            const bool more = z + 1 < z_hi;
            double c_pp = 0.0, b_pp = 0.0, pm1 = 0.0;
            if (more) {
                if (KIND == 2) b_pp = box2(i + 2 * pl);
                if (KIND == 1 || KIND == 3 || KIND == 2) c_pp = ld(p + i + 2 * pl);
                if (a.mode == 2) pm1 = __ldcs(pm + i + pl);
            }
            double Ap, dinv;
            if (KIND == 2) {
                Ap = 27.0 * c_0 - (b_m + b_0 + b_p);
                dinv = a.dinv ? ld(a.dinv + i) : a.dinv_c;
            } else if (KIND == 3) {
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
            } else {
                double nb = (KIND == 1) ? c_m + c_p : 0.0;
                if (ym) nb += ld(p + i - pitch);
                if (xm) nb += ld(p + i - 1);
                if (xp) nb += ld(p + i + 1);
                if (yp) nb += ld(p + i + pitch);
                Ap = g.center * c_0 - nb;
                dinv = a.dinv ? ld(a.dinv + i) : a.dinv_c;
            }
            if (a.mode == 3) {
                const int64_t bi = (int64_t)(z - 1) * bplane + (int64_t)y * g.nx + x;
                w[i] = ld(a.b + bi) - Ap;
            } else {
                __stcs(w + i, Ap);
                if (a.mode >= 1) {
                    const double t = dinv * Ap - a.sigma * c_0;
                    double v = a.coef * t;
                    if (a.mode == 2) v -= pm0;
                    pn[i] = v;
                }
            }
            c_m = c_0;
            c_0 = c_p;
            c_p = c_pp;
            b_m = b_0;
            b_0 = b_p;
            b_p = b_pp;
            pm0 = pm1;
        }
    }
}

// 5-/7-point path, two x-points per thread (16-B loads/stores), x-neighbours
// by warp shuffles, and a two-plane-deep register prefetch of p_j and p_{j-1}
// so that each warp keeps ~2 KB of HBM reads in flight.  Tile = 64 x 8.
__device__ __forceinline__ double2 ld2(const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); }
__device__ __forceinline__ double2 ld2cs(const double *p) { return __ldcs(reinterpret_cast<const double2 *>(p)); }

template <int KIND>
__global__ void __launch_bounds__(BX *BY, 4) k1_lap_vec(Geo g, K1Args a, const DevState *st, K1Work wk)
{
    PDL_ENTRY(st);
    const double *__restrict__ p = a.p;
    const double *__restrict__ pm = a.pm;
    double *__restrict__ w = a.w;
    double *__restrict__ pn = a.pn;
    const int64_t pl = g.plane;
    const int pitch = g.pitch;
    const int ntiles = wk.tiles_x * wk.tiles_y;
    const int lane = threadIdx.x;
    const int64_t bplane = (int64_t)g.nx * g.ny;
    const double2 Z = make_double2(0.0, 0.0);

    for (int64_t item = blockIdx.x; item < wk.nitems; item += gridDim.x) {
        const int chunk = (int)(item / ntiles);
        const int tile = (int)(item - (int64_t)chunk * ntiles);
        const int ty = tile / wk.tiles_x, tx = tile - ty * wk.tiles_x;
        const int x = (tx * BX + lane) * 2;          // first of the pair
        const int y = ty * BY + threadIdx.y;
        int z_lo, z_hi;   // chunk -> planes: range 1 [zb, ze), then range 2 [zb2, ze2)
        if (chunk < wk.nch1) {
            z_lo = a.zb + chunk * wk.zc;
            z_hi = min(a.ze, z_lo + wk.zc);
        } else {
            z_lo = a.zb2 + (chunk - wk.nch1) * wk.zc;
            z_hi = min(a.ze2, z_lo + wk.zc);
        }
        if (y >= g.ny) continue;                      // whole warp (same y)
        const bool in = x < g.nx;                     // pair starts inside the row
        const bool in1 = x + 1 < g.nx;                // second point inside
        const bool ym = y > 0, yp = y + 1 < g.ny;
        int64_t i = (int64_t)z_lo * pl + (int64_t)y * pitch + x;
        const bool m2 = a.mode == 2;

        // sliding window: p at z-1, z, z+1, z+2; p_{j-1} at z, z+1
        double2 c_m = Z, c_0 = Z, c_p = Z, c_pp = Z, q_0 = Z, q_1 = Z;
        if (in) {
            c_0 = ld2(p + i);
            if (KIND == 1) {
                c_m = ld2(p + i - pl);
                c_p = ld2(p + i + pl);
                if (z_lo + 1 < z_hi) c_pp = ld2(p + i + 2 * pl);
            }
            if (m2) {
                q_0 = ld2cs(pm + i);
                if (z_lo + 1 < z_hi) q_1 = ld2cs(pm + i + pl);
            }
        }
        for (int z = z_lo; z < z_hi; ++z, i += pl) {
            double2 c_ppp = Z, q_2 = Z;
            if (in && z + 2 < z_hi) {
                if (KIND == 1) c_ppp = ld2(p + i + 3 * pl);
                if (m2) q_2 = ld2cs(pm + i + 2 * pl);
            }
            double2 yl = Z, yh = Z;
            if (in) {
                if (ym) yl = ld2(p + i - pitch);
                if (yp) yh = ld2(p + i + pitch);
            }
            // x-neighbours: left of the pair = previous lane's .y, right = next lane's .x
            double xl = __shfl_up_sync(0xffffffffu, c_0.y, 1);
            double xr = __shfl_down_sync(0xffffffffu, c_0.x, 1);
            if (lane == 0) xl = (in && x > 0) ? __ldg(p + i - 1) : 0.0;
            if (lane == 31) xr = (in && x + 2 < g.nx) ? __ldg(p + i + 2) : 0.0;
            if (x + 2 >= g.nx) xr = 0.0;   // right Dirichlet ghost (pad column is 0 too)
            double nb0 = yl.x + yh.x + xl + c_0.y;
            double nb1 = yl.y + yh.y + c_0.x + xr;
            if (KIND == 1) {
                nb0 += c_m.x + c_p.x;
                nb1 += c_m.y + c_p.y;
            }
            const double Ap0 = g.center * c_0.x - nb0;
            const double Ap1 = in1 ? g.center * c_0.y - nb1 : 0.0;
            if (in) {
                if (a.mode == 3) {
                    const int64_t bi = (int64_t)(z - 1) * bplane + (int64_t)y * g.nx + x;
                    w[i] = __ldg(a.b + bi) - Ap0;
                    if (in1) w[i + 1] = __ldg(a.b + bi + 1) - Ap1;
                } else {
                    __stcs(reinterpret_cast<double2 *>(w + i), make_double2(Ap0, Ap1));
                    if (a.mode >= 1) {
                        double2 dv;
                        if (a.dinv) dv = ld2(a.dinv + i);
                        else dv = make_double2(a.dinv_c, a.dinv_c);
                        double v0 = a.coef * (dv.x * Ap0 - a.sigma * c_0.x);
                        double v1 = a.coef * (dv.y * Ap1 - a.sigma * c_0.y);
                        if (m2) {
                            v0 -= q_0.x;
                            v1 -= q_0.y;
                        }
                        if (!in1) v1 = 0.0;
                        *reinterpret_cast<double2 *>(pn + i) = make_double2(v0, v1);
                    }
                }
            }
            c_m = c_0;
            c_0 = c_p;
            c_p = c_pp;
            c_pp = c_ppp;
            q_0 = q_1;
            q_1 = q_2;
        }
    }
}

// CSR: one thread per row (single slab; the vector's interior starts one
// "plane" (= n doubles) in, like the stencil layout).
__global__ void __launch_bounds__(256) k1_csr(Geo g, K1Args a, const DevState *st)
{
    PDL_ENTRY(st);
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
    if (!a.skip_w) a.w[i] = Ap;
    if (a.mode >= 1) {
        const double t = (a.dinv ? ld(a.dinv + i) : a.dinv_c) * Ap - a.sigma * ld(a.p + i);
        double v = a.coef * t;
        if (a.mode == 2) v -= ld(a.pm + i);
        a.pn[i] = v;
    }
}

__global__ void k_pack(Geo g, const double *src, double *dst, int nzl, const DevState *st)
{
    PDL_ENTRY(st);
    const int64_t nxy = (int64_t)g.nx * g.ny, tot = nxy * nzl;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t zl = e / nxy, rem = e - zl * nxy;
        const int64_t y = rem / g.nx, x = rem - y * g.nx;
        dst[(zl + 1) * g.plane + y * g.pitch + x] = src[e];
    }
}

__global__ void k_unpack(Geo g, const double *src, double *dst, int nzl)
{
    const int64_t nxy = (int64_t)g.nx * g.ny, tot = nxy * nzl;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
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
        launch_pdl(g.kn.pdl, k1_csr, dim3((unsigned)blocks), dim3(256), 0, s, g, a, st);
        return;
    }
    if (k1t_supported(g, a)) {
        launch_k1t(g, a, st, s);
        return;
    }
    const int n1 = std::max(0, a.ze - a.zb), n2 = std::max(0, a.ze2 - a.zb2);
    const int nplanes = n1 + n2;
    if (nplanes <= 0) return;
    K1Work wk;
    const bool vec = g.kind <= 1;            // 5-/7-point: two points per thread
    wk.tiles_x = (g.nx + (vec ? 2 * BX : BX) - 1) / (vec ? 2 * BX : BX);
    wk.tiles_y = (g.ny + BY - 1) / BY;
    const int64_t tiles = (int64_t)wk.tiles_x * wk.tiles_y;
    static int occ[4] = {0, 0, 0, 0};
    if (!occ[g.kind]) {
        const void *fn = g.kind == 0 ? (const void *)k1_lap_vec<0>
                       : g.kind == 1 ? (const void *)k1_lap_vec<1>
                       : g.kind == 2 ? (const void *)k1_stencil<2> : (const void *)k1_stencil<3>;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[g.kind], fn, BX * BY, 0) != cudaSuccess ||
            occ[g.kind] <= 0)
            occ[g.kind] = CTAS_PER_SM;
    }
    const int sms = (a.sm_cap > 0 && a.sm_cap < k2_grid()) ? a.sm_cap : k2_grid();
    const int64_t resident = (int64_t)sms * occ[g.kind];
    // z-chunks of 16 planes by default (2-plane warm-up amortised); shorter
    // when that leaves fewer than 4 work items per resident CTA
    int zc = std::min(std::max(n1, n2), 16);
    while (zc > 2 && tiles * ((nplanes + zc - 1) / zc) < 4 * resident) zc = (zc + 1) / 2;
    wk.zc = zc;
    wk.nch1 = (n1 + zc - 1) / zc;
    wk.nchunks = wk.nch1 + (n2 + zc - 1) / zc;
    wk.nitems = tiles * wk.nchunks;
    const unsigned grid = (unsigned)std::min<int64_t>(wk.nitems, resident);
    dim3 block(BX, BY);
    switch (g.kind) {
    case 0: launch_pdl(g.kn.pdl, k1_lap_vec<0>, dim3(grid), dim3(block), 0, s, g, a, st, wk); break;
    case 1: launch_pdl(g.kn.pdl, k1_lap_vec<1>, dim3(grid), dim3(block), 0, s, g, a, st, wk); break;
    case 2: launch_pdl(g.kn.pdl, k1_stencil<2>, dim3(grid), dim3(block), 0, s, g, a, st, wk); break;
    case 3: launch_pdl(g.kn.pdl, k1_stencil<3>, dim3(grid), dim3(block), 0, s, g, a, st, wk); break;
    }
}

void launch_pack(const Geo &g, const double *src, double *dst, int nzl, const DevState *st, cudaStream_t s)
{
    if (g.kind == 4) {
        cudaMemcpyAsync(dst + g.plane, src, (size_t)g.n * sizeof(double), cudaMemcpyDeviceToDevice, s);
        return;
    }
    const int64_t tot = (int64_t)g.nx * g.ny * nzl;
    const int64_t blocks = std::min<int64_t>((tot + 255) / 256, 148 * 16);
    launch_pdl(g.kn.pdl, k_pack, dim3((unsigned)blocks), dim3(256), 0, s, g, src, dst, nzl, st);
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
