// K1T -- TMA-staged basis step for the 3D stencils (7-point, 27-point,
// variable-coefficient 7-point): the same operation as K1 (§2 Def.
// Chebyshev Polynomial Basis)
//   w_j     = A p_j
//   p_{j+1} = coef * (M^{-1} w_j - sigma p_j) [- p_{j-1}]
// with the planes of p_j and p_{j-1} brought into shared memory by the
// tensor-memory accelerator instead of per-thread loads.
//
// Work: tiles of TX x TY points in (x, y) times z-chunks of ZC planes,
// chunk-major (all tiles of one chunk run at the same time, so the x/y halo
// cells and the chunk-boundary planes that neighbouring tiles also read are
// L2 hits), walked by a persistent grid.
//
// Per CTA: warp 0 is the producer -- one lane issues, per plane z, a 4-D
// `cp.async.bulk.tensor` box of p_j covering the tile plus a 2-cell x halo
// and a 1-row y halo (global-boundary cells come back zero: the TMA unit's
// out-of-bounds fill is the Dirichlet ghost), and a box of p_{j-1} covering
// the tile, into two rings of NSP / NSM slots guarded by full/empty
// mbarriers.  It runs up to NSP-2 planes ahead of the consumers, across item
// boundaries, so every SM keeps ~100 KB of HBM reads in flight without
// spending registers on it.  Warps 1..8 are consumers: warp w owns tile rows
// 2w and 2w+1, lane l the x pair (2l, 2l+1); the z-neighbours (7-point) or
// the 3x3 in-plane box sums (27-point, A p = 27 p - box3x3x3(p)) slide
// through registers, the x/y neighbours are read from the staged plane.
// w_j and p_{j+1} are written with 16-byte stores straight from registers.
//
// Bytes per launch: p_j, p_{j-1} read, w_j, p_{j+1} written (4 vectors at
// 1 <= j < s-1).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "sscg_internal.cuh"
#include "tma.cuh"

namespace sscg {
namespace {

constexpr int TX = 64, TY = 16;
constexpr int BW = TX + 4, BH = TY + 2;                       // p box: x in [x0-2, x0+TX+2), y in [y0-1, y0+TY+1)
constexpr int PSLOT = ((BW * BH * 8 + 127) / 128) * 128 / 8;  // doubles per p slot (128-B aligned)
constexpr int MSLOT = TX * TY;                                // doubles per p_{j-1} slot
#ifndef K1T_NSP
#define K1T_NSP 6
#endif
constexpr int NSP = K1T_NSP, NSM = 4;
constexpr int NCW = TY / 2;                                   // consumer warps (2 rows each)
constexpr int THREADS = 32 * (NCW + 1);
constexpr uint32_t PBYTES = BW * BH * 8, MBYTES = TX * TY * 8;
constexpr size_t SMEM = (size_t)(NSP * PSLOT + NSM * MSLOT) * sizeof(double);
// KIND 4 (variable coefficients, faces staged by TMA): per plane slot
//   KX: TY rows x 68 faces (row pitch 80 doubles: 128-B aligned TMA rows;
//       row r starts at face x0 - parity(r), see k1t_prepare_faces)
//   KY: TY+1 rows x TX,  KZL / KZH: TY rows x TX (lower / upper z-faces)
constexpr int KXB = 68, KXP = 80, FKX = 0, FKY = TY * KXP, FKZL = FKY + (TY + 1) * TX, FKZH = FKZL + TY * TX;
constexpr int FSLOT = FKZH + TY * TX;     // doubles (34,304 B)
constexpr int NSF = 3;
constexpr uint32_t FBYTES = (TY * KXB + (TY + 1) * TX + 2 * TY * TX) * 8;
constexpr size_t SMEM4 = SMEM + (size_t)NSF * FSLOT * sizeof(double);
static_assert((FKY * 8) % 128 == 0 && (FKZL * 8) % 128 == 0 && (FKZH * 8) % 128 == 0 && (FSLOT * 8) % 128 == 0,
              "TMA destinations must be 128-B aligned");

__device__ __forceinline__ void tma_load_1d(void *dst, const CUtensorMap *map, int x, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_3d_(void *dst, const CUtensorMap *map, int x, int y, int z, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

struct K1TWork {
    int tiles_x, tiles_y, zc, nch1;
    int64_t nitems;
    int zb, ze, zb2, ze2;
    int j;
};

__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, int x, int y, int z, int v,
                                            uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(v), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ double2 lds2(const double *p) { return *reinterpret_cast<const double2 *>(p); }

__device__ __forceinline__ void item_planes(const K1TWork &wk, int64_t item, int ntiles, int &tx, int &ty, int &zlo,
                                            int &zhi)
{
    const int chunk = (int)(item / ntiles);
    const int tile = (int)(item - (int64_t)chunk * ntiles);
    ty = tile / wk.tiles_x;
    tx = tile - ty * wk.tiles_x;
    if (chunk < wk.nch1) {
        zlo = wk.zb + chunk * wk.zc;
        zhi = min(wk.ze, zlo + wk.zc);
    } else {
        zlo = wk.zb2 + (chunk - wk.nch1) * wk.zc;
        zhi = min(wk.ze2, zlo + wk.zc);
    }
}

// 3-point row sums of the pair (x, x+1) from a staged row: (l + c.x + c.y, c.x + c.y + r)
__device__ __forceinline__ double2 rowsum3(const double *row)
{
    const double l = row[-1], r = row[2];
    const double2 c = lds2(row);
    return make_double2(l + c.x + c.y, c.x + c.y + r);
}

template <int KIND>
__global__ void __launch_bounds__(THREADS, KIND >= 3 ? 1 : 2)
    k1t(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmM,
        const __grid_constant__ CUtensorMap tmKX, const __grid_constant__ CUtensorMap tmKY,
        const __grid_constant__ CUtensorMap tmKZ, Geo g, K1Args a, const DevState *st, K1TWork wk)
{
    PDL_ENTRY(st);
    extern __shared__ __align__(128) double smem[];
    double *sp = smem;
    double *sq = smem + NSP * PSLOT;
    double *sf = sq + NSM * MSLOT;   // KIND 4 face ring
    __shared__ uint64_t fullp[NSP], emptyp[NSP], fullm[NSM], emptym[NSM], fullf[NSF], emptyf[NSF];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool m2 = a.mode == 2;
    const int ntiles = wk.tiles_x * wk.tiles_y;

    if (tid == 0) {
        for (int i = 0; i < NSP; ++i) {
            mbar_init(&fullp[i], 1);
            mbar_init(&emptyp[i], NCW);
        }
        for (int i = 0; i < NSM; ++i) {
            mbar_init(&fullm[i], 1);
            mbar_init(&emptym[i], NCW);
        }
        for (int i = 0; i < NSF; ++i) {
            mbar_init(&fullf[i], 1);
            mbar_init(&emptyf[i], NCW);
        }
        mbar_fence_init();
        tma_prefetch_desc(&tmP);
        tma_prefetch_desc(&tmM);
        if (KIND == 4) {
            tma_prefetch_desc(&tmKX);
            tma_prefetch_desc(&tmKY);
            tma_prefetch_desc(&tmKZ);
        }
    }
    __syncthreads();

    if (warp == 0) {
        // ---------------- producer ----------------
        // lane 0 issues the p_j / p_{j-1} boxes; for KIND 4 the whole warp runs
        // the loop and lanes 0..TY-1 issue one kx row box each
        if (lane == 0 || KIND == 4) {
            uint32_t pc = 0, mc = 0, fc = 0;
            for (int64_t item = blockIdx.x; item < wk.nitems; item += gridDim.x) {
                int tx, ty, zlo, zhi;
                item_planes(wk, item, ntiles, tx, ty, zlo, zhi);
                const int x0 = tx * TX, y0 = ty * TY;
                auto loadp = [&](int z) {
                    const int sl = pc % NSP;
                    if (lane == 0) {
                        if (pc >= NSP) mbar_wait(&emptyp[sl], ((pc / NSP) - 1) & 1);
                        mbar_expect_tx(&fullp[sl], PBYTES);
                        tma_load_4d(sp + sl * PSLOT, &tmP, x0 - 2, y0 - 1, z, wk.j, &fullp[sl]);
                    }
                    ++pc;
                };
                auto loadm = [&](int z) {
                    const int sl = mc % NSM;
                    if (lane == 0) {
                        if (mc >= NSM) mbar_wait(&emptym[sl], ((mc / NSM) - 1) & 1);
                        mbar_expect_tx(&fullm[sl], MBYTES);
                        tma_load_4d(sq + sl * MSLOT, &tmM, x0, y0, z, wk.j - 1, &fullm[sl]);
                    }
                    ++mc;
                };
                auto loadf = [&](int z) {   // faces of plane z (slab-local zl = z - 1)
                    const int sl = fc % NSF;
                    double *d = sf + sl * FSLOT;
                    const int zl = z - 1;
                    if (lane == 0) {
                        if (fc >= NSF) mbar_wait(&emptyf[sl], ((fc / NSF) - 1) & 1);
                        mbar_expect_tx(&fullf[sl], FBYTES);
                    }
                    __syncwarp();
                    if (lane < TY) {   // face row (zl, y0 + lane), from the even element at or below its x0
                        const int e0 = (zl * g.ny + y0 + lane) * (g.nx + 1) + x0;
                        tma_load_1d(d + FKX + lane * KXP, &tmKX, e0 & ~1, &fullf[sl]);
                    }
                    if (lane == 0) {
                        tma_load_3d_(d + FKY, &tmKY, x0, y0, zl, &fullf[sl]);
                        tma_load_3d_(d + FKZL, &tmKZ, x0, y0, zl, &fullf[sl]);
                        tma_load_3d_(d + FKZH, &tmKZ, x0, y0, zl + 1, &fullf[sl]);
                    }
                    ++fc;
                };
                loadp(zlo - 1);
                loadp(zlo);
                for (int z = zlo; z < zhi; ++z) {
                    loadp(z + 1);
                    if (m2) loadm(z);
                    if (KIND == 4) loadf(z);
                }
            }
        }
        return;   // no CTA-wide barrier follows
    }

    // ---------------- consumers ----------------
    const int cw = warp - 1;
    double pacc = 0.0;   // dot mode (a.dot_entry): this thread's part of p^T A p
    const int ra = 2 * cw;                          // tile rows ra, ra + 1
    const int oa = (ra + 1) * BW + 2 + 2 * lane;    // pair of row ra in a p slot
    const int ob = oa + BW;
    const int qa = ra * TX + 2 * lane, qb = qa + TX;
    const int64_t pl = g.plane;
    uint32_t pc = 0, mc = 0, fc = 0;
    auto waitp = [&](uint32_t c) -> const double * {
        const int sl = c % NSP;
        mbar_wait(&fullp[sl], (c / NSP) & 1);
        return sp + sl * PSLOT;
    };
    auto relp = [&](uint32_t c) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyp[c % NSP]);
    };

    for (int64_t item = blockIdx.x; item < wk.nitems; item += gridDim.x) {
        int tx, ty, zlo, zhi;
        item_planes(wk, item, ntiles, tx, ty, zlo, zhi);
        const int x = tx * TX + 2 * lane;
        const int ya = ty * TY + ra, yb = ya + 1;
        const bool inx = x < g.nx, in1 = x + 1 < g.nx;
        const bool sa = inx && ya < g.ny, sb = inx && yb < g.ny;
        int64_t ia = (int64_t)zlo * pl + (int64_t)ya * g.pitch + x;

        double2 cma, cmb, c0a, c0b, bma = {}, bmb = {}, b0a = {}, b0b = {};
        // KIND 3: faces of this slab (R12), read straight from global memory
        // (L1-cached; rows of kx have odd length, no TMA view); lower z-faces
        // slide through registers
        const int64_t kxs = (int64_t)g.ny * (g.nx + 1), kys = (int64_t)(g.ny + 1) * g.nx,
                      kzs = (int64_t)g.ny * g.nx;
        double kzma0 = 0.0, kzma1 = 0.0, kzmb0 = 0.0, kzmb1 = 0.0;
        if (KIND == 3) {
            const double *q = a.kz + (int64_t)(zlo - 1) * kzs + (int64_t)ya * g.nx + x;
            if (sa) { kzma0 = __ldg(q); if (in1) kzma1 = __ldg(q + 1); }
            if (sb) { kzmb0 = __ldg(q + g.nx); if (in1) kzmb1 = __ldg(q + g.nx + 1); }
        }
        uint32_t c0;
        {
            const double *s = waitp(pc);
            if (KIND == 2) {
                const double2 r0 = rowsum3(s + oa - BW), r1 = rowsum3(s + oa), r2 = rowsum3(s + ob),
                              r3 = rowsum3(s + ob + BW);
                bma = make_double2(r0.x + r1.x + r2.x, r0.y + r1.y + r2.y);
                bmb = make_double2(r1.x + r2.x + r3.x, r1.y + r2.y + r3.y);
            }
            cma = lds2(s + oa);
            cmb = lds2(s + ob);
            relp(pc);
            ++pc;
            s = waitp(pc);
            c0a = lds2(s + oa);
            c0b = lds2(s + ob);
            if (KIND == 2) {
                const double2 r0 = rowsum3(s + oa - BW), r1 = rowsum3(s + oa), r2 = rowsum3(s + ob),
                              r3 = rowsum3(s + ob + BW);
                b0a = make_double2(r0.x + r1.x + r2.x, r0.y + r1.y + r2.y);
                b0b = make_double2(r1.x + r2.x + r3.x, r1.y + r2.y + r3.y);
                relp(pc);
            }
            c0 = pc;
            ++pc;
        }
        for (int z = zlo; z < zhi; ++z, ia += pl) {
            // KIND 3: issue this plane's face loads before waiting on the ring
            double kxa0 = 0, kxa1 = 0, kxa2 = 0, kxb0 = 0, kxb1 = 0, kxb2 = 0;
            double kya0 = 0, kya1 = 0, kyb0 = 0, kyb1 = 0, kyc0 = 0, kyc1 = 0;
            double kzpa0 = 0, kzpa1 = 0, kzpb0 = 0, kzpb1 = 0;
            if (KIND == 3) {
                const int zl = z - 1;
                const double *qx = a.kx + zl * kxs + (int64_t)ya * (g.nx + 1) + x;
                const double *qy = a.ky + zl * kys + (int64_t)ya * g.nx + x;
                const double *qz = a.kz + (int64_t)(zl + 1) * kzs + (int64_t)ya * g.nx + x;
                if (sa) {
                    kxa0 = __ldg(qx); kxa1 = __ldg(qx + 1);
                    kya0 = __ldg(qy); kyb0 = __ldg(qy + g.nx);
                    kzpa0 = __ldg(qz);
                    if (in1) { kxa2 = __ldg(qx + 2); kya1 = __ldg(qy + 1); kyb1 = __ldg(qy + g.nx + 1); kzpa1 = __ldg(qz + 1); }
                }
                if (sb) {
                    kxb0 = __ldg(qx + g.nx + 1); kxb1 = __ldg(qx + g.nx + 2);
                    kyc0 = __ldg(qy + 2 * g.nx);
                    kzpb0 = __ldg(qz + g.nx);
                    if (in1) { kxb2 = __ldg(qx + g.nx + 3); kyc1 = __ldg(qy + 2 * g.nx + 1); kzpb1 = __ldg(qz + g.nx + 1); }
                }
            }
            if (KIND == 4) {   // faces of plane z from the staged slot
                const int sl = fc % NSF;
                mbar_wait(&fullf[sl], (fc / NSF) & 1);
                const double *F = sf + sl * FSLOT;
                const int xa = 2 * lane;
                const int fa = ((z - 1) * g.ny + ya) * (g.nx + 1) + tx * TX;   // first face of row ya (parity)
                const double *fx = F + FKX + ra * KXP + xa + (fa & 1), *fy = F + FKY + ra * TX + xa;
                const double *fxb = F + FKX + (ra + 1) * KXP + xa + ((fa + g.nx + 1) & 1);
                kxa0 = fx[0]; kxa1 = fx[1]; kxa2 = fx[2];
                kxb0 = fxb[0]; kxb1 = fxb[1]; kxb2 = fxb[2];
                const double2 ya0 = lds2(fy), yb0 = lds2(fy + TX), yc0 = lds2(fy + 2 * TX);
                kya0 = ya0.x; kya1 = ya0.y; kyb0 = yb0.x; kyb1 = yb0.y; kyc0 = yc0.x; kyc1 = yc0.y;
                const double2 zla = lds2(F + FKZL + ra * TX + xa), zlb = lds2(F + FKZL + (ra + 1) * TX + xa);
                const double2 zha = lds2(F + FKZH + ra * TX + xa), zhb = lds2(F + FKZH + (ra + 1) * TX + xa);
                kzma0 = zla.x; kzma1 = zla.y; kzmb0 = zlb.x; kzmb1 = zlb.y;
                kzpa0 = zha.x; kzpa1 = zha.y; kzpb0 = zhb.x; kzpb1 = zhb.y;
                __syncwarp();
                if (lane == 0) mbar_arrive(&emptyf[sl]);
                ++fc;
            }
            const double *s0 = sp + (c0 % NSP) * PSLOT;   // plane z (7-point: still held)
            const double *s1 = waitp(pc);                  // plane z+1
            double2 Apa, Apb;
            double2 Da = {}, Db = {};
            const double2 cpa = lds2(s1 + oa), cpb = lds2(s1 + ob);
            if (KIND == 2) {
                const double2 r0 = rowsum3(s1 + oa - BW), r1 = rowsum3(s1 + oa), r2 = rowsum3(s1 + ob),
                              r3 = rowsum3(s1 + ob + BW);
                const double2 bpa = make_double2(r0.x + r1.x + r2.x, r0.y + r1.y + r2.y);
                const double2 bpb = make_double2(r1.x + r2.x + r3.x, r1.y + r2.y + r3.y);
                relp(pc);
                Apa.x = 27.0 * c0a.x - (bma.x + b0a.x + bpa.x);
                Apa.y = 27.0 * c0a.y - (bma.y + b0a.y + bpa.y);
                Apb.x = 27.0 * c0b.x - (bmb.x + b0b.x + bpb.x);
                Apb.y = 27.0 * c0b.y - (bmb.y + b0b.y + bpb.y);
                bma = b0a; bmb = b0b;
                b0a = bpa; b0b = bpb;
            } else if (KIND == 3 || KIND == 4) {
                const double2 ylo = lds2(s0 + oa - BW), yhi = lds2(s0 + ob + BW);
                const double la = s0[oa - 1], rra = s0[oa + 2], lb = s0[ob - 1], rrb = s0[ob + 2];
                relp(c0);
                // A_ii = sum of the six faces, A_i,nbr = -k_face (R12); order as K1
                Da.x = kzma0 + kya0 + kxa0 + kxa1 + kyb0 + kzpa0;
                Da.y = kzma1 + kya1 + kxa1 + kxa2 + kyb1 + kzpa1;
                Db.x = kzmb0 + kyb0 + kxb0 + kxb1 + kyc0 + kzpb0;
                Db.y = kzmb1 + kyb1 + kxb1 + kxb2 + kyc1 + kzpb1;
                Apa.x = Da.x * c0a.x - (kzma0 * cma.x + kzpa0 * cpa.x + kya0 * ylo.x + kxa0 * la + kxa1 * c0a.y + kyb0 * c0b.x);
                Apa.y = Da.y * c0a.y - (kzma1 * cma.y + kzpa1 * cpa.y + kya1 * ylo.y + kxa1 * c0a.x + kxa2 * rra + kyb1 * c0b.y);
                Apb.x = Db.x * c0b.x - (kzmb0 * cmb.x + kzpb0 * cpb.x + kyb0 * c0a.x + kxb0 * lb + kxb1 * c0b.y + kyc0 * yhi.x);
                Apb.y = Db.y * c0b.y - (kzmb1 * cmb.y + kzpb1 * cpb.y + kyb1 * c0a.y + kxb1 * c0b.x + kxb2 * rrb + kyc1 * yhi.y);
                kzma0 = kzpa0; kzma1 = kzpa1; kzmb0 = kzpb0; kzmb1 = kzpb1;
            } else {
                const double2 ylo = lds2(s0 + oa - BW), yhi = lds2(s0 + ob + BW);
                const double la = s0[oa - 1], rra = s0[oa + 2], lb = s0[ob - 1], rrb = s0[ob + 2];
                relp(c0);
                // centre first, then neighbours in (dz, dy, dx) order
                Apa.x = g.center * c0a.x - (cma.x + ylo.x + la + c0a.y + c0b.x + cpa.x);
                Apa.y = g.center * c0a.y - (cma.y + ylo.y + c0a.x + rra + c0b.y + cpa.y);
                Apb.x = g.center * c0b.x - (cmb.x + c0a.x + lb + c0b.y + yhi.x + cpb.x);
                Apb.y = g.center * c0b.y - (cmb.y + c0a.y + c0b.x + rrb + yhi.y + cpb.y);
            }
            if (!in1) {
                Apa.y = 0.0;
                Apb.y = 0.0;
            }
            double2 qa2 = {}, qb2 = {};
            if (m2) {
                const int sl = mc % NSM;
                mbar_wait(&fullm[sl], (mc / NSM) & 1);
                qa2 = lds2(sq + sl * MSLOT + qa);
                qb2 = lds2(sq + sl * MSLOT + qb);
                __syncwarp();
                if (lane == 0) mbar_arrive(&emptym[sl]);
                ++mc;
            }
            if (a.dot_entry) {   // p^T A p (the fold's Ghat_{s-1,s-1}): own cells only
                if (sa) {
                    pacc = fma(c0a.x, Apa.x, pacc);
                    pacc = fma(c0a.y, Apa.y, pacc);
                }
                if (sb) {
                    pacc = fma(c0b.x, Apb.x, pacc);
                    pacc = fma(c0b.y, Apb.y, pacc);
                }
            }
            if (sa) {
                if (!a.skip_w) __stcs(reinterpret_cast<double2 *>(a.w + ia), Apa);
                if (a.mode >= 1) {
                    const double2 dv = a.dinv ? __ldg(reinterpret_cast<const double2 *>(a.dinv + ia))
                                       : (KIND >= 3) ? make_double2(1.0 / Da.x, in1 ? 1.0 / Da.y : 0.0)
                                                     : make_double2(a.dinv_c, a.dinv_c);
                    double v0 = a.coef * (dv.x * Apa.x - a.sigma * c0a.x);
                    double v1 = a.coef * (dv.y * Apa.y - a.sigma * c0a.y);
                    if (m2) {
                        v0 -= qa2.x;
                        v1 -= qa2.y;
                    }
                    if (!in1) v1 = 0.0;
                    *reinterpret_cast<double2 *>(a.pn + ia) = make_double2(v0, v1);
                }
            }
            if (sb) {
                const int64_t ib = ia + g.pitch;
                if (!a.skip_w) __stcs(reinterpret_cast<double2 *>(a.w + ib), Apb);
                if (a.mode >= 1) {
                    const double2 dv = a.dinv ? __ldg(reinterpret_cast<const double2 *>(a.dinv + ib))
                                       : (KIND >= 3) ? make_double2(1.0 / Db.x, in1 ? 1.0 / Db.y : 0.0)
                                                     : make_double2(a.dinv_c, a.dinv_c);
                    double v0 = a.coef * (dv.x * Apb.x - a.sigma * c0b.x);
                    double v1 = a.coef * (dv.y * Apb.y - a.sigma * c0b.y);
                    if (m2) {
                        v0 -= qb2.x;
                        v1 -= qb2.y;
                    }
                    if (!in1) v1 = 0.0;
                    *reinterpret_cast<double2 *>(a.pn + ib) = make_double2(v0, v1);
                }
            }
            cma = c0a; cmb = c0b;
            c0a = cpa; c0b = cpb;
            c0 = pc;
            ++pc;
        }
        if (KIND != 2) relp(c0);   // the last plane (z_hi) was only read for its centres
    }
    if (a.dot_entry) {
        // fixed-order block sum of the consumer warps (named barrier: the
        // producer warp has returned), per-CTA partial, the last CTA sums the
        // partials in index order (lane-strided, then a fixed xor tree)
        __shared__ double dred[NCW];
        __shared__ bool dlast;
        for (int o = 16; o > 0; o >>= 1) pacc += __shfl_xor_sync(0xffffffffu, pacc, o);
        if (lane == 0) dred[cw] = pacc;
        asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");
        if (cw == 0 && lane == 0) {
            double v = 0.0;
            for (int w = 0; w < NCW; ++w) v += dred[w];
            a.dot_part[blockIdx.x] = v;
            __threadfence();
            dlast = atomicAdd(a.dot_ticket, 1u) == gridDim.x - 1;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");
        if (dlast && cw == 0) {
            __threadfence();
            double v = 0.0;
            for (int b = lane; b < (int)gridDim.x; b += 32) v += __ldcg(a.dot_part + b);
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) {
                *a.dot_entry = v;
                *a.dot_ticket = 0u;
            }
        }
    }
}

}  // namespace

bool k1t_supported(const Geo &g, const K1Args &a)
{
    return g.kn.k1_tma && g.kind >= 1 && g.kind <= 3 && a.mode <= 2 && a.tmP4 && a.tmM4;
}

bool k1t_prepare(const Geo &g, const double *P, int nzl, int s, CUtensorMap *tmP4, CUtensorMap *tmM4)
{
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
        return false;
    auto enc = reinterpret_cast<CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                             CUtensorMapFloatOOBfill)>(fn);
    // [x: nx][y: ny][z: nzl + 2 padded planes][v: s vectors]; out-of-range x/y read as 0
    cuuint64_t dims[4] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)(nzl + 2), (cuuint64_t)s};
    cuuint64_t strides[3] = {(cuuint64_t)g.pitch * 8, (cuuint64_t)g.plane * 8, (cuuint64_t)g.vstride * 8};
    cuuint32_t es[4] = {1, 1, 1, 1};
    cuuint32_t boxp[4] = {BW, BH, 1, 1}, boxm[4] = {TX, TY, 1, 1};
    if (enc(tmP4, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double *>(P), dims, strides, boxp, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (enc(tmM4, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double *>(P), dims, strides, boxm, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (cudaFuncSetAttribute(k1t<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(k1t<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(k1t<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) != cudaSuccess ||
        cudaFuncSetAttribute(k1t<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM4) != cudaSuccess)
        return false;
    return true;
}

// TMA views of the variable-coefficient faces of one slab (nzl planes):
//   kx: 1-D over the slab's (nx+1)*ny*nzl faces, one 68-element box per row
//   ky: [nx][ny+1][nzl], box 64 x 17;  kz: [nx][ny][nzl+1], box 64 x 16
// Needs nx even (16-B strides); otherwise K1T reads the faces directly.
bool k1t_prepare_faces(const Geo &g, const double *kx, const double *ky, const double *kz, int nzl, CUtensorMap *mx,
                       CUtensorMap *my, CUtensorMap *mz)
{
    if (g.nx % 2 != 0 || (reinterpret_cast<uintptr_t>(kx) | reinterpret_cast<uintptr_t>(ky) |
                          reinterpret_cast<uintptr_t>(kz)) % 16 != 0)
        return false;
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
        return false;
    auto enc = reinterpret_cast<CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                             CUtensorMapFloatOOBfill)>(fn);
    const cuuint32_t es[3] = {1, 1, 1};
    const bool dbg = g.kn.debug != 0;
    {
        // rows of kx have an odd length (nx+1), so every other row starts at an
        // odd element: a 1-D view, one 68-element box per face row starting at
        // the row's first face rounded down to an even element (TMA box
        // starts must be 16-B aligned); the consumer adds the row's parity
        cuuint64_t dims[1] = {(cuuint64_t)(g.nx + 1) * g.ny * nzl};
        cuuint64_t str[1] = {0};
        cuuint32_t box[1] = {KXB};
        const CUresult r = enc(mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, const_cast<double *>(kx), dims, str, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (dbg) fprintf(stderr, "sscg: kx tensor map -> %d\n", (int)r);
        if (r != CUDA_SUCCESS) return false;
    }
    {
        cuuint64_t dims[3] = {(cuuint64_t)g.nx, (cuuint64_t)(g.ny + 1), (cuuint64_t)nzl};
        cuuint64_t str[2] = {(cuuint64_t)g.nx * 8, (cuuint64_t)g.nx * (g.ny + 1) * 8};
        cuuint32_t box[3] = {TX, TY + 1, 1};
        if (enc(my, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(ky), dims, str, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    {
        cuuint64_t dims[3] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)(nzl + 1)};
        cuuint64_t str[2] = {(cuuint64_t)g.nx * 8, (cuuint64_t)g.nx * g.ny * 8};
        cuuint32_t box[3] = {TX, TY, 1};
        if (enc(mz, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(kz), dims, str, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    return true;
}

void launch_k1t(const Geo &g, const K1Args &a, const DevState *st, cudaStream_t s)
{
    const int n1 = std::max(0, a.ze - a.zb), n2 = std::max(0, a.ze2 - a.zb2);
    const int nplanes = n1 + n2;
    if (nplanes <= 0) return;
    K1TWork wk;
    wk.tiles_x = (g.nx + TX - 1) / TX;
    wk.tiles_y = (g.ny + TY - 1) / TY;
    wk.zb = a.zb; wk.ze = a.ze; wk.zb2 = a.zb2; wk.ze2 = a.ze2;
    wk.j = a.j;
    const int64_t tiles = (int64_t)wk.tiles_x * wk.tiles_y;
    const int kind = (g.kind == 3 && a.tmKX) ? 4 : g.kind;
    static int occs[5] = {0, 0, 0, 0, 0};
    const int zc_env = g.kn.k1_zc;
    int &occ = occs[kind];
    if (!occ) {
        const void *fn = kind == 1 ? (const void *)k1t<1> : kind == 2 ? (const void *)k1t<2>
                       : kind == 3 ? (const void *)k1t<3> : (const void *)k1t<4>;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, THREADS, kind == 4 ? SMEM4 : SMEM) != cudaSuccess ||
            occ <= 0)
            occ = 1;
    }
    const int sms = (a.sm_cap > 0 && a.sm_cap < k2_grid()) ? a.sm_cap : k2_grid();
    const int64_t resident = (int64_t)sms * occ;
    int zc;
    if (zc_env > 0) {
        zc = std::min(std::max(n1, n2), zc_env);
    } else if (n2 > 0) {
        zc = 1;   // boundary launch: one plane per range
    } else {
        // z-chunks: few and long (each chunk re-reads 2 planes of p_j that
        // the previous chunk of the column already read, ~1/(2 zc) of the
        // launch's bytes), sized so that tiles x chunks fills whole waves of
        // the persistent grid
        double best = -1.0;
        zc = n1;
        for (int nch = 1; nch <= 64 && (n1 + nch - 1) / nch >= 4; ++nch) {
            const int z = (n1 + nch - 1) / nch;
            const int64_t items = tiles * ((n1 + z - 1) / z);   // chunks actually formed with this z
            const int64_t waves = (items + resident - 1) / resident;
            const double score = (double)items / (double)(waves * resident) / (1.0 + 0.5 / z);
            if (score > best + 1e-9) {
                best = score;
                zc = z;
            }
        }
    }
    wk.zc = zc;
    wk.nch1 = (n1 + zc - 1) / zc;
    wk.nitems = tiles * (wk.nch1 + (n2 + zc - 1) / zc);
    const unsigned grid = (unsigned)std::min<int64_t>(wk.nitems, resident);
    const CUtensorMap &P4 = *a.tmP4, &M4 = *a.tmM4;
    if (kind == 1) launch_pdl(g.kn.pdl, k1t<1>, dim3(grid), dim3(THREADS), SMEM, s, P4, M4, P4, P4, P4, g, a, st, wk);
    else if (kind == 2) launch_pdl(g.kn.pdl, k1t<2>, dim3(grid), dim3(THREADS), SMEM, s, P4, M4, P4, P4, P4, g, a, st, wk);
    else if (kind == 3) launch_pdl(g.kn.pdl, k1t<3>, dim3(grid), dim3(THREADS), SMEM, s, P4, M4, P4, P4, P4, g, a, st, wk);
    else launch_pdl(g.kn.pdl, k1t<4>, dim3(grid), dim3(THREADS), SMEM4, s, P4, M4, *a.tmKX, *a.tmKY, *a.tmKZ, g, a, st, wk);
}

}  // namespace sscg
