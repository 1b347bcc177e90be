// K1FV -- two basis steps in one pass for the variable-coefficient 7-point
// operator (BASELINE cfg 4; R12): the pair (j, j+1) of the Chebyshev
// recurrence
//   w_j = A p_j,  p_{j+1} = c_j (D^{-1} w_j - sigma p_j) [- p_{j-1}],
//   w_{j+1} = A p_{j+1},  p_{j+2} = 2 theta (D^{-1} w_{j+1} - sigma p_{j+1}) - p_j,
// with p_{j+1} kept on chip, as K1F does for the constant stencils.  The six
// face coefficients of a cell (A_ii = their sum, A_i,nbr = -k_face) are the
// same for both steps, so a pair streams them once: per pair p_j, p_{j-1}
// and the faces kx, ky, kz in, p_{j+1}, p_{j+2} out -- 7 vectors instead of
// 12 for two K1T steps (W-free schedule).
//
// Same per-point arithmetic, operand for operand, as K1T KIND 3.  Structure
// as K1F KIND 1 (k_stencil_fused.cu): warp r (1..TY+2) owns box row r, lane l
// the pair at column 2 + 2l, the last consumer warp the halo pairs; each
// thread's front cell (step j on tile + 1-cell halo) and back cell (step j+1
// on the tile) coincide, so the z-columns of p_j and p_{j+1} roll through
// registers.  The faces of the front region (kx rows as 1-D boxes from the
// even element at or below x0-2, ky and kz as 3-D boxes) are staged per plane
// by TMA into a 5-slot ring; slot z carries kx(z), ky(z) and the upper kz
// face of plane z.  A thread reads its own cells' kx, ky of plane q (front)
// and again of plane q-1 (back) from it; its kz faces roll through registers
// (the lower face of plane q is the upper one of q-1, and the back reuses the
// pair the front had one plane earlier), so two slots are live and three
// planes of faces are in flight; it keeps D^{-1} of its cells from the front
// for the back.  Faces of cells outside the grid are not zeroed: those cells'
// D^{-1}, u and stores are selected away.  Tile 64 x 12, 15 consumer warps
// and three producer warps (p_j / p_{j-1}; ky + kz boxes; the kx rows), 96
// registers (18 warps: five on one scheduler).  With ONE producer warp, ncu
// (384^3, profiles/r02o_*k1fv*) showed ~20 % of the consumers' samples on the
// p_j / face mbarrier waits while the producer was never blocked on an empty
// slot and busy ~94 % of its time: its ~19 TMA issues per plane (14 of them
// the kx rows, serialised over lanes) were the critical path, not issue slots
// of the consumers (29 fewer instructions per plane changed nothing) nor
// DRAM (54 %).  Split producers: 0.718 -> 0.623 ms per pair at 384^3
// (0.78 of copy), 0.0938 -> 0.086 ms at 192^3 (0.70).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "sscg_internal.cuh"
#include "tma.cuh"

// K1FV_TREE=1: the face terms summed as a tree, as K1M/K1F do; measured neutral
// at cfg 4 (0.0964-0.0966 ms per pair either way), so the chain is kept
#ifndef K1FV_TREE
#define K1FV_TREE 0
#endif

namespace sscg {
namespace {

#ifndef K1FV_TY
#define K1FV_TY 12
#endif
#ifndef K1FV_NSP
#define K1FV_NSP 4
#endif
constexpr int TX = 64, TY = K1FV_TY;
constexpr int BW = TX + 4;                 // staged planes: x in [x0-2, x0+TX+2)
constexpr int BHP = TY + 4;                // p_j: y in [y0-2, y0+TY+2)
constexpr int BHM = TY + 2;                // p_{j-1}: y in [y0-1, y0+TY+1)
constexpr int r128(int d) { return ((d * 8 + 127) / 128) * 128 / 8; }
constexpr int PS = r128(BW * BHP), MS = r128(BW * BHM);
constexpr int NSP = K1FV_NSP, NSM = 4, NU = 4;   // powers of two
constexpr int NROW = TY + 2;               // row warps 1..TY+2
constexpr int NCW = NROW + 1;              // + one warp for the 2*(TY+2) halo pairs
constexpr int NCT = NCW * 32;
constexpr int NPW = 3;                    // producer warps: p_j / p_{j-1}, ky + kz faces, kx face rows
constexpr int THREADS = NCT + 32 * NPW;
constexpr uint32_t PBYTES = BW * BHP * 8, MBYTES = BW * BHM * 8;
// face slots (per plane z of the march, the front cells' rows y0-1 .. y0+TY):
//   KX: TY+2 rows of 70 faces from the even element at or below x0-2 (pitch 80)
//   KY: TY+3 rows x BW (ky rows y0-1 .. y0+TY+1),  KZ: TY+2 rows x BW (kz[z-1], the lower faces)
constexpr int KXN = 70, KXP = 80;
constexpr int FKX = 0, FKY = r128(FKX + (TY + 2) * KXP), FKZ = FKY + r128((TY + 3) * BW), FS = FKZ + r128((TY + 2) * BW);
constexpr uint32_t KXBYTES = (TY + 2) * KXN * 8, KYBYTES = (TY + 3) * BW * 8, KZBYTES = (TY + 2) * BW * 8;
constexpr int NSF = 5;   // not a power of two: slot = seq % NSF
constexpr size_t SMEM = (size_t)(NSP * PS + NSM * MS + NU * PS + NSF * FS) * sizeof(double);
static_assert(2 * NROW <= 32, "halo pairs fit one warp");
static_assert(SMEM <= 227 * 1024, "shared memory");

struct K1FVWork {
    int tiles_x, tiles_y, zc;
    int64_t nitems;
    int nzl;
    int zb, ze;            // planes written by both steps: [zb, ze) within [1, nzl]
    int j;
    int front_pm;          // p_{j-1} term in the front step (j >= 1)
    int back_pn;           // the back step writes p_{j+2} (j+1 < s-1)
    int kx_shift;          // elements the 1-D kx view starts before the slab's kx (16-B alignment)
    double coef_front, coef_back, sigma;
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

__device__ __forceinline__ uint32_t pin_u32(uint32_t v)
{
    uint32_t r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}

__device__ __forceinline__ double2 lds2(const double *p) { return *reinterpret_cast<const double2 *>(p); }

struct ItemPlan {
    int tx, ty, zlo, zhi, plo, phi, mlo, mhi, flo, fhi;   // face slots [flo, fhi]
};

__device__ __forceinline__ ItemPlan plan_item(const K1FVWork &wk, int64_t item)
{
    const int ntiles = wk.tiles_x * wk.tiles_y;
    const int chunk = (int)(item / ntiles);
    const int tile = (int)(item - (int64_t)chunk * ntiles);
    ItemPlan p;
    p.ty = tile / wk.tiles_x;
    p.tx = tile - p.ty * wk.tiles_x;
    p.zlo = wk.zb + chunk * wk.zc;
    p.zhi = min(wk.ze, p.zlo + wk.zc);
    p.plo = max(p.zlo - 2, 0);
    p.phi = min(p.zhi + 1, wk.nzl + 1);
    p.mlo = max(p.zlo - 1, 1);
    p.mhi = min(p.zhi, wk.nzl);
    // the fronts at [zlo-1, zhi] inside [1, nzl] read slot q (kx, ky and the upper kz face of
    // plane q); slot flo, one plane below the first front, carries only its lower kz face
    p.flo = max(p.zlo - 1, 1) - 1;
    p.fhi = min(p.zhi, wk.nzl);
    return p;
}

// the faces of a cell pair at one plane (R12), and its diagonal
struct PairFaces {
    double kxw0, kxe0, kxe1;   // kx[x], kx[x+1] (= west of x+1), kx[x+2]
    double2 kys, kyn;          // ky[y], ky[y+1]
    double2 kzu;               // kz[z+1] (the upper face; the lower one is the previous plane's upper)
};

// A p on the pair (order as K1T KIND 3) and the diagonal
__device__ __forceinline__ double2 vc_apply(const PairFaces &F, double2 kzd, double2 c, double2 dn, double2 up,
                                            double2 ylo, double2 yhi, double l, double rr, double2 &D)
{
    D.x = kzd.x + F.kys.x + F.kxw0 + F.kxe0 + F.kyn.x + F.kzu.x;
    D.y = kzd.y + F.kys.y + F.kxe0 + F.kxe1 + F.kyn.y + F.kzu.y;
    double2 Ap;
#if K1FV_TREE
    // z, y, x face pairs summed as a tree (depth 4 instead of a 6-long FMA chain)
    Ap.x = D.x * c.x - (((kzd.x * dn.x + F.kzu.x * up.x) + (F.kys.x * ylo.x + F.kyn.x * yhi.x)) +
                        (F.kxw0 * l + F.kxe0 * c.y));
    Ap.y = D.y * c.y - (((kzd.y * dn.y + F.kzu.y * up.y) + (F.kys.y * ylo.y + F.kyn.y * yhi.y)) +
                        (F.kxe0 * c.x + F.kxe1 * rr));
#else
    Ap.x = D.x * c.x - (kzd.x * dn.x + F.kzu.x * up.x + F.kys.x * ylo.x + F.kxw0 * l + F.kxe0 * c.y + F.kyn.x * yhi.x);
    Ap.y = D.y * c.y - (kzd.y * dn.y + F.kzu.y * up.y + F.kys.y * ylo.y + F.kxe0 * c.x + F.kxe1 * rr + F.kyn.y * yhi.y);
#endif
    return Ap;
}

__device__ __forceinline__ void tma_load_1d(void *dst, const CUtensorMap *map, int x, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int x, int y, int z, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

struct FaceMaps {
    CUtensorMap kx, ky, kz;
};

__global__ void __launch_bounds__(THREADS, 1)
    k1fv(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmM,
         const __grid_constant__ FaceMaps fm, Geo g, K1Args a, const DevState *st, K1FVWork wk)
{
    PDL_ENTRY(st);
    extern __shared__ __align__(128) double smem[];
    double *sp = smem;                       // p_j ring
    double *sm = smem + NSP * PS;            // p_{j-1} ring
    double *su = sm + NSM * MS;              // U = p_{j+1} on tile + halo, NU planes
    double *sf = su + NU * PS;               // face slots
    __shared__ uint64_t fullp[NSP], emptyp[NSP], fullm[NSM], emptym[NSM], ufull[NU], fullf[NSF], emptyf[NSF];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < NSP; ++i) {
            mbar_init(&fullp[i], 1);
            mbar_init(&emptyp[i], NCT);
        }
        for (int i = 0; i < NSM; ++i) {
            mbar_init(&fullm[i], 1);
            mbar_init(&emptym[i], NCT);
        }
        for (int i = 0; i < NSF; ++i) {
            mbar_init(&fullf[i], 1);
            mbar_init(&emptyf[i], NCT);
        }
        for (int i = 0; i < NU; ++i) mbar_init(&ufull[i], NCT);
        mbar_fence_init();
        tma_prefetch_desc(&tmP);
        tma_prefetch_desc(&tmM);
        tma_prefetch_desc(&fm.kx);
        tma_prefetch_desc(&fm.ky);
        tma_prefetch_desc(&fm.kz);
    }
    __syncthreads();

    // two producer warps -- one warp issuing all ~19 loads of a plane was the
    // critical path (ncu r02o: never blocked on an empty slot, busy ~94 % of the time)
    if (warp == 0) {   // p_j and p_{j-1} planes: lane 0 issues
        if (lane != 0) return;
        uint32_t pc = 0, mc = 0;
        for (int64_t item = blockIdx.x; item < wk.nitems; item += gridDim.x) {
            const ItemPlan it = plan_item(wk, item);
            const int x0 = it.tx * TX, y0 = it.ty * TY;
            int pnext = it.plo;
            for (int q = it.zlo - 1; q <= it.zhi; ++q) {
                while (pnext <= min(q + 1, it.phi)) {
                    const int sl = pc & (NSP - 1);
                    if (pc >= NSP) mbar_wait(&emptyp[sl], ((pc / NSP) - 1) & 1);
                    mbar_expect_tx(&fullp[sl], PBYTES);
                    tma_load_4d(sp + sl * PS, &tmP, x0 - 2, y0 - 2, pnext, wk.j, &fullp[sl]);
                    ++pc;
                    ++pnext;
                }
                if (wk.front_pm && q >= it.mlo && q <= it.mhi) {
                    const int sl = mc & (NSM - 1);
                    if (mc >= NSM) mbar_wait(&emptym[sl], ((mc / NSM) - 1) & 1);
                    mbar_expect_tx(&fullm[sl], MBYTES);
                    tma_load_4d(sm + sl * MS, &tmM, x0 - 2, y0 - 1, q, wk.j - 1, &fullm[sl]);
                    ++mc;
                }
            }
        }
        return;
    }
    if (warp < NPW) {   // face slots, as far ahead as the ring allows: warp 1 lane 0 the ky / kz boxes (and the
                        // slot's byte count), warp 2 lanes 0..TY+1 the kx face rows (both wait for the empty slot)
        const bool wkx = warp == 2;
        uint32_t fc = 0;
        for (int64_t item = blockIdx.x; item < wk.nitems; item += gridDim.x) {
            const ItemPlan it = plan_item(wk, item);
            const int x0 = it.tx * TX, y0 = it.ty * TY;
            // face slot z holds kx(z), ky(z) (flo < z <= fhi) and kz(z), the upper face of plane z
            // (flo <= z <= fhi; kz index 0 is the bottom boundary face)
            for (int z = it.flo; z <= it.fhi; ++z) {
                const int sl = fc % NSF;
                const int zl = z - 1;
                const bool xy = z != it.flo;
                double *d = sf + sl * FS;
                if (lane == 0) {
                    if (fc >= NSF) mbar_wait(&emptyf[sl], ((fc / NSF) - 1) & 1);
                    if (!wkx) mbar_expect_tx(&fullf[sl], (xy ? KXBYTES + KYBYTES : 0u) + KZBYTES);
                }
                __syncwarp();
                if (wkx && xy && lane < TY + 2) {   // kx row (zl, y0-1+lane) from the even element at or below x0-2
                    const int64_t e0 = ((int64_t)zl * g.ny + (y0 - 1 + lane)) * (g.nx + 1) + x0 - 2 + wk.kx_shift;
                    tma_load_1d(d + FKX + lane * KXP, &fm.kx, (int)(e0 & ~(int64_t)1), &fullf[sl]);
                }
                if (!wkx && lane == 0) {
                    if (xy) tma_load_3d(d + FKY, &fm.ky, x0 - 2, y0 - 1, zl, &fullf[sl]);
                    tma_load_3d(d + FKZ, &fm.kz, x0 - 2, y0 - 1, z, &fullf[sl]);
                }
                __syncwarp();
                ++fc;
            }
        }
        return;
    }

    int rk, ck;
    bool task;
    if (warp - (NPW - 1) <= NROW) {   // consumer warps NPW .. NPW+NCW-1
        rk = warp - (NPW - 1);
        ck = 2 + 2 * lane;
        task = true;
    } else {
        const int h = lane;
        task = h < 2 * NROW;
        rk = task ? 1 + (h >> 1) : 1;
        ck = (h & 1) ? TX + 2 : 0;
    }
    const int ok = rk * BW + ck, omk = (rk - 1) * BW + ck;
    const int ofy = FKY + (rk - 1) * BW + ck, ofz = FKZ + (rk - 1) * BW + ck;   // own ky (south) / kz rows
    const bool ownk = task && rk >= 2 && rk < TY + 2 && ck >= 2 && ck < TX + 2;
    const bool lgk = ck > 0, rgk = ck + 2 < BW;
    const bool skip_w = a.skip_w, skip_w2 = a.skip_w2, back_pn = wk.back_pn, front_pm = wk.front_pm;
    double *const gw = a.w, *const gpn = a.pn, *const gw2 = a.w2, *const gpn2 = a.pn2;
    const int nzl = wk.nzl;
    const double sigma = wk.sigma, cfr = wk.coef_front, cbk = wk.coef_back;
    const int64_t pl = g.plane;
    uint32_t pc = 0, mc = 0, uc = 0, fc = 0;
    const uint32_t fp_a = pin_u32(smem_u32(fullp)), ep_a = pin_u32(smem_u32(emptyp)),
                   fm_a = pin_u32(smem_u32(fullm)), em_a = pin_u32(smem_u32(emptym)),
                   uf_a = pin_u32(smem_u32(ufull)), ff_a = pin_u32(smem_u32(fullf)), ef_a = pin_u32(smem_u32(emptyf));
    for (int64_t item = blockIdx.x; item < wk.nitems; item += gridDim.x) {
        const ItemPlan it = plan_item(wk, item);
        const int x0 = it.tx * TX, y0 = it.ty * TY;
        const int gx = x0 - 2 + ck, gy = y0 - 2 + rk;
        const bool vy = gy >= 0 && gy < g.ny;
        const bool v0 = task && vy && gx >= 0 && gx < g.nx, v1 = task && vy && gx + 1 >= 0 && gx + 1 < g.nx;
        const bool wown = ownk && v0;
        // kx offset of the own pair in a face slot: the row was loaded from its
        // first face (x0 - 2) rounded down to an even element
        const int64_t fa = ((int64_t)0 * g.ny + (gy)) * (g.nx + 1) + x0 - 2;   // parity only (plane term below)
        const uint32_t pbase = pc, fbase = fc;
        auto slotp = [&](int z) -> const double * {
            return sp + ((pbase + (uint32_t)(z - it.plo)) & (NSP - 1)) * PS;
        };
        auto slotf = [&](int z) -> const double * {
            return sf + ((fbase + (uint32_t)(z - it.flo)) % NSF) * FS;
        };
        auto release = [&](int z) { mbar_arrive_a(ep_a + 8 * ((pbase + (uint32_t)(z - it.plo)) & (NSP - 1))); };
        auto waitp = [&](int z) {
            const uint32_t c = pbase + (uint32_t)(z - it.plo);
            mbar_wait_a(fp_a + 8 * (c & (NSP - 1)), (c / NSP) & 1);
        };
        auto waitf = [&](int z) {
            const uint32_t c = fbase + (uint32_t)(z - it.flo);
            mbar_wait_a(ff_a + 8 * (c % NSF), (c / NSF) & 1);
        };
        auto releasef = [&](int z) { mbar_arrive_a(ef_a + 8 * ((fbase + (uint32_t)(z - it.flo)) % NSF)); };
        for (int z = it.plo; z <= min(it.zlo, it.phi); ++z) waitp(z);
        double2 pdn = make_double2(0.0, 0.0);
        if (it.zlo - 2 >= it.plo) {
            pdn = lds2(slotp(it.zlo - 2) + ok);
            release(it.zlo - 2);
        }
        double2 pc0 = lds2(slotp(it.zlo - 1) + ok);
        double2 um2 = make_double2(0.0, 0.0), um1 = make_double2(0.0, 0.0);
        double2 dinvb = make_double2(0.0, 0.0);   // D^{-1} of the back's cells (from the previous front)
        // the own pair's kz faces roll through registers: at plane q, kza = kz(q-2), kzb = kz(q-1)
        // (the back's lower / upper face, the front's lower face); the front loads kz(q)
        waitf(it.flo);
        double2 kza = make_double2(0.0, 0.0), kzb = lds2(slotf(it.flo) + ofz);
        releasef(it.flo);
        int64_t off = (int64_t)(it.zlo - 1) * pl + (int64_t)gy * g.pitch + gx;
        const int64_t rowfaces = (int64_t)g.ny * (g.nx + 1);
        // the own pair's kx, ky faces at plane z (slot z) with the given upper kz face
        auto faces_at = [&](int z, double2 kzu) -> PairFaces {
            PairFaces F;
            const double *Fz = slotf(z);
            const int px = ck + (int)((fa + (int64_t)(z - 1) * rowfaces + wk.kx_shift) & 1);
            const double *kxr = Fz + FKX + (rk - 1) * KXP + px;
            F.kxw0 = kxr[0];
            F.kxe0 = kxr[1];
            F.kxe1 = kxr[2];
            F.kys = lds2(Fz + ofy);
            F.kyn = lds2(Fz + ofy + BW);
            F.kzu = kzu;
            // a cell outside the grid keeps whatever its face slots hold: its D^{-1}, u and
            // stores are selected away below (never multiplied away), and a valid cell reads
            // only its own faces (26 fewer selects per plane than zeroing them here)
            return F;
        };
        auto plane = [&](int q, auto steady) {
            constexpr bool S = decltype(steady)::value;
            const bool inside = S || (q >= 1 && q <= nzl);
            const bool has_up = S || q + 1 <= it.phi;
            const double *P0 = slotp(q);
            double2 pup = make_double2(0.0, 0.0);
            if (has_up) {
                if (S || q >= it.zlo) waitp(q + 1);
                pup = lds2(slotp(q + 1) + ok);
            }
            if (inside) waitf(q);
            const bool mloaded = front_pm && (S || (q >= it.mlo && q <= it.mhi));
            const uint32_t ms = mc & (NSM - 1);
            if (mloaded) mbar_wait_a(fm_a + 8 * ms, (mc / NSM) & 1);
            // ---------------- front(q): step j on tile + halo ----------------
            double2 u = make_double2(0.0, 0.0), dinv = make_double2(0.0, 0.0), kzc = kzb;
            if (inside) {
                kzc = lds2(slotf(q) + ofz);
                const double2 kzd = kzb;
                const PairFaces F = faces_at(q, kzc);
                const double2 c = pc0;
                const double2 ylo = lds2(P0 + ok - BW), yhi = lds2(P0 + ok + BW);
                const double l = lgk ? P0[ok - 1] : 0.0;
                const double rr = rgk ? P0[ok + 2] : 0.0;
                double2 D;
                double2 Ap = vc_apply(F, kzd, c, pdn, pup, ylo, yhi, l, rr, D);
                dinv = make_double2(v0 ? 1.0 / D.x : 0.0, v1 ? 1.0 / D.y : 0.0);
                u.x = cfr * (dinv.x * Ap.x - sigma * c.x);
                u.y = cfr * (dinv.y * Ap.y - sigma * c.y);
                if (mloaded) {
                    const double2 pm = lds2(sm + ms * MS + omk);
                    u.x -= pm.x;
                    u.y -= pm.y;
                }
                if (!v0) u.x = 0.0;
                if (!v1) u.y = 0.0;
                if (wown && (S || (q >= it.zlo && q < it.zhi))) {
                    if (!v1) Ap.y = 0.0;
                    if (!skip_w) __stcs(reinterpret_cast<double2 *>(gw + off), Ap);
                    *reinterpret_cast<double2 *>(gpn + off) = u;
                }
            }
            if (task) *reinterpret_cast<double2 *>(su + (uc & (NU - 1)) * PS + ok) = u;
            mbar_arrive_a(uf_a + 8 * (uc & (NU - 1)));
            if (mloaded) {
                mbar_arrive_a(em_a + 8 * ms);
                ++mc;
            }
            release(q);
            // ---------------- back(z = q-1): step j+1 on the tile ----------------
            if (S || uc > 0) mbar_wait_a(uf_a + 8 * ((uc - 1) & (NU - 1)), ((uc - 1) / NU) & 1);
            if (wown && (S || (q - 1 >= it.zlo && q - 1 < it.zhi))) {
                const double *U0 = su + ((uc - 1) & (NU - 1)) * PS;
                const double2 c = um1, dn = um2, up = u;
                const double2 ylo = lds2(U0 + ok - BW), yhi = lds2(U0 + ok + BW);
                const double l = U0[ok - 1], rr = U0[ok + 2];
                double2 D;
                const double2 kzdb = kza;
                const PairFaces Fb = faces_at(q - 1, kzb);   // face slot q-1 is released after this
                double2 Ap = vc_apply(Fb, kzdb, c, dn, up, ylo, yhi, l, rr, D);
                if (!v1) Ap.y = 0.0;
                if (!skip_w2) __stcs(reinterpret_cast<double2 *>(gw2 + off - pl), Ap);
                if (back_pn) {
                    const double2 pj = pdn;
                    const double v0b = cbk * (dinvb.x * Ap.x - sigma * c.x) - pj.x;
                    double v1b = cbk * (dinvb.y * Ap.y - sigma * c.y) - pj.y;
                    if (!v1) v1b = 0.0;
                    *reinterpret_cast<double2 *>(gpn2 + off - pl) = make_double2(v0b, v1b);
                }
            }
            if (S || (q - 1 > it.flo && q - 1 <= it.fhi)) releasef(q - 1);   // faces of plane q-1 done
            if (inside) {
                kza = kzb;
                kzb = kzc;
            }
            ++uc;
            um2 = um1;
            um1 = u;
            pdn = pc0;
            pc0 = pup;
            dinvb = dinv;
            off += pl;
        };
        using Gen = std::integral_constant<bool, false>;
        using Steady = std::integral_constant<bool, true>;
        int q = it.zlo - 1;
        plane(q++, Gen());
        if (q < it.zhi) plane(q++, Gen());
#pragma unroll 1
        for (; q < it.zhi; ++q) plane(q, Steady());
        for (; q <= it.zhi; ++q) plane(q, Gen());
        for (int z = max(it.zhi + 1, it.plo); z <= it.phi; ++z) release(z);
        for (int z = max(it.zhi, it.flo + 1); z <= it.fhi; ++z) releasef(z);
        pc = pbase + (it.phi - it.plo + 1);
        fc = fbase + (it.fhi - it.flo + 1);
    }
}

}  // namespace

bool k1fv_prepare(const Geo &g, const double *P, int nzl, int s, CUtensorMap *tmP, CUtensorMap *tmM)
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
    cuuint64_t dims[4] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)(nzl + 2), (cuuint64_t)s};
    cuuint64_t strides[3] = {(cuuint64_t)g.pitch * 8, (cuuint64_t)g.plane * 8, (cuuint64_t)g.vstride * 8};
    cuuint32_t es[4] = {1, 1, 1, 1};
    cuuint32_t boxp[4] = {BW, BHP, 1, 1}, boxm[4] = {BW, BHM, 1, 1};
    if (enc(tmP, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double *>(P), dims, strides, boxp, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (enc(tmM, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double *>(P), dims, strides, boxm, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    return cudaFuncSetAttribute(k1fv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) == cudaSuccess;
}

// tensor maps of the faces for the K1FV boxes (nx even, 16-B aligned arrays):
// kx as a 1-D view (rows have odd length nx+1: one 70-face box per row from
// the even element at or below its first face), ky / kz as 3-D views
bool k1fv_prepare_faces(const Geo &g, const double *kx, const double *ky, const double *kz, int nzl, CUtensorMap *mx,
                        CUtensorMap *my, CUtensorMap *mz, int *kx_shift)
{
    // kx of a slab after the first starts at an odd element when (nx+1)*ny*z0
    // is odd: the 1-D view then starts one element earlier (*kx_shift = 1)
    const int shift = (int)((reinterpret_cast<uintptr_t>(kx) % 16) / 8);
    if (g.nx % 2 != 0 || reinterpret_cast<uintptr_t>(kx) % 8 != 0 ||
        (reinterpret_cast<uintptr_t>(ky) | reinterpret_cast<uintptr_t>(kz)) % 16 != 0)
        return false;
    *kx_shift = shift;
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
    {
        cuuint64_t dims[1] = {(cuuint64_t)(g.nx + 1) * g.ny * nzl + shift};
        cuuint64_t str[1] = {0};
        cuuint32_t box[1] = {KXN};
        if (enc(mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, const_cast<double *>(kx - shift), dims, str, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    {
        cuuint64_t dims[3] = {(cuuint64_t)g.nx, (cuuint64_t)(g.ny + 1), (cuuint64_t)nzl};
        cuuint64_t str[2] = {(cuuint64_t)g.nx * 8, (cuuint64_t)g.nx * (g.ny + 1) * 8};
        cuuint32_t box[3] = {BW, TY + 3, 1};
        if (enc(my, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(ky), dims, str, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    {
        cuuint64_t dims[3] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)(nzl + 1)};
        cuuint64_t str[2] = {(cuuint64_t)g.nx * 8, (cuuint64_t)g.nx * g.ny * 8};
        cuuint32_t box[3] = {BW, TY + 2, 1};
        if (enc(mz, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(kz), dims, str, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    return true;
}

// SSCG_K1_FUSE=0 / SSCG_K1_FUSE_VC=0 forbid the pair, SSCG_K1_FUSE_VC=1 forces
// it; default: slabs with >= 8 tile-planes per SM.  Measured (faces staged
// by TMA, 64 x 12 tiles, 16 warps): cfg 4 192^3 0.109 ms per pair vs 2 x 0.063
// for two K1T steps (1.19 vs 1.29 ms per outer), 384^3 0.82 vs 2 x 0.457 ms
// (9.25 vs 10.5 ms per outer).  It moves 7 instead of 12 vectors per two
// steps, so its fraction of the copy peak (0.55) is lower than K1T's (0.81)
// while the time is shorter.
bool k1fv_enabled(const Geo &g, int nzl)
{
    if (g.kn.k1_fuse == 0) return false;
    if (g.kn.k1_fuse_vc >= 0) return g.kn.k1_fuse_vc == 1;
    const int64_t tiles = (int64_t)((g.nx + TX - 1) / TX) * ((g.ny + TY - 1) / TY);
    return tiles * nzl >= 8 * k2_grid();
}

void launch_k1fv(const Geo &g, const K1Args &a, double theta, int s, const DevState *st, cudaStream_t strm)
{
    K1FVWork wk;
    wk.tiles_x = (g.nx + TX - 1) / TX;
    wk.tiles_y = (g.ny + TY - 1) / TY;
    wk.nzl = a.nzl;
    wk.zb = a.zb;
    wk.ze = a.ze;
    wk.j = a.j;
    wk.front_pm = a.j > 0;
    wk.back_pn = (a.j + 1 < s - 1) ? 1 : 0;
    wk.kx_shift = a.kx_shift;
    wk.coef_front = (a.j == 0) ? theta : 2.0 * theta;
    wk.coef_back = 2.0 * theta;
    wk.sigma = a.sigma;
    const int64_t tiles = (int64_t)wk.tiles_x * wk.tiles_y;
    const int64_t resident = (a.sm_cap > 0 && a.sm_cap < k2_grid()) ? a.sm_cap : k2_grid();
    const int n1 = a.ze - a.zb;
    if (n1 <= 0) return;
    int zc = n1;
    double best = -1.0;
    for (int nch = 1; nch <= 64 && (n1 + nch - 1) / nch >= 4; ++nch) {
        const int z = (n1 + nch - 1) / nch;
        const int64_t items = tiles * ((n1 + z - 1) / z);
        const int64_t waves = (items + resident - 1) / resident;
        const double score = (double)items / (double)(waves * resident) / (1.0 + 1.0 / z);
        if (score > best + 1e-9) {
            best = score;
            zc = z;
        }
    }
    wk.zc = zc;
    wk.nitems = tiles * ((n1 + zc - 1) / zc);
    const unsigned grid = (unsigned)std::min<int64_t>(wk.nitems, resident);
    FaceMaps fmaps{*a.tmKX, *a.tmKY, *a.tmKZ};
    launch_pdl(g.kn.pdl, k1fv, dim3(grid), dim3(THREADS), SMEM, strm, *a.tmF_P, *a.tmF_M, fmaps, g, a, st, wk);
}

}  // namespace sscg
