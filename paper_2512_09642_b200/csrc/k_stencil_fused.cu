// K1F -- two basis steps in one pass (7-point and 27-point): the pair
// (j, j+1) of the Chebyshev recurrence
//   w_j     = A p_j,      p_{j+1} = c_j (D^{-1} w_j - sigma p_j) [- p_{j-1}]
//   w_{j+1} = A p_{j+1},  p_{j+2} = 2 theta (D^{-1} w_{j+1} - sigma p_{j+1}) - p_j
// with p_{j+1} kept on chip between the two steps (SURVEY §8(f) NEXT-3,
// "matrix-powers" blocking of depth 2).  Per pair it streams p_j and p_{j-1}
// in and p_{j+1}, p_{j+2} out (+ w_j, w_{j+1} when the schedule stores W): 4
// vectors instead of the 6 of two single steps in the W-free schedule (the
// default for small 7-point slabs and every slab with neighbours; large
// single slabs run K1M triples, k_stencil_mp3.cu).
//
// Same arithmetic, operand for operand, as K1T (k_stencil_tma.cu): the
// front step computes p_{j+1} on the tile plus a one-cell x/y halo (the halo
// values are recomputed redundantly by neighbouring tiles) from p_j staged by
// TMA with a two-cell halo; cells outside the global grid are forced to the
// Dirichlet value 0.
//
// Pipeline over the planes q of a z-chunk [zlo, zhi):
//   front(q):  w_j(q), p_{j+1}(q) on the tile (written when zlo <= q < zhi),
//              p_{j+1}(q) on tile + halo into the shared ring U (4 planes)
//   back(q-1): w_{j+1}, p_{j+2} at plane q-1 from U(q-2..q) and p_j(q-1)
// Warp 0 produces (TMA boxes of p_j and p_{j-1} into mbarrier rings), warps
// 1..NCW consume.  7-point: row-aligned tasks whose front and back cells
// coincide, z-columns in registers, per-plane mbarriers on U (see the KIND 1
// branch); 27-point: one front and one back task per thread and plane with
// one named barrier per plane.  7-point at 0.92 of its 2:2 mix ceiling
// (DESIGN.md §6).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "sscg_internal.cuh"
#include "tma.cuh"

// sum of the six neighbour terms of the 7-point A p (z pair, y pair, x pair):
// a depth-3 tree (K1F_TREE, as K1M) or the left-to-right chain of K1T
// (measured: cfg 2 neutral, 0.0193 ms per pair either way; cfg 5 pairs 0.525 vs 0.530)
#ifndef K1F_TREE
#define K1F_TREE 1
#endif
#if K1F_TREE
#define K1F_SUM6(zd, zu, yl, yh, xl, xr) ((((zd) + (zu)) + ((yl) + (yh))) + ((xl) + (xr)))
#else
#define K1F_SUM6(zd, zu, yl, yh, xl, xr) ((zd) + (yl) + (xl) + (xr) + (yh) + (zu))
#endif

namespace sscg {
namespace {

// Tile 64 x 8 with two CTAs per SM (two planes in flight per SM; the per-plane
// work of one CTA is latency-bound) -- K1F_TY=16 builds the one-CTA variant.
#ifndef K1F_TY
#define K1F_TY 16
#endif
constexpr int TX = 64, TY = K1F_TY;
constexpr int MINB = (TY <= 8) ? 2 : 1;    // CTAs per SM
constexpr int BW = TX + 4;                 // all staged planes: x in [x0-2, x0+TX+2)
constexpr int BHP = TY + 4;                // p_j: y in [y0-2, y0+TY+2)
constexpr int BHM = TY + 2;                // p_{j-1}: y in [y0-1, y0+TY+1)
constexpr int PS = ((BW * BHP * 8 + 127) / 128) * 128 / 8;   // doubles per p_j / U slot (128-B multiple)
constexpr int MS = ((BW * BHM * 8 + 127) / 128) * 128 / 8;
constexpr int NSP = 8, NSM = 8, NU = 4;   // powers of two (slot = seq & (N - 1))
// one front task per consumer thread (27-point), or TY+2 row warps plus the
// halo-column warps (7-point)
constexpr int NCW = std::max(((TY + 2) * (BW / 2) + 31) / 32, (TY + 2) + (2 * (TY + 2) + 31) / 32);
constexpr int NCT = NCW * 32;
constexpr int THREADS = NCT + 32;
constexpr uint32_t PBYTES = BW * BHP * 8, MBYTES = BW * BHM * 8;
constexpr size_t SMEM = (size_t)(NSP * PS + NSM * MS + NU * PS) * sizeof(double);
constexpr int FRONT_TASKS = (TY + 2) * (BW / 2);   // 18 rows x 34 pairs
constexpr int BACK_TASKS = TY * (TX / 2);          // 16 rows x 32 pairs
static_assert(NCT >= FRONT_TASKS && NCT >= BACK_TASKS, "one front and one back task per consumer thread");

struct K1FWork {
    int tiles_x, tiles_y, zc;
    int64_t nitems;
    int nzl;
    int zb, ze;            // planes written by both steps: [zb, ze) within [1, nzl]
    int j;
    int front_pm;          // p_{j-1} term in the front step (j >= 1)
    int back_pn;           // the back step writes p_{j+2} (j+1 < s-1)
    double coef_front, coef_back, sigma, center, dinv_c;
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

__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NCT) : "memory"); }

// an opaque copy: keeps a value the compiler would rematerialise in a register
__device__ __forceinline__ uint32_t pin_u32(uint32_t v)
{
    uint32_t r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}

__device__ __forceinline__ double2 lds2(const double *p) { return *reinterpret_cast<const double2 *>(p); }

// planes of p_j loaded for an item: [plo, phi] (the front needs q-1..q+1 for
// q in [zlo-1, zhi] inside the slab's padded range [0, nzl+1])
struct ItemPlan {
    int tx, ty, zlo, zhi, plo, phi, mlo, mhi;
};

__device__ __forceinline__ ItemPlan plan_item(const K1FWork &wk, int64_t item)
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
    p.mlo = max(p.zlo - 1, 1);   // p_{j-1} planes used by front(q), 1 <= q <= nzl
    p.mhi = min(p.zhi, wk.nzl);
    return p;
}

// 3-point row sums of the pair (c, c+1) of a staged row: (l + c.x + c.y, c.x + c.y + r)
__device__ __forceinline__ double2 rowsum3(const double *row)
{
    const double l = row[-1], r = row[2];
    const double2 c = lds2(row);
    return make_double2(l + c.x + c.y, c.x + c.y + r);
}

// 3x3 in-plane box sums of the pair at offset o (27-point: A p = 27 p - box3x3x3(p))
__device__ __forceinline__ double2 box9(const double *P, int o)
{
    const double2 r0 = rowsum3(P + o - BW), r1 = rowsum3(P + o), r2 = rowsum3(P + o + BW);
    return make_double2(r0.x + r1.x + r2.x, r0.y + r1.y + r2.y);
}

template <int KIND>
__global__ void __launch_bounds__(THREADS, MINB)
    k1f(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmM, Geo g, K1Args a,
        const DevState *st, K1FWork wk)
{
    PDL_ENTRY(st);
    extern __shared__ __align__(128) double smem[];
    double *sp = smem;                       // p_j ring
    double *sm = smem + NSP * PS;            // p_{j-1} ring
    double *su = sm + NSM * MS;              // U = p_{j+1} on tile + halo, NU planes
    __shared__ uint64_t fullp[NSP], emptyp[NSP], fullm[NSM], emptym[NSM], ufull[NU];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        // 7-point: every consumer thread arrives; 27-point: one arrival per warp
        const int consumers = (KIND == 1) ? NCT : NCW;
        for (int i = 0; i < NSP; ++i) {
            mbar_init(&fullp[i], 1);
            mbar_init(&emptyp[i], consumers);
        }
        for (int i = 0; i < NSM; ++i) {
            mbar_init(&fullm[i], 1);
            mbar_init(&emptym[i], consumers);
        }
        for (int i = 0; i < NU; ++i) mbar_init(&ufull[i], consumers);
        mbar_fence_init();
        tma_prefetch_desc(&tmP);
        tma_prefetch_desc(&tmM);
    }
    __syncthreads();

    if (warp == 0) {
        if (lane == 0) {
            uint32_t pc = 0, mc = 0;
            for (int64_t item = blockIdx.x; item < wk.nitems; item += gridDim.x) {
                const ItemPlan it = plan_item(wk, item);
                const int x0 = it.tx * TX, y0 = it.ty * TY;
                int pnext = it.plo, mnext = it.mlo;
                for (int q = it.zlo - 1; q <= it.zhi; ++q) {
                    while (pnext <= min(q + 1, it.phi)) {
                        const int sl = pc % NSP;
                        if (pc >= NSP) mbar_wait(&emptyp[sl], ((pc / NSP) - 1) & 1);
                        mbar_expect_tx(&fullp[sl], PBYTES);
                        tma_load_4d(sp + sl * PS, &tmP, x0 - 2, y0 - 2, pnext, wk.j, &fullp[sl]);
                        ++pc;
                        ++pnext;
                    }
                    if (wk.front_pm && q >= it.mlo && q <= it.mhi) {
                        const int sl = mc % NSM;
                        if (mc >= NSM) mbar_wait(&emptym[sl], ((mc / NSM) - 1) & 1);
                        mbar_expect_tx(&fullm[sl], MBYTES);
                        tma_load_4d(sm + sl * MS, &tmM, x0 - 2, y0 - 1, q, wk.j - 1, &fullm[sl]);
                        ++mc;
                        ++mnext;
                    }
                }
            }
        }
        return;
    }

    // one front task (pair of a tile + halo row) and at most one back task
    // (pair of a tile row) per consumer thread; their smem offsets and masks
    // are fixed for the kernel, the global ones per item
    const int ct = tid - 32;
    const bool has_f = ct < FRONT_TASKS, has_b = ct < BACK_TASKS;
    const int rf = 1 + ct / (BW / 2), cf = 2 * (ct % (BW / 2));        // box row 1..18, col 0..66
    const int rb = 2 + ct / (TX / 2), cb = 2 + 2 * (ct % (TX / 2));    // box row 2..17, col 2..65
    const int of = rf * BW + cf, omf = (rf - 1) * BW + cf;
    const int ob = has_b ? rb * BW + cb : 2 * BW + 2;   // threads without a back task read a safe cell
    const bool own_cell = rf >= 2 && rf < TY + 2 && cf >= 2 && cf < TX + 2;
    const bool lgf = cf > 0, rgf = cf + 2 < BW;
    uint32_t pc = 0, mc = 0;   // sequence numbers of the next p_j / p_{j-1} slot to consume
    const int64_t pl = g.plane;
    const double center = wk.center, dinv_c = wk.dinv_c, sigma = wk.sigma;
    const double cfr = wk.coef_front, cbk = wk.coef_back;
    if constexpr (KIND == 1) {
        // 7-point: row-aligned tasks with the z-column in registers.  Warps
        // 1..TY+2 take box row r = warp and the tile's 32 pairs c = 2 + 2*lane;
        // the warps after them the halo pairs c = 0 and c = TX+2 of rows
        // 1..TY+2.  Each task's front and back cell are the same cell, so
        // p_j(q-1), p_j(q), u(z-1), u(z) and u(q) at the own cell roll through
        // registers along z and only the in-plane neighbours come from shared
        // memory.  U(q) is published through ufull (split barrier: a thread
        // waits for U(q-1) of all threads, not for everyone's U(q)); with
        // NU = 4 slots a thread that waited U(q-2) knows every read of U(q-4)
        // is done before it overwrites that slot.  Every consumer thread
        // arrives on the mbarriers itself (no warp elect).
        int rk, ck;
        bool task;
        if (warp <= TY + 2) {
            rk = warp;
            ck = 2 + 2 * lane;
            task = true;
        } else {
            const int h = (warp - TY - 3) * 32 + lane;
            task = h < 2 * (TY + 2);
            rk = task ? 1 + (h >> 1) : 1;
            ck = (h & 1) ? TX + 2 : 0;
        }
        const int ok = rk * BW + ck, omk = (rk - 1) * BW + ck;
        const bool ownk = task && rk >= 2 && rk < TY + 2 && ck >= 2 && ck < TX + 2;
        const bool lgk = ck > 0, rgk = ck + 2 < BW;
        const bool skip_w = a.skip_w, skip_w2 = a.skip_w2, back_pn = wk.back_pn, front_pm = wk.front_pm;
        double *const gw = a.w, *const gpn = a.pn, *const gw2 = a.w2, *const gpn2 = a.pn2;
        const int nzl = wk.nzl;
        uint32_t uc = 0;   // sequence number of the next U plane (slot uc % NU)
        // shared-window addresses, pinned in registers
        const uint32_t fp_a = pin_u32(smem_u32(fullp)), ep_a = pin_u32(smem_u32(emptyp)),
                       fm_a = pin_u32(smem_u32(fullm)), em_a = pin_u32(smem_u32(emptym)),
                       uf_a = pin_u32(smem_u32(ufull));
        for (int64_t item = blockIdx.x; item < wk.nitems; item += gridDim.x) {
            const ItemPlan it = plan_item(wk, item);
            const int x0 = it.tx * TX, y0 = it.ty * TY;
            const int gx = x0 - 2 + ck, gy = y0 - 2 + rk;
            const bool vy = gy >= 0 && gy < g.ny;
            const bool v0 = task && vy && gx >= 0 && gx < g.nx, v1 = task && vy && gx + 1 >= 0 && gx + 1 < g.nx;
            const bool wown = ownk && v0;   // the tile's own cell: all four outputs go to HBM
            const uint32_t pbase = pc;      // sequence number of plane plo
            auto slotp = [&](int z) -> const double * {
                return sp + ((pbase + (uint32_t)(z - it.plo)) & (NSP - 1)) * PS;
            };
            auto release = [&](int z) { mbar_arrive_a(ep_a + 8 * ((pbase + (uint32_t)(z - it.plo)) & (NSP - 1))); };
            auto waitp = [&](int z) {
                const uint32_t c = pbase + (uint32_t)(z - it.plo);
                mbar_wait_a(fp_a + 8 * (c & (NSP - 1)), (c / NSP) & 1);
            };
            for (int z = it.plo; z <= min(it.zlo, it.phi); ++z) waitp(z);
            double2 pdn = make_double2(0.0, 0.0);   // p_j(q-1), own cell
            if (it.zlo - 2 >= it.plo) {
                pdn = lds2(slotp(it.zlo - 2) + ok);
                release(it.zlo - 2);
            }
            double2 pc0 = lds2(slotp(it.zlo - 1) + ok);   // p_j(q)
            double2 um2 = make_double2(0.0, 0.0), um1 = make_double2(0.0, 0.0);   // u(q-2), u(q-1)
            int64_t off = (int64_t)(it.zlo - 1) * pl + (int64_t)gy * g.pitch + gx;   // global index, plane q
            // one plane: front(q), then back(q-1).  STEADY: zlo < q < zhi, where
            // every plane condition below is known to hold.
            auto plane = [&](int q, auto steady) {
                constexpr bool S = decltype(steady)::value;
                const bool inside = S || (q >= 1 && q <= nzl);
                const bool has_up = S || q + 1 <= it.phi;
                const double *P0 = slotp(q);
                double2 pup = make_double2(0.0, 0.0);   // p_j(q+1)
                if (has_up) {
                    if (S || q >= it.zlo) waitp(q + 1);
                    pup = lds2(slotp(q + 1) + ok);
                }
                const bool mloaded = front_pm && (S || (q >= it.mlo && q <= it.mhi));
                const uint32_t ms = mc & (NSM - 1);
                if (mloaded) mbar_wait_a(fm_a + 8 * ms, (mc / NSM) & 1);
                // ---------------- front(q): step j on tile + halo ----------------
                double2 u = make_double2(0.0, 0.0);
                if (inside) {
                    const double2 c = pc0, dn = pdn, up = pup;
                    const double2 ylo = lds2(P0 + ok - BW), yhi = lds2(P0 + ok + BW);
                    const double l = lgk ? P0[ok - 1] : 0.0;
                    const double rr = rgk ? P0[ok + 2] : 0.0;
                    double2 Ap;
                    Ap.x = center * c.x - K1F_SUM6(dn.x, up.x, ylo.x, yhi.x, l, c.y);
                    Ap.y = center * c.y - K1F_SUM6(dn.y, up.y, ylo.y, yhi.y, c.x, rr);
                    u.x = cfr * (dinv_c * Ap.x - sigma * c.x);
                    u.y = cfr * (dinv_c * Ap.y - sigma * c.y);
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
                release(q);   // p_j plane q is done (front(q+1) reads q+1, q+2)
                // ---------------- back(z = q-1): step j+1 on the tile ----------------
                if (S || uc > 0) mbar_wait_a(uf_a + 8 * ((uc - 1) & (NU - 1)), ((uc - 1) / NU) & 1);
                if (wown && (S || (q - 1 >= it.zlo && q - 1 < it.zhi))) {
                    const double *U0 = su + ((uc - 1) & (NU - 1)) * PS;
                    const double2 c = um1, dn = um2, up = u;
                    const double2 ylo = lds2(U0 + ok - BW), yhi = lds2(U0 + ok + BW);
                    const double l = U0[ok - 1], rr = U0[ok + 2];
                    double2 Ap;
                    Ap.x = center * c.x - K1F_SUM6(dn.x, up.x, ylo.x, yhi.x, l, c.y);
                    Ap.y = center * c.y - K1F_SUM6(dn.y, up.y, ylo.y, yhi.y, c.x, rr);
                    if (!v1) Ap.y = 0.0;
                    if (!skip_w2) __stcs(reinterpret_cast<double2 *>(gw2 + off - pl), Ap);
                    if (back_pn) {
                        const double2 pj = pdn;   // p_j(z)
                        const double v0b = cbk * (dinv_c * Ap.x - sigma * c.x) - pj.x;
                        double v1b = cbk * (dinv_c * Ap.y - sigma * c.y) - pj.y;
                        if (!v1) v1b = 0.0;
                        *reinterpret_cast<double2 *>(gpn2 + off - pl) = make_double2(v0b, v1b);
                    }
                }
                ++uc;
                um2 = um1;
                um1 = u;
                pdn = pc0;
                pc0 = pup;
                off += pl;
            };
            using Gen = std::integral_constant<bool, false>;
            using Steady = std::integral_constant<bool, true>;
            int q = it.zlo - 1;
            plane(q++, Gen());
            if (q < it.zhi) plane(q++, Gen());   // q = zlo: no back output yet
#pragma unroll 1
            for (; q < it.zhi; ++q) plane(q, Steady());
            for (; q <= it.zhi; ++q) plane(q, Gen());
            if (it.zhi + 1 <= it.phi) release(it.zhi + 1);
            pc = pbase + (it.phi - it.plo + 1);
        }
        return;
    } else {
    for (int64_t item = blockIdx.x; item < wk.nitems; item += gridDim.x) {
        const ItemPlan it = plan_item(wk, item);
        const int x0 = it.tx * TX, y0 = it.ty * TY;
        const int gxf = x0 - 2 + cf, gyf = y0 - 2 + rf, gxb = x0 - 2 + cb, gyb = y0 - 2 + rb;
        const bool vyf = gyf >= 0 && gyf < g.ny;
        const bool v0f = has_f && vyf && gxf >= 0 && gxf < g.nx, v1f = has_f && vyf && gxf + 1 >= 0 && gxf + 1 < g.nx;
        const bool wf = own_cell && v0f;                         // writes w_j, p_{j+1} of its own cell
        const bool wb = has_b && gyb < g.ny && gxb < g.nx, v1b = gxb + 1 < g.nx;
        const int64_t gif = (int64_t)gyf * g.pitch + gxf, gib = (int64_t)gyb * g.pitch + gxb;
        const uint32_t pbase = pc;   // p_j plane z lives in slot (pbase + z - plo) % NSP
        int pwaited = it.plo - 1;
        double2 bf_m = {}, bf_0 = {}, bf_p = {}, bb_m = {}, bb_0 = {}, bb_p = {};   // 27-point windows
        bool bvalid = false;
        for (int q = it.zlo - 1; q <= it.zhi; ++q) {
            const int need = min(q + 1, it.phi);
            while (pwaited < need) {
                ++pwaited;
                const uint32_t c = pbase + (pwaited - it.plo);
                mbar_wait(&fullp[c % NSP], (c / NSP) & 1);
            }
            const uint32_t cq = pbase + (q - it.plo);   // slot sequence of plane q (q >= plo except q = -1)
            const double *P0 = sp + (cq % NSP) * PS;
            double *U = su + ((q + 8) % NU) * PS;
            // ---------------- front(q): step j on tile + halo ----------------
            const bool inside = q >= 1 && q <= wk.nzl;
            const bool mloaded = wk.front_pm && q >= it.mlo && q <= it.mhi;
            const double *M = sm + (mc % NSM) * MS;
            if (mloaded) mbar_wait(&fullm[mc % NSM], (mc / NSM) & 1);
            if (has_f) {
                double2 u = make_double2(0.0, 0.0);
                if (KIND == 2 && inside) {
                    // box sums of p_j slide through registers: B(q-1), B(q) kept, B(q+1) new
                    if (q == it.zlo - 1 || !bvalid) {
                        bf_m = box9(sp + ((cq - 1) % NSP) * PS, of);
                        bf_0 = box9(P0, of);
                    }
                    bf_p = box9(sp + ((cq + 1) % NSP) * PS, of);
                }
                if (inside) {
                    const double2 c = lds2(P0 + of);
                    double2 Ap;
                    if (KIND == 2) {
                        Ap.x = 27.0 * c.x - (bf_m.x + bf_0.x + bf_p.x);
                        Ap.y = 27.0 * c.y - (bf_m.y + bf_0.y + bf_p.y);
                    } else {
                        const double *Pm = sp + ((cq - 1) % NSP) * PS, *Pp = sp + ((cq + 1) % NSP) * PS;
                        const double2 dn = lds2(Pm + of), up = lds2(Pp + of);
                        const double2 ylo = lds2(P0 + of - BW), yhi = lds2(P0 + of + BW);
                        const double l = lgf ? P0[of - 1] : 0.0;
                        const double rr = rgf ? P0[of + 2] : 0.0;
                        Ap.x = center * c.x - K1F_SUM6(dn.x, up.x, ylo.x, yhi.x, l, c.y);
                        Ap.y = center * c.y - K1F_SUM6(dn.y, up.y, ylo.y, yhi.y, c.x, rr);
                    }
                    u.x = cfr * (dinv_c * Ap.x - sigma * c.x);
                    u.y = cfr * (dinv_c * Ap.y - sigma * c.y);
                    if (mloaded) {
                        const double2 pm = lds2(M + omf);
                        u.x -= pm.x;
                        u.y -= pm.y;
                    }
                    if (!v0f) u.x = 0.0;
                    if (!v1f) u.y = 0.0;
                    if (wf && q >= it.zlo && q < it.zhi) {   // the tile's own cells: w_j, p_{j+1} to HBM
                        const int64_t i = (int64_t)q * pl + gif;
                        if (!v1f) Ap.y = 0.0;
                        if (!a.skip_w) __stcs(reinterpret_cast<double2 *>(a.w + i), Ap);
                        *reinterpret_cast<double2 *>(a.pn + i) = u;
                    }
                }
                *reinterpret_cast<double2 *>(U + of) = u;
                if (KIND == 2) {
                    bvalid = inside;
                    bf_m = bf_0;
                    bf_0 = bf_p;
                }
            }
            if (mloaded) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&emptym[mc % NSM]);
                ++mc;
            }
            consumers_sync();   // U(q) complete; U(q-4) no longer read
            // ---------------- back(q-1): step j+1 on the tile ----------------
            const int z = q - 1;
            if (KIND == 2 && wb) {   // box sums of U(q) for the back task (window U(z-1), U(z), U(q))
                bb_m = bb_0;
                bb_0 = bb_p;
                bb_p = box9(U, ob);
            }
            if (wb && z >= it.zlo && z < it.zhi) {
                const double *Um = su + ((z - 1 + 8) % NU) * PS, *U0 = su + ((z + 8) % NU) * PS;
                const double2 c = lds2(U0 + ob);
                double2 Ap;
                if (KIND == 2) {
                    Ap.x = 27.0 * c.x - (bb_m.x + bb_0.x + bb_p.x);
                    Ap.y = 27.0 * c.y - (bb_m.y + bb_0.y + bb_p.y);
                } else {
                    const double2 dn = lds2(Um + ob), up = lds2(U + ob);
                    const double2 ylo = lds2(U0 + ob - BW), yhi = lds2(U0 + ob + BW);
                    const double l = U0[ob - 1], rr = U0[ob + 2];
                    Ap.x = center * c.x - K1F_SUM6(dn.x, up.x, ylo.x, yhi.x, l, c.y);
                    Ap.y = center * c.y - K1F_SUM6(dn.y, up.y, ylo.y, yhi.y, c.x, rr);
                }
                if (!v1b) Ap.y = 0.0;
                const int64_t i = (int64_t)z * pl + gib;
                if (!a.skip_w2) __stcs(reinterpret_cast<double2 *>(a.w2 + i), Ap);
                if (wk.back_pn) {
                    const double2 pj = lds2(sp + ((cq - 1) % NSP) * PS + ob);   // p_j(z)
                    const double v0 = cbk * (dinv_c * Ap.x - sigma * c.x) - pj.x;
                    double v1 = cbk * (dinv_c * Ap.y - sigma * c.y) - pj.y;
                    if (!v1b) v1 = 0.0;
                    *reinterpret_cast<double2 *>(a.pn2 + i) = make_double2(v0, v1);
                }
            }
            // p_j plane q-1 is no longer needed (front(q+1) reads q..q+2)
            if (q - 1 >= it.plo) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&emptyp[(cq - 1) % NSP]);
            }
        }
        // release the p_j planes of this item not released in the loop: zhi, zhi+1 (if loaded)
        for (int z = max(it.zhi, it.plo); z <= it.phi; ++z) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&emptyp[(pbase + (z - it.plo)) % NSP]);
        }
        pc = pbase + (it.phi - it.plo + 1);
    }
    }   // KIND != 1
}

}  // namespace

bool k1f_prepare(const Geo &g, const double *P, int nzl, int s, CUtensorMap *tmP, CUtensorMap *tmM)
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
    return cudaFuncSetAttribute(k1f<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) == cudaSuccess &&
           cudaFuncSetAttribute(k1f<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) == cudaSuccess;
}

// SSCG_K1_FUSE (read at every sscg_setup): "0" never, "1" always (7/27-point),
// unset: 7-point slabs with at least K1F_MIN_WORK tile-planes per SM.  Since
// the register-column K1F (z-columns in registers, per-thread mbarriers) the
// fused pair beats two K1T steps down to cfg 2 (128^3: 0.243 vs 0.263 ms per
// outer, profiles/r01r_*); the 27-point pair is bound by its in-plane box sums
// and gains nothing over two K1T steps (profiles/r01g_workloads.jsonl).
constexpr int64_t K1F_MIN_WORK = 8;

bool k1f_enabled(const Geo &g, int nzl)
{
    if (g.kn.k1_fuse == 0) return false;
    if (g.kn.k1_fuse == 1) return true;
    const int64_t tiles = (int64_t)((g.nx + TX - 1) / TX) * ((g.ny + TY - 1) / TY);
    return g.kind == 1 && tiles * nzl >= K1F_MIN_WORK * k2_grid();
}

// steps j and j+1 over the planes [a.zb, a.ze) of one slab (a.p = p_j, a.pm =
// p_{j-1} or null, a.w = w_j, a.pn = p_{j+1}, a.w2 = w_{j+1}, a.pn2 = p_{j+2}
// or null).  The halo planes of p_j must be current.  With [1, nzl+1) the
// slab is treated as bounded by Dirichlet planes in z (p_{j+1} = 0 outside),
// so a slab with neighbours passes [2, nzl) and runs its boundary planes with
// single steps around the exchange of p_{j+1}.
void launch_k1f(const Geo &g, const K1Args &a, double theta, int s, const DevState *st, cudaStream_t strm)
{
    K1FWork wk;
    wk.tiles_x = (g.nx + TX - 1) / TX;
    wk.tiles_y = (g.ny + TY - 1) / TY;
    wk.nzl = a.nzl;
    wk.zb = a.zb;
    wk.ze = a.ze;
    wk.j = a.j;
    wk.front_pm = a.j > 0;
    wk.back_pn = (a.j + 1 < s - 1) ? 1 : 0;
    wk.coef_front = (a.j == 0) ? theta : 2.0 * theta;
    wk.coef_back = 2.0 * theta;
    wk.sigma = a.sigma;
    wk.center = g.center;
    wk.dinv_c = g.dinv_c;
    const int64_t tiles = (int64_t)wk.tiles_x * wk.tiles_y;
    // one CTA per SM (fewer with a.sm_cap: SMs left to the overlapped NCCL exchange)
    const int64_t resident = (int64_t)MINB * ((a.sm_cap > 0 && a.sm_cap < k2_grid()) ? a.sm_cap : k2_grid());
    const int zc_env = g.kn.k1_zc;
    const int n1 = a.ze - a.zb;
    if (n1 <= 0) return;
    int zc = n1;
    if (zc_env > 0) {
        zc = std::min(n1, zc_env);
    } else {
        // few long chunks (each re-reads 4 planes of p_j and recomputes 2
        // front planes), tiles x chunks filling whole waves of the grid
        double best = -1.0;
        for (int nch = 1; nch <= 64 && (n1 + nch - 1) / nch >= 4; ++nch) {
            const int z = (n1 + nch - 1) / nch;
            const int64_t items = tiles * ((n1 + z - 1) / z);   // chunks actually formed with this z
            const int64_t waves = (items + resident - 1) / resident;
            const double score = (double)items / (double)(waves * resident) / (1.0 + 1.0 / z);
            if (score > best + 1e-9) {
                best = score;
                zc = z;
            }
        }
    }
    wk.zc = zc;
    wk.nitems = tiles * ((n1 + zc - 1) / zc);
    const unsigned grid = (unsigned)std::min<int64_t>(wk.nitems, resident);
    if (g.kind == 2) launch_pdl(g.kn.pdl, k1f<2>, dim3(grid), dim3(THREADS), SMEM, strm, *a.tmF_P, *a.tmF_M, g, a, st, wk);
    else launch_pdl(g.kn.pdl, k1f<1>, dim3(grid), dim3(THREADS), SMEM, strm, *a.tmF_P, *a.tmF_M, g, a, st, wk);
}

}  // namespace sscg
