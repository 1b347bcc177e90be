// K1M -- three basis steps in one pass (7-point): steps j, j+1, j+2 of the
// Chebyshev recurrence
//   w_j = A p_j,  p_{j+1} = c_j (D^{-1} w_j - sigma p_j) [- p_{j-1}],
// and the same for j+1 and j+2, with p_{j+1} and p_{j+2} kept on chip
// (matrix-powers blocking of depth 3).  Per triple it
// streams p_j and p_{j-1} in and p_{j+1}, p_{j+2}, p_{j+3} out (w only where
// the schedule stores it): 5 vectors for three steps instead of 6 for a K1F
// pair plus half of the next one.
//
// Same per-point arithmetic as K1T/K1F, with the six neighbour terms of A p
// summed as a tree (K1M_TREE) rather than left to right.  Level l = 1..3
// computes step j+l-1 on the tile (56 x 16) plus a (3-l)-cell halo in y and a
// 2(3-l)-cell halo in x (x work is done in pairs of cells); p_j is staged by
// TMA with a 3-cell y / 6-cell x halo.  Cells outside the grid are forced to
// the Dirichlet value 0, planes outside [1, nzl] likewise.
//
// Thread map: consumer warp r (1..20) owns box row r, lane l the cell pair
// at box column 2 + 2l -- every thread computes all the levels its cell
// belongs to, so the z-columns p_j(q-1..q+1), p_{j+1}(q-2..q) and
// p_{j+2}(q-3..q-1) of its own cell roll through registers; only in-plane
// neighbours come from shared memory (rings U1, U2 of the level-1/2
// outputs).  Plane q of the march runs level 1 at q, level 2 at q-1, level 3
// at q-2.  U1/U2 planes are published through per-plane mbarriers (every
// consumer thread arrives -- one elected lane per warp after __syncwarp measured
// 0.69-0.70 vs 0.65 ms per launch); with 4 slots per ring a thread that waited for
// U1(q-2) / U2(q-3) knows every read of the slot it overwrites is done.
// Measured and not kept: waiting only for the two neighbour rows a warp reads
// (per-row mbarriers per ring slot: 0.795 vs 0.743 ms per triple; spinning on
// acquire loads of per-row plane counters: 1.18 ms) -- the CTA-wide plane
// barrier keeps the rows in lockstep, which the shared stage ring relies on;
// a 56 x 20 tile (24 row warps, 5 stages, 3 U slots; K1M_TY=20): 0.722 vs 0.743
// ms per triple in the profiled pass, within box noise on the whole step; two
// box rows per warp (10 warps, the pair's inner y-neighbours from registers at
// every level: ~20 % fewer consumer shared-memory wavefronts, parity green):
// 0.764 vs 0.741 ms -- half the warps hide less latency than the wavefronts save;
// the x-neighbours from the neighbouring lanes by shuffles instead of shared
// memory (64-bit shuffles through the same MIO path): 0.837 vs 0.744 ms.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "sscg_internal.cuh"
#include "tma.cuh"

namespace sscg {
namespace {

#ifndef K1M_TY
#define K1M_TY 16
#endif
constexpr int TX = 56, TY = K1M_TY;
constexpr int BW = TX + 12;    // p_j box: x in [x0-6, x0+TX+6)  (68)
constexpr int BHP = TY + 6;    // p_j box: y in [y0-3, y0+TY+3)  (22)
constexpr int MW = TX + 8;     // p_{j-1} box: x in [x0-4, x0+TX+4) (64), the level-1 cells
constexpr int MH = TY + 4;     // y in [y0-2, y0+TY+2) (20)
constexpr int U1H = TY + 4;    // level-1 rows 1..TY+4 of the p_j box, pitch BW
constexpr int U2H = TY + 2;    // level-2 rows 2..TY+3
constexpr int r128(int d) { return ((d * 8 + 127) / 128) * 128 / 8; }
constexpr int PS = r128(BW * BHP), MS = r128(MW * MH), U1S = r128(BW * U1H), U2S = r128(BW * U2H);
constexpr int STG = PS + MS;              // one stage: p_j(z) and p_{j-1}(z-1), one barrier
#ifndef K1M_NST
#define K1M_NST 6
#endif
#ifndef K1M_NU
#define K1M_NU 4
#endif
// stages: slot = seq % NST.  U rings: one barrier per plane orders every
// access of plane n-1 before any of plane n+1 (a thread arrives for plane n
// only after finishing it), so 3 slots would suffice; measured 6 stages / 4 U
// slots 0.641 ms per launch, 7 / 3 0.656, 6 / 3 0.646
constexpr int NST = K1M_NST, NU = K1M_NU;
constexpr int NCW = TY + 4;               // one consumer warp per level-1 row
constexpr int NCT = NCW * 32;
constexpr int THREADS = NCT + 32;
constexpr uint32_t PBYTES = BW * BHP * 8, MBYTES = MW * MH * 8;
constexpr size_t SMEM = (size_t)(NST * STG + NU * U1S + NU * U2S) * sizeof(double);
static_assert(SMEM <= 227 * 1024, "shared memory");
static_assert(BW / 2 - 2 == 32, "one lane per level-1 pair");

struct K1MWork {
    int tiles_x, tiles_y, zc;
    int64_t nitems;
    int nzl;
    // up to two level-3 plane ranges per launch (the boundary launch of the deep
    // halo schedule covers both ends of the slab): write range of each level,
    // level 3's range the one chunked; range 1 is empty when nch[1] == 0
    int zb[2][3], ze[2][3];
    int nch0;              // chunks of range 0 (items: tiles x (nch0 + chunks of range 1))
    // planes where level 1 / level 2 are formed (outside: the Dirichlet value 0):
    // [1, nzl] against the global boundary, extended by 2 / 1 ghost planes on a
    // side whose 3-plane halo of p_j (and 2 planes of p_{j-1}) is current
    // (deep halos)
    int lo1, hi1, lo2, hi2;
    int zoff;              // tensor-map plane coordinate of plane 0 (2 with guard planes)
    int j;                 // vector coordinate of p_j in the tensor maps
    int front_pm;          // level 1 subtracts p_{j-1} (j >= 1)
    double coef1, coef, sigma, center, dinv_c;
};

struct Outs {
    double *w[3], *pn[3];  // null: not stored
    // peer-store halos: p_{j+2}, p_{j+3} of the neighbour below / above, offset so
    // that own offset + pointer is the neighbour's ghost cell (null: none)
    double *lo[2], *hi[2];
    int sys_fence;   // the peer stores go to another process's memory (CUDA IPC over NVLink)
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

#ifndef K1M_PN_STCS
#define K1M_PN_STCS 0
#endif
// store of a p_{j+l} pair (K1M_PN_STCS: evict-first)
__device__ __forceinline__ void st_pn(double *p, double2 v)
{
#if K1M_PN_STCS
    __stcs(reinterpret_cast<double2 *>(p), v);
#else
    *reinterpret_cast<double2 *>(p) = v;
#endif
}

struct ItemPlan {
    int tx, ty, zlo, zhi;      // level-3 planes [zlo, zhi)
    int r;                     // plane range of the launch
    int q0, q1;                // march: level-1 planes q0..q1
    int plo, phi, mlo, mhi;    // p_j / p_{j-1} planes loaded
    int first, last;           // first / last chunk (levels 1, 2 write their range's ends)
};

__device__ __forceinline__ ItemPlan plan_item(const K1MWork &wk, int64_t item)
{
    const int ntiles = wk.tiles_x * wk.tiles_y;
    const int chunk = (int)(item / ntiles);
    const int tile = (int)(item - (int64_t)chunk * ntiles);
    ItemPlan p;
    p.ty = tile / wk.tiles_x;
    p.tx = tile - p.ty * wk.tiles_x;
    p.r = chunk >= wk.nch0;
    const int c = chunk - (p.r ? wk.nch0 : 0);
    p.zlo = wk.zb[p.r][2] + c * wk.zc;
    p.zhi = min(wk.ze[p.r][2], p.zlo + wk.zc);
    p.first = p.zlo == wk.zb[p.r][2];
    p.last = p.zhi == wk.ze[p.r][2];
    p.q0 = max(p.zlo - 2, wk.lo1 - 1);
    p.q1 = p.zhi + 1;   // level 3 reaches zhi - 1 at q = zhi + 1 (level 1 is outside past hi1)
    p.plo = max(p.q0 - 1, wk.lo1 - 1);
    p.phi = min(p.q1 + 1, wk.hi1 + 1);
    p.mlo = max(p.q0, wk.lo1);
    p.mhi = min(p.q1, wk.hi1);
    return p;
}

// K1M_TREE: the six neighbour terms summed as a tree (depth 3) instead of a
// chain (depth 5); rounds differently from K1T/K1F in the last bits (within
// the parity tolerances), measured 0.632-0.641 vs 0.652-0.653 ms per launch.
// Folding the recurrence as fma(c D^{-1}, A p, fma(-c sigma, p, -p_prev)) (one
// FMA after A p instead of three operations) measured slower: 0.68 vs 0.64 ms
#ifndef K1M_TREE
#define K1M_TREE 1
#endif

// 7-point A p on the pair at smem offset o of plane P0, own z-neighbours given
__device__ __forceinline__ double2 stencil(const double *P0, int o, double2 c, double2 dn, double2 up, double center)
{
    const double2 ylo = lds2(P0 + o - BW), yhi = lds2(P0 + o + BW);
    const double l = P0[o - 1], rr = P0[o + 2];
    double2 Ap;
#if K1M_TREE
    Ap.x = center * c.x - (((dn.x + up.x) + (ylo.x + yhi.x)) + (l + c.y));
    Ap.y = center * c.y - (((dn.y + up.y) + (ylo.y + yhi.y)) + (c.x + rr));
#else
    Ap.x = center * c.x - (dn.x + ylo.x + l + c.y + yhi.x + up.x);
    Ap.y = center * c.y - (dn.y + ylo.y + c.x + rr + yhi.y + up.y);
#endif
    return Ap;
}

#ifndef K1M_EO
#define K1M_EO 1
#endif
// U rings in even/odd-split rows: cell 2k of a row at [k], cell 2k+1 at [HW + k],
// so the x-neighbour of a pair is a contiguous 8-B load across the warp (two
// wavefronts) instead of a 16-B-strided one (four): ~12 % fewer shared
// wavefronts per plane, measured 0.654-0.658 vs 0.659-0.662 ms per launch
// (K1M_EO=0: interleaved pairs)
constexpr int HW = BW / 2;
__device__ __forceinline__ double2 stencil_eo(const double *U, int oe, double2 c, double2 dn, double2 up,
                                              double center)
{
    const double ylx = U[oe - BW], yly = U[oe - BW + HW], yhx = U[oe + BW], yhy = U[oe + BW + HW];
    const double l = U[oe + HW - 1], rr = U[oe + 1];
    double2 Ap;
#if K1M_TREE
    Ap.x = center * c.x - (((dn.x + up.x) + (ylx + yhx)) + (l + c.y));
    Ap.y = center * c.y - (((dn.y + up.y) + (yly + yhy)) + (c.x + rr));
#else
    Ap.x = center * c.x - (dn.x + ylx + l + c.y + yhx + up.x);
    Ap.y = center * c.y - (dn.y + yly + c.x + rr + yhy + up.y);
#endif
    return Ap;
}

__device__ __forceinline__ void st_u(double *U, int o, int oe, double2 v)
{
#if K1M_EO
    U[oe] = v.x;
    U[oe + HW] = v.y;
#else
    *reinterpret_cast<double2 *>(U + o) = v;
#endif
}

// HASW: some level stores w (the stored-W schedule, or a triple that ends at
// step s-1); HASN2: level 3 stores p_{j+3} (j+3 <= s-1).  p_{j+1} and p_{j+2}
// are always stored.  Compile-time, so the common W-free triple carries no
// per-plane tests of the output pointers.
template <bool HASW, bool HASN2>
__global__ void __launch_bounds__(THREADS, 1)
    k1m(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmM, Geo g, Outs out,
        const DevState *st, K1MWork wk)
{
    PDL_ENTRY(st);
    extern __shared__ __align__(128) double smem[];
    double *sstg = smem;                 // stages: [p_j(z) box | p_{j-1}(z-1) box]
    double *su1 = sstg + NST * STG;      // level-1 outputs (p_{j+1})
    double *su2 = su1 + NU * U1S;        // level-2 outputs (p_{j+2})
    __shared__ uint64_t full[NST], empty[NST], ubar[NU];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NCT);
        }
        for (int i = 0; i < NU; ++i) mbar_init(&ubar[i], NCT);
        mbar_fence_init();
        tma_prefetch_desc(&tmP);
        tma_prefetch_desc(&tmM);
    }
    __syncthreads();

    if (warp == 0) {   // producer: stage z = p_j(z) [+ p_{j-1}(z-1)], z = plo..phi, in march order
        if (lane == 0) {
            uint32_t sc = 0;
            for (int64_t item = blockIdx.x; item < wk.nitems; item += gridDim.x) {
                const ItemPlan it = plan_item(wk, item);
                const int x0 = it.tx * TX, y0 = it.ty * TY;
                for (int z = it.plo; z <= it.phi; ++z, ++sc) {
                    const int sl = sc % NST;
                    if (sc >= NST) mbar_wait(&empty[sl], ((sc / NST) - 1) & 1);
                    const bool m = wk.front_pm && z - 1 >= it.mlo && z - 1 <= it.mhi;
                    mbar_expect_tx(&full[sl], PBYTES + (m ? MBYTES : 0u));
                    tma_load_4d(sstg + sl * STG, &tmP, x0 - 6, y0 - 3, z + wk.zoff, wk.j, &full[sl]);
                    if (m)
                        tma_load_4d(sstg + sl * STG + PS, &tmM, x0 - 4, y0 - 2, z - 1 + wk.zoff, wk.j - 1, &full[sl]);
                }
            }
        }
        return;
    }

    const int rk = warp, ck = 2 + 2 * lane;                  // box row 1..20, column 2..64
    const int ok = rk * BW + ck;                             // p_j offset in a stage
    const int omk = PS + (rk - 1) * MW + (ck - 2);           // p_{j-1} offset in a stage
    const int o1 = (rk - 1) * BW + ck;                       // U1 offset (rows from 1)
    const int o2 = (rk - 2) * BW + ck;                       // U2 offset (rows from 2)
    const int oe1 = (rk - 1) * BW + 1 + lane, oe2 = (rk - 2) * BW + 1 + lane;   // the same, even/odd split
    const bool in2 = rk >= 2 && rk <= TY + 3 && lane >= 1 && lane <= 30;   // level-2 cell
    const bool in3 = rk >= 3 && rk <= TY + 2 && lane >= 2 && lane <= 29;   // level 3 = the tile
    const bool front_pm = wk.front_pm;
    const int lo1 = wk.lo1, hi1 = wk.hi1, lo2 = wk.lo2, hi2 = wk.hi2;
    const double center = wk.center, dinv_c = wk.dinv_c, sigma = wk.sigma, cf1 = wk.coef1, cf = wk.coef;
    double *const w0 = out.w[0], *const w1 = out.w[1], *const w2 = out.w[2];
    double *const n0 = out.pn[0], *const n1 = out.pn[1], *const n2 = out.pn[2];
    const int64_t pl = g.plane;
    const uint32_t full_a = pin_u32(smem_u32(full)), empty_a = pin_u32(smem_u32(empty)),
                   ubar_a = pin_u32(smem_u32(ubar));
    uint32_t sc = 0, uc = 0;   // stage / U sequence numbers
    for (int64_t item = blockIdx.x; item < wk.nitems; item += gridDim.x) {
        const ItemPlan it = plan_item(wk, item);
        const int x0 = it.tx * TX, y0 = it.ty * TY;
        const int gx = x0 - 6 + ck, gy = y0 - 3 + rk;
        const bool vy = gy >= 0 && gy < g.ny;
        const bool v0 = vy && gx >= 0 && gx < g.nx, v1 = vy && gx + 1 >= 0 && gx + 1 < g.nx;
        const bool own = in3 && v0;   // the tile's own cell: outputs go to HBM
        const int wb1 = it.first ? wk.zb[it.r][0] : it.zlo, we1 = it.last ? wk.ze[it.r][0] : it.zhi;
        const int wb2 = it.first ? wk.zb[it.r][1] : it.zlo, we2 = it.last ? wk.ze[it.r][1] : it.zhi;
        // stage slots and phases are recomputed from sequence numbers per plane;
        // rolling them plane by plane (no division by NST) cost registers (28 B
        // of spill) and measured 0.70 vs 0.655 ms per launch
        const uint32_t sbase = sc;   // sequence number of stage plo
        auto stg = [&](int z) -> const double * {
            return sstg + ((sbase + (uint32_t)(z - it.plo)) % NST) * STG;
        };
        auto release = [&](int z) { mbar_arrive_a(empty_a + 8 * ((sbase + (uint32_t)(z - it.plo)) % NST)); };
        auto waits = [&](int z) {
            const uint32_t c = sbase + (uint32_t)(z - it.plo);
            mbar_wait_a(full_a + 8 * (c % NST), (c / NST) & 1);
        };
        for (int z = it.plo; z <= min(it.q0, it.phi); ++z) waits(z);
        double2 pdn = make_double2(0.0, 0.0);     // p_j(q-1), own cell
        if (it.q0 - 1 >= it.plo) {
            pdn = lds2(stg(it.q0 - 1) + ok);
            release(it.q0 - 1);
        }
        double2 pc0 = lds2(stg(it.q0) + ok);     // p_j(q)
        double2 u1m2 = make_double2(0.0, 0.0), u1m1 = make_double2(0.0, 0.0);   // p_{j+1}(q-2), (q-1)
        double2 u2m2 = make_double2(0.0, 0.0), u2m1 = make_double2(0.0, 0.0);   // p_{j+2}(q-3), (q-2)
        int64_t off = (int64_t)it.q0 * pl + (int64_t)gy * g.pitch + gx;   // global index, plane q
        // one plane of the march; S: zlo + 2 <= q < zhi, where every plane
        // condition below is known to hold
        auto plane = [&](int q, auto steady) {
            constexpr bool S = decltype(steady)::value;
            // ---------------- level 1: step j at plane q ----------------
            const bool inside1 = S || (q >= lo1 && q <= hi1);
            const bool has_up = S || q + 1 <= it.phi;
            const double *P0 = stg(q), *P1 = stg(q + 1);
            double2 pup = make_double2(0.0, 0.0);   // p_j(q+1)
            if (has_up) {
                waits(q + 1);
                pup = lds2(P1 + ok);
            }
            const bool mloaded = front_pm && (S || (q >= it.mlo && q <= it.mhi));
            double2 u1 = make_double2(0.0, 0.0);
            if (inside1) {
                const double2 c = pc0;
                double2 Ap = stencil(P0, ok, c, pdn, pup, center);
                u1.x = cf1 * (dinv_c * Ap.x - sigma * c.x);
                u1.y = cf1 * (dinv_c * Ap.y - sigma * c.y);
                if (mloaded) {
                    const double2 pm = lds2(P1 + omk);   // p_{j-1}(q) rides in stage q+1
                    u1.x -= pm.x;
                    u1.y -= pm.y;
                }
                if (!v0) u1.x = 0.0;
                if (!v1) u1.y = 0.0;
                if (own && (S || (q >= wb1 && q < we1))) {
                    if (!v1) Ap.y = 0.0;
                    if (HASW && w0) __stcs(reinterpret_cast<double2 *>(w0 + off), Ap);
                    st_pn(n0 + off, u1);
                }
            }
            st_u(su1 + (uc % NU) * U1S, o1, oe1, u1);
            if (S || (q >= it.plo && q <= it.phi)) release(q);
            // one barrier per plane: U1(q-1) and U2(q-2) of every thread are written
            if (S || uc > 0) mbar_wait_a(ubar_a + 8 * ((uc - 1) % NU), ((uc - 1) / NU) & 1);
            // ---------------- level 2: step j+1 at plane q-1 ----------------
            const int z2 = q - 1;
            double2 u2 = make_double2(0.0, 0.0);
            if (in2 && (S || (z2 >= lo2 && z2 <= hi2))) {
                const double *U = su1 + ((uc - 1) % NU) * U1S;
                const double2 c = u1m1;
#if K1M_EO
                double2 Ap = stencil_eo(U, oe1, c, u1m2, u1, center);
#else
                double2 Ap = stencil(U, o1, c, u1m2, u1, center);
#endif
                u2.x = cf * (dinv_c * Ap.x - sigma * c.x) - pdn.x;   // pdn = p_j(q-1)
                u2.y = cf * (dinv_c * Ap.y - sigma * c.y) - pdn.y;
                if (!v0) u2.x = 0.0;
                if (!v1) u2.y = 0.0;
                if (own && (S || (z2 >= wb2 && z2 < we2))) {
                    if (!v1) Ap.y = 0.0;
                    if (HASW && w1) __stcs(reinterpret_cast<double2 *>(w1 + off - pl), Ap);
                    st_pn(n1 + off - pl, u2);
                    if (!S) {   // peer-store halo (the steady range excludes these planes)
                        if (out.lo[0] && z2 <= 2) st_pn(out.lo[0] + off - pl, u2);
                        if (out.hi[0] && z2 >= wk.nzl - 1) st_pn(out.hi[0] + off - pl, u2);
                    }
                }
            }
            if (in2) st_u(su2 + ((uc - 1) % NU) * U2S, o2, oe2, u2);
            // ---------------- level 3: step j+2 at plane q-2 ----------------
            const int z3 = q - 2;
            if (own && (S || (z3 >= it.zlo && z3 < it.zhi))) {
                const double *U = su2 + ((uc - 2) % NU) * U2S;
                const double2 c = u2m1;
#if K1M_EO
                double2 Ap = stencil_eo(U, oe2, c, u2m2, u2, center);
#else
                double2 Ap = stencil(U, o2, c, u2m2, u2, center);
#endif
                if (!v1) Ap.y = 0.0;
                if (HASW && w2) __stcs(reinterpret_cast<double2 *>(w2 + off - 2 * pl), Ap);
                if (HASN2) {
                    const double v0b = cf * (dinv_c * Ap.x - sigma * c.x) - u1m2.x;   // u1m2 = p_{j+1}(q-2)
                    double v1b = cf * (dinv_c * Ap.y - sigma * c.y) - u1m2.y;
                    if (!v1) v1b = 0.0;
                    st_pn(n2 + off - 2 * pl, make_double2(v0b, v1b));
                    if (!S) {
                        if (out.lo[1] && z3 <= 3) st_pn(out.lo[1] + off - 2 * pl, make_double2(v0b, v1b));
                        if (out.hi[1] && z3 >= wk.nzl - 2) st_pn(out.hi[1] + off - 2 * pl, make_double2(v0b, v1b));
                    }
                }
            }
            mbar_arrive_a(ubar_a + 8 * (uc % NU));   // this thread's U1(q), U2(q-1) are written
            ++uc;
            u2m2 = u2m1;
            u2m1 = u2;
            u1m2 = u1m1;
            u1m1 = u1;
            pdn = pc0;
            pc0 = pup;
            off += pl;
        };
        using Gen = std::integral_constant<bool, false>;
        using Steady = std::integral_constant<bool, true>;
        // steady planes [qs, qe): with peer stores, level 2 / 3 planes the
        // neighbours take (1..3, nzl-2..nzl) run in the general form
        const int qs = out.lo[0] ? max(it.zlo + 2, 6) : it.zlo + 2;
        const int qe = out.hi[0] ? min(it.zhi, wk.nzl) : it.zhi;
        int q = it.q0;
        for (; q < qs && q <= it.q1; ++q) plane(q, Gen());
#pragma unroll 1
        for (; q < qe; ++q) plane(q, Steady());
        for (; q <= it.q1; ++q) plane(q, Gen());
        for (int z = max(it.q1 + 1, it.plo); z <= it.phi; ++z) release(z);
        sc = sbase + (it.phi - it.plo + 1);
    }
    // stores into another rank's ghost planes are performed system-wide before
    // this thread exits: the token the stream sends after the kernel (the
    // ordering step of the cross-rank peer-store halo) then follows them
    if (out.sys_fence) __threadfence_system();
}

}  // namespace

// TMA L2 promotion of the p_j / p_{j-1} boxes; 128 B or none measured the same
// as 256 B (0.652-0.655 vs 0.656-0.660 ms per launch, within box noise), as
// did evict-first stores of p_{j+l} (K1M_PN_STCS: 0.660-0.664 ms)
#ifndef K1M_L2P
#define K1M_L2P CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif

// guard: planes allocated below plane 0 (and above nzl+1) of every vector --
// the deep halo's ghost planes; the maps then start `guard` planes early
bool k1m_prepare(const Geo &g, const double *P, int nzl, int s, CUtensorMap *tmP, CUtensorMap *tmM, int guard)
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
    cuuint64_t dims[4] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)(nzl + 2 + 2 * guard), (cuuint64_t)s};
    cuuint64_t strides[3] = {(cuuint64_t)g.pitch * 8, (cuuint64_t)g.plane * 8, (cuuint64_t)g.vstride * 8};
    cuuint32_t es[4] = {1, 1, 1, 1};
    cuuint32_t boxp[4] = {BW, BHP, 1, 1}, boxm[4] = {MW, MH, 1, 1};
    P -= (int64_t)guard * g.plane;
    if (enc(tmP, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double *>(P), dims, strides, boxp, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, K1M_L2P,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (enc(tmM, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double *>(P), dims, strides, boxm, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, K1M_L2P,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    return cudaFuncSetAttribute(k1m<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) == cudaSuccess &&
           cudaFuncSetAttribute(k1m<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) == cudaSuccess &&
           cudaFuncSetAttribute(k1m<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) == cudaSuccess &&
           cudaFuncSetAttribute(k1m<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM) == cudaSuccess;
}

// SSCG_K1_MP3 (read at every sscg_setup): "1" / "0" force / forbid the
// triples; unset: 7-point slabs with at least 64 tile-planes per SM (cfg 2,
// 128^3 with ~21, runs faster with K1F pairs: 0.234 vs 0.267 ms per outer).
// Measured at cfg 5: 8.06-8.12 ms per outer with triples against 8.36-8.39
// with K1F pairs.  The first version (separate p_j / p_{j-1} rings, two
// barriers per plane) took 1.006 ms per triple and was issue-bound
// (profiles/r01s_*); p_{j-1} riding in the p_j stage, one barrier per plane, a
// compile-time steady state and a 6-stage ring (4 stages left two planes of
// prefetch) brought it to ~0.70 ms.
bool k1m_enabled(const Geo &g, int nzl)
{
    if (g.kind != 1) return false;
    if (g.kn.k1_mp3 >= 0) return g.kn.k1_mp3 == 1;
    if (g.kn.k1_fuse == 0) return false;   // SSCG_K1_FUSE=0: no fused basis kernels at all
    const int64_t tiles = (int64_t)((g.nx + TX - 1) / TX) * ((g.ny + TY - 1) / TY);
    return tiles * nzl >= 64 * k2_grid();
}

// steps j, j+1, j+2 of one slab.  a.zb[l] / a.ze[l]: planes level l writes
// (level 3's range is split into z-chunks; levels 1 and 2 may extend it at
// either end by up to 2 / 1 planes).  The tensor maps view P with the vector
// index as the 4th coordinate, so one pair of maps serves every j.
void launch_k1m(const Geo &g, const K1MArgs &a, double theta, const DevState *st, cudaStream_t strm)
{
    K1MWork wk;
    wk.tiles_x = (g.nx + TX - 1) / TX;
    wk.tiles_y = (g.ny + TY - 1) / TY;
    wk.nzl = a.nzl;
    for (int l = 0; l < 3; ++l) {
        wk.zb[0][l] = a.zb[l];
        wk.ze[0][l] = a.ze[l];
        wk.zb[1][l] = a.zb2[l];
        wk.ze[1][l] = a.ze2[l];
    }
    wk.lo1 = a.deep_lo ? -1 : 1;
    wk.lo2 = a.deep_lo ? 0 : 1;
    wk.hi1 = a.deep_hi ? a.nzl + 2 : a.nzl;
    wk.hi2 = a.deep_hi ? a.nzl + 1 : a.nzl;
    wk.zoff = a.guard;
    wk.j = a.j;
    wk.front_pm = a.j > 0;
    wk.coef1 = (a.j == 0) ? theta : 2.0 * theta;
    wk.coef = 2.0 * theta;
    wk.sigma = a.sigma;
    wk.center = g.center;
    wk.dinv_c = g.dinv_c;
    Outs out;
    for (int l = 0; l < 3; ++l) {
        out.w[l] = a.w[l];
        out.pn[l] = a.pn[l];
    }
    // peer-store halos: own plane z -> plane nzl_lo + z of the slab below,
    // plane z - nzl of the slab above (p_{j+3} only when this triple forms it)
    for (int l = 0; l < 2; ++l) {
        const bool formed = l == 0 || a.pn[2];
        out.lo[l] = (formed && a.peer_lo[l]) ? a.peer_lo[l] + (int64_t)a.peer_nzl_lo * g.plane : nullptr;
        out.hi[l] = (formed && a.peer_hi[l]) ? a.peer_hi[l] - (int64_t)a.nzl * g.plane : nullptr;
    }
    out.sys_fence = a.peer_sys_fence;
    if (!out.lo[0]) out.lo[1] = nullptr;   // the kernel keys the steady range on level 2's pointer
    if (!out.hi[0]) out.hi[1] = nullptr;
    const int64_t tiles = (int64_t)wk.tiles_x * wk.tiles_y;
    const int64_t resident = (a.sm_cap > 0 && a.sm_cap < k2_grid()) ? a.sm_cap : k2_grid();
    const int zc_env = g.kn.k1_zc;
    const int n1 = std::max(0, a.ze[2] - a.zb[2]), n2 = std::max(0, a.ze2[2] - a.zb2[2]);
    if (n1 <= 0) return;
    int zc = n1;
    if (zc_env > 0) {
        zc = std::min(n1, zc_env);
    } else if (n2 > 0) {
        zc = std::max(n1, n2);   // boundary launch (deep halos): one chunk per range
    } else {
        // each chunk re-reads 5 planes of p_j and recomputes 4 level-1/2 planes:
        // few long chunks, tiles x chunks filling whole waves
        double best = -1.0;
        for (int nch = 1; nch <= 64 && (n1 + nch - 1) / nch >= 6; ++nch) {
            const int z = (n1 + nch - 1) / nch;
            const int64_t items = tiles * ((n1 + z - 1) / z);
            const int64_t waves = (items + resident - 1) / resident;
            const double score = (double)items / (double)(waves * resident) / (1.0 + 2.0 / z);
            if (score > best + 1e-9) {
                best = score;
                zc = z;
            }
        }
    }
    wk.zc = zc;
    wk.nch0 = (n1 + zc - 1) / zc;
    wk.nitems = tiles * (wk.nch0 + (n2 + zc - 1) / zc);
    const unsigned grid = (unsigned)std::min<int64_t>(wk.nitems, resident);
    // p_{j+1} and p_{j+2} always exist in a triple (j + 2 <= s - 1)
    const bool hasw = out.w[0] || out.w[1] || out.w[2], hasn2 = out.pn[2] != nullptr;
    auto kern = hasw ? (hasn2 ? k1m<true, true> : k1m<true, false>) : (hasn2 ? k1m<false, true> : k1m<false, false>);
    launch_pdl(g.kn.pdl, kern, dim3(grid), dim3(THREADS), SMEM, strm, *a.tmP, *a.tmM, g, out, st, wk);
}

}  // namespace sscg
