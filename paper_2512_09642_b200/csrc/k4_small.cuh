// K4 for s <= 32: Ruhe scaling + nu Forward Gauss-Seidel sweeps + stopping
// test + history on ONE warp, as a device function run by
// the one-warp kernel k4_fgs_warp (k_fgs_update.cu; tools/k4_probe.cu times
// it in isolation).
//
//   d_i = Ghat_ii^{-1/2};  G = S Ghat S with G_ii := 1;  c~ = S c
//   FGS sweep (I + L) a^(l+1) = c~ - L^T a^(l) in residual form: with
//   rho = c~ - G a (unit diagonal), coordinate j takes a_j += rho_j and every
//   row updates rho_i -= G_ij rho_j (for i = j this gives exactly 0 since
//   G_jj = 1) -- the forward substitution a_j = c~_j - sum_{i != j} G_ji a_i
//   of PAPER.md:94-97.  Lane i holds row i of G and rho_i.
//
// Coordinates go in blocks of four (NB4 = ceil(s/4) blocks, a template
// parameter; coordinates s..4*NB4-1 have G = 0 and c~ = 0, so their
// corrections are exactly 0 and change nothing): the block's four residual
// entries come over in four independent shuffles, every lane forms the
// block's corrections e_0..e_3 by forward substitution with the block's
// strictly lower entries (held by every lane), then applies them to its own
// rho_i -- the same FMAs in the same order as coordinate-by-coordinate FGS
// (bitwise equal), with a dependent chain per block of one shuffle round and
// four FMAs instead of four of each.  tools/k4_probe.cu (one call, in-kernel
// clock): s = 16, nu = 25 ~13k cycles, ~89 per block of four coordinates
// (DFMA latency 8 cycles, profiles/r02a_lat_probe.txt).  Forming the next
// block's residual entries redundantly in every lane (no shuffle on the
// chain, 26 instead of 10 FMAs per block) measured slower (~100 per block:
// the single warp is then FP64-issue-bound).
#pragma once
#include "sscg_internal.cuh"

namespace sscg {

__device__ __forceinline__ double k4_warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// scratch: >= s*s + s + 32 doubles of shared memory owned by this warp.
// STAGED: the caller has already put the block [Ghat | c] at scratch (KS, the
// single-CTA outer iteration, reduces it there); otherwise it is read from a.blk
template <int NB4, bool STAGED = false>
__device__ __forceinline__ void k4_fgs_small(const K4Args &a, DevState *st, double *scratch)
{
    constexpr int SP = 4 * NB4;
    const int s = a.s, lane = threadIdx.x & 31;
#ifdef K4_TIMING
    unsigned long long t00;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t00));
#endif
    // every input in flight at once: the device state (one struct copy) and the block
    const DevState S = *st;
    const int k = S.k;
    const int nent = s * s + s;
    double *Bs = scratch, *dsh = scratch + nent;
    if (!STAGED)
        for (int q = lane; q < nent; q += 32) Bs[q] = __ldcg(a.blk + q);
    __syncwarp();
    const bool rec = k < S.hist_cap, recg = k < S.gram_cap;
    if (recg)
        for (int q = lane; q < nent; q += 32) a.h_gram[(int64_t)k * nent + q] = Bs[q];
    const double *Gh = Bs, *c = Bs + s * s;

    const double rn = sqrt(a.rn2 ? __ldcg(a.rn2) : c[0]);
    const double r0 = (k == 0) ? rn : S.r0norm;
    if (lane == 0) {
        if (k == 0) st->r0norm = rn;
        if (rec) a.h_relres[k] = (r0 > 0.0) ? rn / r0 : 0.0;
    }
    if (!isfinite(rn)) {
        if (lane == 0) { st->nonfinite = 1; st->done = 1; st->outer = k; }
        return;
    }
    if (rn <= S.rtol * r0) {
        if (lane == 0) { st->converged = 1; st->done = 1; st->outer = k; }
        return;
    }
    if (k >= S.max_outer) {
        if (lane == 0) { st->done = 1; st->outer = k; }
        return;
    }
#ifdef K4_TIMING
    unsigned long long ta, tb, tc;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ta));
#endif
    // Ruhe scaling
    const bool v0 = lane < s;
    double d0 = 0.0;
    bool ok = true;
    if (v0) {
        const double gd = Gh[lane * s + lane];
        ok = (gd > 0.0) && isfinite(gd);
        d0 = 1.0 / sqrt(gd);
    }
    if (!__all_sync(0xffffffffu, ok)) {
        if (lane == 0) { st->breakdown = 1; st->done = 1; st->outer = k; }
        return;
    }
    dsh[lane] = v0 ? d0 : 0.0;
    __syncwarp();
    const double ct0 = v0 ? d0 * c[lane] : 0.0;
    double g[SP];
#pragma unroll
    for (int j = 0; j < SP; ++j)   // G_ij read as G_ji (the block is mirrored): lanes on consecutive banks
        g[j] = (v0 && j < s) ? ((j == lane) ? 1.0 : (d0 * Gh[j * s + lane]) * dsh[j]) : 0.0;
    double lnorm_part = 0.0;
#pragma unroll
    for (int j = 0; j < SP; ++j)
        if (j < lane) lnorm_part = fma(g[j], g[j], lnorm_part);
    // the block's strictly lower entries
    double Lb[NB4][6];
#pragma unroll
    for (int b = 0; b < NB4; ++b) {
        const int j = 4 * b;
        Lb[b][0] = __shfl_sync(0xffffffffu, g[j], j + 1);       // G_{j+1,j}
        Lb[b][1] = __shfl_sync(0xffffffffu, g[j], j + 2);       // G_{j+2,j}
        Lb[b][2] = __shfl_sync(0xffffffffu, g[j + 1], j + 2);   // G_{j+2,j+1}
        Lb[b][3] = __shfl_sync(0xffffffffu, g[j], j + 3);       // G_{j+3,j}
        Lb[b][4] = __shfl_sync(0xffffffffu, g[j + 1], j + 3);   // G_{j+3,j+1}
        Lb[b][5] = __shfl_sync(0xffffffffu, g[j + 2], j + 3);   // G_{j+3,j+2}
    }
    double rho = ct0, al0 = 0.0;
#ifdef K4_TIMING
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tb));
#endif
    for (int sw = 0; sw < a.nu; ++sw) {
#pragma unroll
        for (int b = 0; b < NB4; ++b) {
            const int j = 4 * b;
            const double r0b = __shfl_sync(0xffffffffu, rho, j), r1 = __shfl_sync(0xffffffffu, rho, j + 1),
                         r2 = __shfl_sync(0xffffffffu, rho, j + 2), r3 = __shfl_sync(0xffffffffu, rho, j + 3);
            const double e0 = r0b;
            const double e1 = fma(-Lb[b][0], e0, r1);
            const double e2 = fma(-Lb[b][2], e1, fma(-Lb[b][1], e0, r2));
            const double e3 = fma(-Lb[b][5], e2, fma(-Lb[b][4], e1, fma(-Lb[b][3], e0, r3)));
            rho = fma(-g[j], e0, rho);
            rho = fma(-g[j + 1], e1, rho);
            rho = fma(-g[j + 2], e2, rho);
            rho = fma(-g[j + 3], e3, rho);
            al0 += (lane == j) ? e0 : 0.0;   // a~ of this lane's coordinate (selects, no branches)
            al0 += (lane == j + 1) ? e1 : 0.0;
            al0 += (lane == j + 2) ? e2 : 0.0;
            al0 += (lane == j + 3) ? e3 : 0.0;
        }
    }
#ifdef K4_TIMING
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tc));
    if (lane == 0) printf("K4 phases ns: loads+stop test %llu  scaling %llu  sweeps %llu\n", ta - t00, tb - ta, tc - tb);
#endif
    // residual c~ - G a~ of the final iterate, this lane's row (PAPER.md:259-262 monitor)
    double res0 = ct0;
#pragma unroll
    for (int j = 0; j < SP; ++j) res0 = fma(-g[j], __shfl_sync(0xffffffffu, al0, j), res0);
    // ||L||_F^2 = sum_{i > j} G_ij^2
    const double ll = k4_warp_sum(lnorm_part);
    const double rr = k4_warp_sum(res0 * res0);
    const double cc = k4_warp_sum(ct0 * ct0);
    if (v0) a.alpha[lane] = d0 * al0;
    if (recg && v0) {
        a.h_d[(int64_t)k * s + lane] = d0;
        a.h_at[(int64_t)k * s + lane] = al0;
        a.h_al[(int64_t)k * s + lane] = d0 * al0;
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

// dispatch on ceil(s/4) (s <= 32)
__device__ __forceinline__ void k4_fgs_dispatch(const K4Args &a, DevState *st, double *scratch)
{
    switch ((a.s + 3) >> 2) {
    case 1: k4_fgs_small<1>(a, st, scratch); break;
    case 2: k4_fgs_small<2>(a, st, scratch); break;
    case 3: k4_fgs_small<3>(a, st, scratch); break;
    case 4: k4_fgs_small<4>(a, st, scratch); break;
    case 5: k4_fgs_small<5>(a, st, scratch); break;
    case 6: k4_fgs_small<6>(a, st, scratch); break;
    case 7: k4_fgs_small<7>(a, st, scratch); break;
    default: k4_fgs_small<8>(a, st, scratch); break;
    }
}

}  // namespace sscg
