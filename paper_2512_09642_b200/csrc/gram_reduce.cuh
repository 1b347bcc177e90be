// Shared by the Gram kernels K2 (k_gram.cu) and K2D (k_gram_dmma.cu).
#pragma once
#include <stdint.h>

namespace sscg {

// Fixed-order sum of the per-CTA partial blocks [nparts][s*s + s] into out
// (upper triangle mirrored, then c), run by the last CTA of a Gram launch.
// Teams of 8 lanes own one entry: lane m sums partials m, m+8, ... in order
// (its loads are independent, so ~nparts/8 L2 reads are in flight per lane),
// then the team combines with a fixed xor tree -- deterministic, and the
// tail of small launches drops from ~nparts dependent L2 round trips.
__device__ __forceinline__ void last_cta_sum(const double *part, int nparts, int s, double *out)
{
    const int nup = s * (s + 1) / 2, nent = s * s + s;
    const int team = threadIdx.x >> 3, m = threadIdx.x & 7, nteams = blockDim.x >> 3;
    const int rounds = (nup + s + nteams - 1) / nteams;   // uniform trip count: whole warps shuffle
    for (int rd = 0; rd < rounds; ++rd) {
        const int u = team + rd * nteams;
        const bool act = u < nup + s;
        int i = 0, j = -1, q = 0;
        if (!act) {
        } else if (u < nup) {   // u -> (i, j), i <= j, row-major over the upper triangle
            i = 0;
            int rem = u;
            while (rem >= s - i) { rem -= s - i; ++i; }
            j = i + rem;
            q = i * s + j;
        } else {
            i = u - nup;
            j = -1;
            q = s * s + i;
        }
        double v = 0.0;
        if (act) {
            // all of a lane's partials loaded before the first add (registers, up to
            // 8 x LCS_R partials): one L2 round trip instead of one per partial; the
            // adds keep the loop's order (b ascending; absent ones add +0.0)
            constexpr int LCS_R = 24;
            if (nparts <= 8 * LCS_R) {
                double t[LCS_R];
#pragma unroll
                for (int i = 0; i < LCS_R; ++i) {
                    const int b = m + 8 * i;
                    t[i] = (b < nparts) ? __ldcg(part + (int64_t)b * nent + q) : 0.0;
                }
#pragma unroll
                for (int i = 0; i < LCS_R; ++i) v += t[i];
            } else {
                for (int b = m; b < nparts; b += 8) v += __ldcg(part + (int64_t)b * nent + q);
            }
        }
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        if (act && m == 0) {
            if (j >= 0) {
                out[i * s + j] = v;
                out[j * s + i] = v;
            } else {
                out[q] = v;
            }
        }
    }
}

}  // namespace sscg
