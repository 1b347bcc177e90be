/*
 * solve_poisson.c -- the C ABI used directly (no Python, no CUDA calls in the
 * caller): 3D 7-point Poisson on an n^3 grid, Jacobi preconditioning, analytic
 * spectral bounds of D^{-1}A, host b and x through sscg_solve_host.  Checks the
 * true residual ||b - A x|| / ||b|| on the host and exits 0 when it is at rtol.
 *
 *   gcc -O2 examples/solve_poisson.c -Iinclude -Lpaper_2512_09642_b200 -l:libsscg.so \
 *       -Wl,-rpath,paper_2512_09642_b200 -lm -o examples/solve_poisson
 *   examples/solve_poisson [n] [s] [nu]
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "sscg.h"

static double apply7(const double *x, int64_t n, int64_t i, int64_t j, int64_t k)
{
#define X(a, b, c) (((a) < 0 || (a) >= n || (b) < 0 || (b) >= n || (c) < 0 || (c) >= n) ? 0.0 : x[(a) + n * ((b) + n * (c))])
    return 6.0 * X(i, j, k) - X(i - 1, j, k) - X(i + 1, j, k) - X(i, j - 1, k) - X(i, j + 1, k) - X(i, j, k - 1) -
           X(i, j, k + 1);
#undef X
}

int main(int argc, char **argv)
{
    const int64_t n = argc > 1 ? atoll(argv[1]) : 64;
    const int s = argc > 2 ? atoi(argv[2]) : 16, nu = argc > 3 ? atoi(argv[3]) : 25;
    const double rtol = 1e-8;
    const int64_t N = n * n * n;
    double *b = malloc(N * sizeof(double)), *x = malloc(N * sizeof(double));
    uint64_t h = 42;
    for (int64_t i = 0; i < N; ++i) {   /* any right-hand side: xorshift in [-1, 1) */
        h ^= h << 13, h ^= h >> 7, h ^= h << 17;
        b[i] = (double)(h >> 11) * 0x1.0p-52 - 1.0;
    }
    /* eigenvalues of D^{-1}A for the Dirichlet 7-point Laplacian: 1 - cos(k pi/(n+1)) averaged over 3 axes */
    const double c = cos(M_PI / (double)(n + 1));
    const double lmin = 1.0 - c, lmax = 1.0 + c;
    sscg_operator A = {0};
    A.kind = SSCG_OP_STENCIL7;
    A.nx = A.ny = A.nz = n;
    sscg_ctx *ctx = NULL;
    if (sscg_setup(&A, NULL, lmin, lmax, s, nu, NULL, NULL, &ctx) != SSCG_OK) {
        fprintf(stderr, "setup: %s\n", sscg_last_error());
        return 2;
    }
    const sscg_status st = sscg_solve_host(ctx, b, x, rtol, 5000, SSCG_SOLVE_X0_ZERO);
    sscg_stats_t stats;
    sscg_stats(ctx, &stats);
    sscg_destroy(ctx);
    if (st != SSCG_OK) {
        fprintf(stderr, "solve: %s\n", sscg_last_error());
        return 2;
    }
    double rr = 0.0, bb = 0.0;
    for (int64_t k = 0; k < n; ++k)
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < n; ++i) {
                const int64_t q = i + n * (j + n * k);
                const double r = b[q] - apply7(x, n, i, j, k);
                rr += r * r;
                bb += b[q] * b[q];
            }
    const double true_rel = sqrt(rr / bb);
    printf("n=%lld s=%d nu=%d: %d outer iterations, converged=%d, recurrence relres %.3e, true relres %.3e, "
           "%.3f ms\n",
           (long long)n, s, nu, stats.outer_iterations, stats.converged, stats.relres_final, true_rel, stats.ms_total);
    free(b);
    free(x);
    return (stats.converged && true_rel <= rtol * 1.05) ? 0 : 1;
}
