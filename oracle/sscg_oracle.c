/*
 * sscg_oracle.c -- plain, slow, obviously-correct CPU FP64 oracle for the
 * Chebyshev-basis s-step PCG with nu-sweep Forward Gauss-Seidel (FGS) Gram
 * solves of Thomas & D'Ambra, arxiv 2512.09642 ("PAPER.md").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code, header, constant or helper with the CUDA product path
 * (paper_2512_09642_b200/csrc); neither side includes or links the other.
 *
 * Every routine follows the paper's definition or algorithm step by step, in
 * the paper's order and notation; there is no blocking, fusion or reordering
 * beyond what the definition states.  Where the paper is silent the reading
 * taken is the one listed in DESIGN.md "Readings" (R-numbers cited inline).
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (see oracle/build.py).
 * -ffp-contract=off: no fused multiply-add, so every product and sum is a
 * separately rounded IEEE operation as written.
 *
 * Operator kinds (R11, R12):
 *   0  2D 5-point  : A = 4 on the diagonal, -1 for the 4 lattice neighbours
 *   1  3D 7-point  : 6 / -1
 *   2  3D 27-point : 26 / -1 for all 26 neighbours (graph-Laplacian weights)
 *   3  3D variable-coefficient 7-point (cell-centred FV): A_ii = sum of the
 *      6 face coefficients around i (boundary faces included), A_i,nbr = -k_face
 *   4  CSR (row-major, both triangles stored)
 * All stencils act on the interior grid with homogeneous Dirichlet boundaries
 * (ghost values are zero), PAPER.md:308 (§8 "homogeneous Dirichlet").
 * Grid index of point (x,y,z) is g = x + nx*(y + ny*z).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int kind;
    long nx, ny, nz;
    /* variable-coefficient faces (kind 3):
     *   kx[(z*ny + y)*(nx+1) + f]  face between x=f-1 and x=f, f in [0,nx]
     *   ky[(z*(ny+1) + f)*nx + x]  face between y=f-1 and y=f, f in [0,ny]
     *   kz[(f*ny + y)*nx + x]      face between z=f-1 and z=f, f in [0,nz]  */
    const double *kx, *ky, *kz;
    /* CSR (kind 4) */
    long n;
    const long *rowptr;
    const int *colind;
    const double *val;
} orc_op;

typedef struct {
    /* filled by orc_sstep_cg; every pointer may be NULL; arrays have room for
     * (max_outer + 1) outer iterations */
    int outer;          /* number of updates x += P~ alpha~ applied            */
    int converged;      /* 1 if ||r_k|| <= rtol ||r_0|| was reached            */
    int breakdown;      /* 1 if some Ghat_ii <= 0 or is not finite             */
    double r0norm;      /* ||r_0||_2                                           */
    double *relres;     /* [k]     sqrt(c_0^(k)) / ||r_0||                      */
    double *ghat;       /* [k*s*s] raw Gram P^T A P (mirrored, row-major)       */
    double *c;          /* [k*s]   P^T r                                       */
    double *d;          /* [k*s]   Ruhe scaling                                 */
    double *alpha_t;    /* [k*s]   alpha~ after nu FGS sweeps                   */
    double *alpha;      /* [k*s]   alpha = d o alpha~                           */
    double *delta;      /* [k]     ||c~ - G alpha~|| / ||c~||                    */
    double *energy;     /* [k]     2 alpha~^T c~ - alpha~^T G alpha~             */
    int dump_iter;      /* outer index whose basis is copied out (-1: none)    */
    double *P_dump;     /* n*s column-major                                    */
    double *W_dump;     /* n*s column-major                                    */
    /* block-conjugate mode (ORC_OPT_BLOCKCG): the Gram system actually solved */
    double *gconj;      /* [k*s*s] G_k = Q_k^T A Q_k (= Ghat at k = 0)          */
    double *cconj;      /* [k*s]   c_k = Q_k^T r_k                             */
} orc_trace;

/* ------------------------------------------------------------------ */
/* operator                                                           */
/* ------------------------------------------------------------------ */

long orc_n(const orc_op *A)
{
    if (A->kind == 4) return A->n;
    return A->nx * A->ny * A->nz;
}

static double at(const orc_op *A, const double *x, long i, long j, long k)
{
    /* value of grid function x at (i,j,k); zero outside the interior grid */
    if (i < 0 || j < 0 || k < 0 || i >= A->nx || j >= A->ny || k >= A->nz) return 0.0;
    return x[i + A->nx * (j + A->ny * k)];
}

/* y = A x.  Canonical per-row order: centre term first, then neighbour terms in
 * lexicographic (dz, dy, dx) order (R10: summation order is otherwise silent). */
void orc_apply(const orc_op *A, const double *x, double *y)
{
    if (A->kind == 4) {
#pragma omp parallel for schedule(static)
        for (long r = 0; r < A->n; ++r) {
            double acc = 0.0;
            for (long q = A->rowptr[r]; q < A->rowptr[r + 1]; ++q) acc += A->val[q] * x[A->colind[q]];
            y[r] = acc;
        }
        return;
    }
    const long nx = A->nx, ny = A->ny, nz = A->nz;
#pragma omp parallel for schedule(static)
    for (long k = 0; k < nz; ++k)
        for (long j = 0; j < ny; ++j)
            for (long i = 0; i < nx; ++i) {
                long g = i + nx * (j + ny * k);
                double acc;
                if (A->kind == 0) {          /* 2D 5-point */
                    acc = 4.0 * x[g];
                    acc -= at(A, x, i, j - 1, k);
                    acc -= at(A, x, i - 1, j, k);
                    acc -= at(A, x, i + 1, j, k);
                    acc -= at(A, x, i, j + 1, k);
                } else if (A->kind == 1) {   /* 3D 7-point */
                    acc = 6.0 * x[g];
                    acc -= at(A, x, i, j, k - 1);
                    acc -= at(A, x, i, j - 1, k);
                    acc -= at(A, x, i - 1, j, k);
                    acc -= at(A, x, i + 1, j, k);
                    acc -= at(A, x, i, j + 1, k);
                    acc -= at(A, x, i, j, k + 1);
                } else if (A->kind == 2) {   /* 3D 27-point */
                    acc = 26.0 * x[g];
                    for (int dz = -1; dz <= 1; ++dz)
                        for (int dy = -1; dy <= 1; ++dy)
                            for (int dx = -1; dx <= 1; ++dx) {
                                if (dx == 0 && dy == 0 && dz == 0) continue;
                                acc -= at(A, x, i + dx, j + dy, k + dz);
                            }
                } else {                     /* kind 3: variable-coefficient 7-point */
                    double kzm = A->kz[(k * ny + j) * nx + i];
                    double kym = A->ky[(k * (ny + 1) + j) * nx + i];
                    double kxm = A->kx[(k * ny + j) * (nx + 1) + i];
                    double kxp = A->kx[(k * ny + j) * (nx + 1) + i + 1];
                    double kyp = A->ky[(k * (ny + 1) + j + 1) * nx + i];
                    double kzp = A->kz[((k + 1) * ny + j) * nx + i];
                    double diag = kzm + kym + kxm + kxp + kyp + kzp;
                    acc = diag * x[g];
                    acc -= kzm * at(A, x, i, j, k - 1);
                    acc -= kym * at(A, x, i, j - 1, k);
                    acc -= kxm * at(A, x, i - 1, j, k);
                    acc -= kxp * at(A, x, i + 1, j, k);
                    acc -= kyp * at(A, x, i, j + 1, k);
                    acc -= kzp * at(A, x, i, j, k + 1);
                }
                y[g] = acc;
            }
}

/* d = diag(A) (the Jacobi preconditioner M = diag(A), BASELINE configs) */
void orc_diag(const orc_op *A, double *d)
{
    long n = orc_n(A);
    if (A->kind == 4) {
        for (long r = 0; r < n; ++r) {
            d[r] = 0.0;
            for (long q = A->rowptr[r]; q < A->rowptr[r + 1]; ++q)
                if (A->colind[q] == r) d[r] += A->val[q];
        }
        return;
    }
    const long nx = A->nx, ny = A->ny, nz = A->nz;
    for (long k = 0; k < nz; ++k)
        for (long j = 0; j < ny; ++j)
            for (long i = 0; i < nx; ++i) {
                long g = i + nx * (j + ny * k);
                if (A->kind == 0) d[g] = 4.0;
                else if (A->kind == 1) d[g] = 6.0;
                else if (A->kind == 2) d[g] = 26.0;
                else {
                    double kzm = A->kz[(k * ny + j) * nx + i];
                    double kym = A->ky[(k * (ny + 1) + j) * nx + i];
                    double kxm = A->kx[(k * ny + j) * (nx + 1) + i];
                    double kxp = A->kx[(k * ny + j) * (nx + 1) + i + 1];
                    double kyp = A->ky[(k * (ny + 1) + j + 1) * nx + i];
                    double kzp = A->kz[((k + 1) * ny + j) * nx + i];
                    d[g] = kzm + kym + kxm + kxp + kyp + kzp;
                }
            }
}

/* ------------------------------------------------------------------ */
/* reductions                                                         */
/* ------------------------------------------------------------------ */

static double pairwise(const double *x, const double *y, long n)
{
    if (n <= 8) {
        double acc = 0.0;
        for (long i = 0; i < n; ++i) acc += x[i] * y[i];
        return acc;
    }
    long h = n / 2;
    return pairwise(x, y, h) + pairwise(x + h, y + h, n - h);
}

/* x^T y by fixed-block pairwise summation: 2^16-element blocks, each summed
 * pairwise, block sums added in index order (R10: independent of threads). */
double orc_dot(long n, const double *x, const double *y)
{
    const long B = 1L << 16;
    long nb = (n + B - 1) / B;
    double *part = (double *)malloc((size_t)(nb > 0 ? nb : 1) * sizeof(double));
#pragma omp parallel for schedule(static)
    for (long b = 0; b < nb; ++b) {
        long lo = b * B, m = (n - lo < B) ? n - lo : B;
        part[b] = pairwise(x + lo, y + lo, m);
    }
    double acc = 0.0;
    for (long b = 0; b < nb; ++b) acc += part[b];
    free(part);
    return acc;
}

/* ------------------------------------------------------------------ */
/* Chebyshev basis  (§2 Definition)                    */
/* ------------------------------------------------------------------ */

/* P, W are n x s column-major (column j at P + j*n).
 *   p_0 = r
 *   p_1 = theta (M^{-1}A - sigma I) p_0
 *   p_{j+1} = 2 theta (M^{-1}A - sigma I) p_j - p_{j-1}
 * with theta = 2/(lmax-lmin), sigma = (lmax+lmin)/2, M = diag
 * given in D.  W collects w_j = A p_j (needed for the Gram matrix P^T A P). */
void orc_chebyshev_basis(const orc_op *A, const double *D, double lmin, double lmax, int s,
                         const double *r, double *P, double *W)
{
    const long n = orc_n(A);
    const double theta = 2.0 / (lmax - lmin);
    const double sigma = (lmax + lmin) / 2.0;
    memcpy(P, r, (size_t)n * sizeof(double));
    for (int j = 0; j < s; ++j) {
        const double *pj = P + (long)j * n;
        double *wj = W + (long)j * n;
        orc_apply(A, pj, wj);                            /* w_j = A p_j */
        if (j == s - 1) break;
        double *pn = P + (long)(j + 1) * n;
        const double *pm = (j > 0) ? P + (long)(j - 1) * n : NULL;
#pragma omp parallel for schedule(static)
        for (long i = 0; i < n; ++i) {
            double t = wj[i] / D[i] - sigma * pj[i];    /* (M^{-1}A - sigma I) p_j */
            if (j == 0) pn[i] = theta * t;
            else pn[i] = (2.0 * theta) * t - pm[i];
        }
    }
}

/* Monomial basis p_j = (M^{-1}A)^j r. */
void orc_monomial_basis(const orc_op *A, const double *D, int s, const double *r, double *P, double *W)
{
    const long n = orc_n(A);
    memcpy(P, r, (size_t)n * sizeof(double));
    for (int j = 0; j < s; ++j) {
        orc_apply(A, P + (long)j * n, W + (long)j * n);
        if (j == s - 1) break;
        for (long i = 0; i < n; ++i) P[(long)(j + 1) * n + i] = W[(long)j * n + i] / D[i];
    }
}

/* ------------------------------------------------------------------ */
/* Gram system                                */
/* ------------------------------------------------------------------ */

/* Ghat = P^T A P = P^T W (s x s row-major; entries i<=j computed, mirrored, R9)
 * c = P^T r with r = p_0 (the residual is the first basis column). */
void orc_gram(long n, int s, const double *P, const double *W, double *Ghat, double *c)
{
    for (int i = 0; i < s; ++i)
        for (int j = i; j < s; ++j) {
            double v = orc_dot(n, P + (long)i * n, W + (long)j * n);
            Ghat[i * s + j] = v;
            Ghat[j * s + i] = v;
        }
    for (int i = 0; i < s; ++i) c[i] = orc_dot(n, P + (long)i * n, P);
}

/* Ruhe column scaling: d_i = (p_i^T A p_i)^{-1/2}, S = diag(d),
 * G = S Ghat S with diag(G) = I set exactly (R6), c~ = S c = P~^T r.
 * Returns 0, or (i+1) if Ghat_ii <= 0 or is not finite (breakdown, R19). */
int orc_scale(int s, const double *Ghat, const double *c, double *d, double *G, double *ct)
{
    for (int i = 0; i < s; ++i) {
        double g = Ghat[i * s + i];
        if (!(g > 0.0) || !isfinite(g)) return i + 1;
        d[i] = 1.0 / sqrt(g);
    }
    for (int i = 0; i < s; ++i) {
        for (int j = 0; j < s; ++j) G[i * s + j] = (i == j) ? 1.0 : (d[i] * Ghat[i * s + j]) * d[j];
        ct[i] = d[i] * c[i];
    }
    return 0;
}

/* FGS (general diagonal PAPER.md:64-66 §3 Prop.):
 *   (D + L) alpha^(l+1) = rhs - L^T alpha^(l),   alpha^(0) = 0,
 * computed by forward substitution:
 *   alpha_j = (rhs_j - sum_{i<j} G_ji alpha_i^(l+1) - sum_{i>j} G_ji alpha_i^(l)) / G_jj
 * in place, i ascending (R8).  For the Ruhe-scaled G, G_jj = 1 exactly, so the
 * division is exact and this is the paper's (I + L) form.  If hist != NULL it
 * receives ||rhs - G alpha^(l)||_2 for l = 0..nu. */
void orc_fgs(int s, const double *G, const double *rhs, int nu, double *alpha, double *hist)
{
    for (int j = 0; j < s; ++j) alpha[j] = 0.0;
    for (int l = 0; l <= nu; ++l) {
        if (hist) {
            double ss = 0.0;
            for (int i = 0; i < s; ++i) {
                double ri = rhs[i];
                for (int k = 0; k < s; ++k) ri -= G[i * s + k] * alpha[k];
                ss += ri * ri;
            }
            hist[l] = sqrt(ss);
        }
        if (l == nu) break;
        for (int j = 0; j < s; ++j) {
            double acc = rhs[j];
            for (int i = 0; i < s; ++i)
                if (i != j) acc -= G[j * s + i] * alpha[i];
            alpha[j] = acc / G[j * s + j];
        }
    }
}

/* exact Gram solve by dense Cholesky G = R^T R (the O(s^3)
 * alternative FGS replaces).  Returns 0 or (k+1) if pivot k is not positive. */
int orc_cholesky_solve(int s, const double *G, const double *rhs, double *x)
{
    double *R = (double *)calloc((size_t)s * s, sizeof(double));
    for (int k = 0; k < s; ++k) {
        double a = G[k * s + k];
        for (int m = 0; m < k; ++m) a -= R[m * s + k] * R[m * s + k];
        if (!(a > 0.0)) { free(R); return k + 1; }
        R[k * s + k] = sqrt(a);
        for (int j = k + 1; j < s; ++j) {
            double b = G[k * s + j];
            for (int m = 0; m < k; ++m) b -= R[m * s + k] * R[m * s + j];
            R[k * s + j] = b / R[k * s + k];
        }
    }
    double *y = (double *)malloc((size_t)s * sizeof(double));
    for (int i = 0; i < s; ++i) {           /* R^T y = rhs */
        double a = rhs[i];
        for (int m = 0; m < i; ++m) a -= R[m * s + i] * y[m];
        y[i] = a / R[i * s + i];
    }
    for (int i = s - 1; i >= 0; --i) {      /* R x = y */
        double a = y[i];
        for (int m = i + 1; m < s; ++m) a -= R[i * s + m] * x[m];
        x[i] = a / R[i * s + i];
    }
    free(R);
    free(y);
    return 0;
}

/* MGS in the A-inner product (§5 Thm Algebraic Equivalence):
 *   w_0 = v;  for j: gamma_j = w_{j-1}^T A p~_j,  w_j = w_{j-1} - gamma_j p~_j.
 * Pt: n x s column-major scaled basis.  wout (n) receives w_s if non-NULL. */
void orc_mgs_anorm(const orc_op *A, int s, const double *Pt, const double *v, double *gamma, double *wout)
{
    long n = orc_n(A);
    double *w = (double *)malloc((size_t)n * sizeof(double));
    double *Ap = (double *)malloc((size_t)n * sizeof(double));
    memcpy(w, v, (size_t)n * sizeof(double));
    for (int j = 0; j < s; ++j) {
        orc_apply(A, Pt + (long)j * n, Ap);
        gamma[j] = orc_dot(n, w, Ap);
        for (long i = 0; i < n; ++i) w[i] = w[i] - gamma[j] * Pt[(long)j * n + i];
    }
    if (wout) memcpy(wout, w, (size_t)n * sizeof(double));
    free(w);
    free(Ap);
}

/* ------------------------------------------------------------------ */
/* s-step CG outer iteration (§2; restart form, R3-R5)     */
/* ------------------------------------------------------------------ */

/* D: diag(M) (NULL => diag(A)).  x: in x_0, out x_k.  Returns 0 or 1 on breakdown.
 * Per outer k:
 *   a. P = Chebyshev basis of K_s(M^{-1}A, r_k) with p_0 = r_k
 *   b. Ghat = P^T A P, c = P^T r_k
 *   c. stop if sqrt(c_0) <= rtol ||r_0|| (c_0 = ||r_k||^2), or k = max_outer
 *   e. Ruhe scaling d, G = S Ghat S, c~ = S c
 *   f. nu FGS sweeps from alpha~ = 0
 *   g. alpha = S alpha~; x += P alpha; r -= W alpha (= A P alpha)  */
/* Restart s-step CG with the Chebyshev basis and nu FGS sweeps
 * (the north_star path).  orc_sstep_cg_ex adds the two variants of SURVEY
 * §8(f) NEXT-2 that share the boundary:
 *   opts & ORC_OPT_CHOLESKY  exact Gram solve G a~ = c~ by dense Cholesky
 *                            (the O(s^3) method FGS replaces)
 *   opts & ORC_OPT_MONOMIAL  monomial basis p_{j+1} = M^{-1} A p_j
 *                            ("For monomial bases")
 * A Cholesky breakdown (non-positive pivot) is reported as a Gram breakdown. */
/*   opts & ORC_OPT_BLOCKCG   block-conjugate s-step CG (
 *                            the paper updates only
 *                            x += P alpha, i.e. the restart
 *                            form; this is the classical alternative, DESIGN.md
 *                            R24).  With the previous search block Q' and
 *                            Z' = A Q' kept, per outer k >= 1:
 *                              G' = Q'^T Z',  C = Z'^T P_k,  e = Q'^T r_k
 *                              B  = G'^{-1} C                (Cholesky of G')
 *                              Q_k = P_k - Q' B,  Z_k = W_k - Z' B
 *                              G_k = Ghat - C^T B,  c_k = c - B^T e
 *                            (G_k = Q_k^T A Q_k and c_k = Q_k^T r_k, expanded
 *                            with B^T G' B = C^T B, so one Gram pass over
 *                            [P_k | Q'] gives every entry); then the same
 *                            scaling + FGS / Cholesky on (G_k, c_k), and
 *                            x += Q_k alpha, r -= Z_k alpha.  k = 0: Q = P. */
#define ORC_OPT_CHOLESKY 1
#define ORC_OPT_MONOMIAL 2
#define ORC_OPT_BLOCKCG 4
int orc_sstep_cg_ex(const orc_op *A, const double *Dm, double lmin, double lmax, int s, int nu,
                    const double *b, double *x, double rtol, int max_outer, orc_trace *tr, int opts);

int orc_sstep_cg(const orc_op *A, const double *Dm, double lmin, double lmax, int s, int nu,
                 const double *b, double *x, double rtol, int max_outer, orc_trace *tr)
{
    return orc_sstep_cg_ex(A, Dm, lmin, lmax, s, nu, b, x, rtol, max_outer, tr, 0);
}

int orc_sstep_cg_ex(const orc_op *A, const double *Dm, double lmin, double lmax, int s, int nu,
                    const double *b, double *x, double rtol, int max_outer, orc_trace *tr, int opts)
{
    const long n = orc_n(A);
    double *D = (double *)malloc((size_t)n * sizeof(double));
    if (Dm) memcpy(D, Dm, (size_t)n * sizeof(double));
    else orc_diag(A, D);
    double *r = (double *)malloc((size_t)n * sizeof(double));
    double *P = (double *)malloc((size_t)n * s * sizeof(double));
    double *W = (double *)malloc((size_t)n * s * sizeof(double));
    double *Ghat = (double *)malloc((size_t)s * s * sizeof(double));
    double *G = (double *)malloc((size_t)s * s * sizeof(double));
    double *c = (double *)malloc((size_t)s * sizeof(double));
    double *d = (double *)malloc((size_t)s * sizeof(double));
    double *ct = (double *)malloc((size_t)s * sizeof(double));
    double *at_ = (double *)malloc((size_t)s * sizeof(double));
    double *al = (double *)malloc((size_t)s * sizeof(double));
    /* block-conjugate mode: previous search block Q', Z' = A Q' and the work arrays */
    const int blockcg = (opts & ORC_OPT_BLOCKCG) != 0;
    double *Qp = NULL, *Zp = NULL, *Gp = NULL, *Cx = NULL, *Bm = NULL, *e = NULL, *Gk = NULL, *ck = NULL,
           *colb = NULL, *colx = NULL;
    if (blockcg) {
        Qp = (double *)malloc((size_t)n * s * sizeof(double));
        Zp = (double *)malloc((size_t)n * s * sizeof(double));
        Gp = (double *)malloc((size_t)s * s * sizeof(double));
        Cx = (double *)malloc((size_t)s * s * sizeof(double));
        Bm = (double *)malloc((size_t)s * s * sizeof(double));
        e = (double *)malloc((size_t)s * sizeof(double));
        Gk = (double *)malloc((size_t)s * s * sizeof(double));
        ck = (double *)malloc((size_t)s * sizeof(double));
        colb = (double *)malloc((size_t)s * sizeof(double));
        colx = (double *)malloc((size_t)s * sizeof(double));
    }

    /* r_0 = b - A x_0 */
    orc_apply(A, x, r);
    for (long i = 0; i < n; ++i) r[i] = b[i] - r[i];
    double r0norm = sqrt(orc_dot(n, r, r));
    int k = 0, converged = 0, breakdown = 0;
    if (tr) { tr->r0norm = r0norm; }
    for (;;) {
        if (opts & ORC_OPT_MONOMIAL) orc_monomial_basis(A, D, s, r, P, W);
        else orc_chebyshev_basis(A, D, lmin, lmax, s, r, P, W);
        orc_gram(n, s, P, W, Ghat, c);
        double rn = sqrt(c[0]);
        if (tr) {
            if (tr->relres) tr->relres[k] = (r0norm > 0.0) ? rn / r0norm : 0.0;
            if (tr->ghat) memcpy(tr->ghat + (long)k * s * s, Ghat, (size_t)s * s * sizeof(double));
            if (tr->c) memcpy(tr->c + (long)k * s, c, (size_t)s * sizeof(double));
            if (tr->dump_iter == k) {
                if (tr->P_dump) memcpy(tr->P_dump, P, (size_t)n * s * sizeof(double));
                if (tr->W_dump) memcpy(tr->W_dump, W, (size_t)n * s * sizeof(double));
            }
        }
        if (rn <= rtol * r0norm) { converged = 1; break; }
        if (k == max_outer) break;
        const double *Gsys = Ghat, *csys = c;   /* the Gram system solved this outer */
        if (blockcg && k > 0) {
            /* G' = Q'^T Z' (i <= j, mirrored), C = Z'^T P_k, e = Q'^T r_k */
            for (int i = 0; i < s; ++i)
                for (int j = i; j < s; ++j) {
                    const double v = orc_dot(n, Qp + (long)i * n, Zp + (long)j * n);
                    Gp[i * s + j] = v;
                    Gp[j * s + i] = v;
                }
            for (int i = 0; i < s; ++i) {
                for (int j = 0; j < s; ++j) Cx[i * s + j] = orc_dot(n, Zp + (long)i * n, P + (long)j * n);
                e[i] = orc_dot(n, Qp + (long)i * n, r);
            }
            /* B = G'^{-1} C, column by column */
            for (int j = 0; j < s; ++j) {
                for (int i = 0; i < s; ++i) colb[i] = Cx[i * s + j];
                if (orc_cholesky_solve(s, Gp, colb, colx) != 0) { breakdown = 1; break; }
                for (int i = 0; i < s; ++i) Bm[i * s + j] = colx[i];
            }
            if (breakdown) break;
            /* G_k = Ghat - C^T B (i <= j, mirrored),  c_k = c - B^T e */
            for (int i = 0; i < s; ++i)
                for (int j = i; j < s; ++j) {
                    double v = 0.0;
                    for (int m = 0; m < s; ++m) v += Cx[m * s + i] * Bm[m * s + j];
                    Gk[i * s + j] = Ghat[i * s + j] - v;
                    Gk[j * s + i] = Gk[i * s + j];
                }
            for (int i = 0; i < s; ++i) {
                double v = 0.0;
                for (int m = 0; m < s; ++m) v += Bm[m * s + i] * e[m];
                ck[i] = c[i] - v;
            }
            /* Q_k = P_k - Q' B,  Z_k = W_k - Z' B, in place of P, W */
#pragma omp parallel for schedule(static)
            for (long q = 0; q < n; ++q) {
                double pq[64], wq[64];
                for (int j = 0; j < s; ++j) {
                    double sp = 0.0, sw = 0.0;
                    for (int m = 0; m < s; ++m) {
                        sp += Qp[(long)m * n + q] * Bm[m * s + j];
                        sw += Zp[(long)m * n + q] * Bm[m * s + j];
                    }
                    pq[j] = P[(long)j * n + q] - sp;
                    wq[j] = W[(long)j * n + q] - sw;
                }
                for (int j = 0; j < s; ++j) {
                    P[(long)j * n + q] = pq[j];
                    W[(long)j * n + q] = wq[j];
                }
            }
            Gsys = Gk;
            csys = ck;
        }
        if (blockcg && tr) {
            if (tr->gconj) memcpy(tr->gconj + (long)k * s * s, Gsys, (size_t)s * s * sizeof(double));
            if (tr->cconj) memcpy(tr->cconj + (long)k * s, csys, (size_t)s * sizeof(double));
        }
        if (orc_scale(s, Gsys, csys, d, G, ct) != 0) { breakdown = 1; break; }
        if (opts & ORC_OPT_CHOLESKY) {
            if (orc_cholesky_solve(s, G, ct, at_) != 0) { breakdown = 1; break; }
        } else {
            orc_fgs(s, G, ct, nu, at_, NULL);
        }
        for (int j = 0; j < s; ++j) al[j] = d[j] * at_[j];
        /* x += P alpha ; r -= A P alpha = W alpha */
#pragma omp parallel for schedule(static)
        for (long i = 0; i < n; ++i) {
            double ax = 0.0, aw = 0.0;
            for (int j = 0; j < s; ++j) {
                ax += al[j] * P[(long)j * n + i];
                aw += al[j] * W[(long)j * n + i];
            }
            x[i] = x[i] + ax;
            r[i] = r[i] - aw;
        }
        if (blockcg) {   /* this block becomes Q', Z' of the next outer */
            memcpy(Qp, P, (size_t)n * s * sizeof(double));
            memcpy(Zp, W, (size_t)n * s * sizeof(double));
        }
        if (tr) {
            if (tr->d) memcpy(tr->d + (long)k * s, d, (size_t)s * sizeof(double));
            if (tr->alpha_t) memcpy(tr->alpha_t + (long)k * s, at_, (size_t)s * sizeof(double));
            if (tr->alpha) memcpy(tr->alpha + (long)k * s, al, (size_t)s * sizeof(double));
            if (tr->delta || tr->energy) {
                double rr = 0.0, cc = 0.0, e1 = 0.0, e2 = 0.0;
                for (int i = 0; i < s; ++i) {
                    double gi = 0.0;
                    for (int j = 0; j < s; ++j) gi += G[i * s + j] * at_[j];
                    rr += (ct[i] - gi) * (ct[i] - gi);
                    cc += ct[i] * ct[i];
                    e1 += at_[i] * ct[i];
                    e2 += at_[i] * gi;
                }
                if (tr->delta) tr->delta[k] = sqrt(rr) / sqrt(cc);
                if (tr->energy) tr->energy[k] = 2.0 * e1 - e2;
            }
        }
        ++k;
    }
    if (tr) { tr->outer = k; tr->converged = converged; tr->breakdown = breakdown; }
    free(D); free(r); free(P); free(W); free(Ghat); free(G); free(c); free(d); free(ct); free(at_); free(al);
    if (blockcg) {
        free(Qp); free(Zp); free(Gp); free(Cx); free(Bm); free(e); free(Gk); free(ck); free(colb); free(colx);
    }
    return breakdown;
}

/* classical Jacobi-PCG (context only; >= 2 reductions per iteration) */
int orc_pcg(const orc_op *A, const double *Dm, const double *b, double *x, double rtol, int max_iter)
{
    const long n = orc_n(A);
    double *D = (double *)malloc((size_t)n * sizeof(double));
    if (Dm) memcpy(D, Dm, (size_t)n * sizeof(double));
    else orc_diag(A, D);
    double *r = (double *)malloc((size_t)n * sizeof(double));
    double *z = (double *)malloc((size_t)n * sizeof(double));
    double *p = (double *)malloc((size_t)n * sizeof(double));
    double *q = (double *)malloc((size_t)n * sizeof(double));
    orc_apply(A, x, r);
    for (long i = 0; i < n; ++i) r[i] = b[i] - r[i];
    double r0 = sqrt(orc_dot(n, r, r));
    for (long i = 0; i < n; ++i) { z[i] = r[i] / D[i]; p[i] = z[i]; }
    double rz = orc_dot(n, r, z);
    int it = 0;
    while (it < max_iter && sqrt(orc_dot(n, r, r)) > rtol * r0) {
        orc_apply(A, p, q);
        double a = rz / orc_dot(n, p, q);
        for (long i = 0; i < n; ++i) { x[i] += a * p[i]; r[i] -= a * q[i]; }
        for (long i = 0; i < n; ++i) z[i] = r[i] / D[i];
        double rz1 = orc_dot(n, r, z);
        double beta = rz1 / rz;
        rz = rz1;
        for (long i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        ++it;
    }
    free(D); free(r); free(z); free(p); free(q);
    return it;
}

/* ------------------------------------------------------------------ */
/* Lanczos spectral bounds (§8; R13)                      */
/* ------------------------------------------------------------------ */

/* number of eigenvalues of the symmetric tridiagonal (a, b) below x (Sturm) */
static int sturm_count(int m, const double *a, const double *b, double x)
{
    int cnt = 0;
    double q = a[0] - x;
    if (q < 0) ++cnt;
    for (int i = 1; i < m; ++i) {
        double qq = (q != 0.0) ? q : 1e-300;
        q = a[i] - x - b[i - 1] * b[i - 1] / qq;
        if (q < 0) ++cnt;
    }
    return cnt;
}

/* k-th smallest eigenvalue (0-based) of the tridiagonal by bisection */
double orc_tridiag_eig(int m, const double *a, const double *b, int kth)
{
    double lo = a[0], hi = a[0];
    for (int i = 0; i < m; ++i) {
        double rad = (i > 0 ? fabs(b[i - 1]) : 0.0) + (i < m - 1 ? fabs(b[i]) : 0.0);
        if (a[i] - rad < lo) lo = a[i] - rad;
        if (a[i] + rad > hi) hi = a[i] + rad;
    }
    for (int it = 0; it < 200; ++it) {
        double mid = 0.5 * (lo + hi);
        if (mid == lo || mid == hi) break;
        if (sturm_count(m, a, b, mid) > kth) hi = mid;
        else lo = mid;
    }
    return 0.5 * (lo + hi);
}

/* `iters` Lanczos steps on the symmetric D^{-1/2} A D^{-1/2} (same spectrum as
 * M^{-1}A), start v0/||v0||, no reorthogonalisation.  Returns the extreme Ritz
 * values widened multiplicatively: lmin (1 - margin), lmax (1 + margin).
 * Returns the number of steps taken (fewer on breakdown beta = 0). */
int orc_lanczos_bounds_tri(const orc_op *A, const double *Dm, int iters, const double *v0, double margin,
                           double *lmin, double *lmax, double *al_out, double *be_out);

int orc_lanczos_bounds(const orc_op *A, const double *Dm, int iters, const double *v0, double margin,
                       double *lmin, double *lmax)
{
    return orc_lanczos_bounds_tri(A, Dm, iters, v0, margin, lmin, lmax, NULL, NULL);
}

/* same, and copies the tridiagonal (alpha_k, k < m; beta_k, k < m-1) out */
int orc_lanczos_bounds_tri(const orc_op *A, const double *Dm, int iters, const double *v0, double margin,
                           double *lmin, double *lmax, double *al_out, double *be_out)
{
    const long n = orc_n(A);
    double *D = (double *)malloc((size_t)n * sizeof(double));
    if (Dm) memcpy(D, Dm, (size_t)n * sizeof(double));
    else orc_diag(A, D);
    double *v = (double *)malloc((size_t)n * sizeof(double));
    double *vp = (double *)calloc((size_t)n, sizeof(double));
    double *u = (double *)malloc((size_t)n * sizeof(double));
    double *t = (double *)malloc((size_t)n * sizeof(double));
    double *al = (double *)malloc((size_t)iters * sizeof(double));
    double *be = (double *)malloc((size_t)iters * sizeof(double));
    double nv = sqrt(orc_dot(n, v0, v0));
    for (long i = 0; i < n; ++i) v[i] = v0[i] / nv;
    double beta = 0.0;
    int m = 0;
    for (int k = 0; k < iters; ++k) {
        for (long i = 0; i < n; ++i) t[i] = v[i] / sqrt(D[i]);
        orc_apply(A, t, u);
        for (long i = 0; i < n; ++i) u[i] = u[i] / sqrt(D[i]);
        double a = orc_dot(n, u, v);
        for (long i = 0; i < n; ++i) u[i] = u[i] - a * v[i] - beta * vp[i];
        al[k] = a;
        m = k + 1;
        beta = sqrt(orc_dot(n, u, u));
        if (k == iters - 1 || beta == 0.0) break;
        be[k] = beta;
        for (long i = 0; i < n; ++i) { vp[i] = v[i]; v[i] = u[i] / beta; }
    }
    if (al_out) memcpy(al_out, al, (size_t)m * sizeof(double));
    if (be_out && m > 1) memcpy(be_out, be, (size_t)(m - 1) * sizeof(double));
    *lmin = orc_tridiag_eig(m, al, be, 0) * (1.0 - margin);
    *lmax = orc_tridiag_eig(m, al, be, m - 1) * (1.0 + margin);
    free(D); free(v); free(vp); free(u); free(t); free(al); free(be);
    return m;
}

/* ------------------------------------------------------------------ */
/* AMG coarse grid: Galerkin operator A_c = P^T A_f P and Forward      */
/* Gauss-Seidel on it (§6 "AMG Coarse-Grid            */
/* Extension", §8; R25) */
/* ------------------------------------------------------------------ */

/* R25: P is the piecewise-constant (unsmoothed aggregation) prolongation of
 * bx x by x bz blocks of fine cells: coarse point (I, J, K) aggregates the
 * fine cells x in [bx I, min(bx I + bx, nx)), likewise y, z; the last block
 * of each axis may be partial.  P_{g, c} = 1 if fine cell g lies in aggregate
 * c, else 0.  Coarse points are numbered c = I + ncx (J + ncy K). */
static long cdiv(long a, long b) { return (a + b - 1) / b; }

long orc_coarse_n(const orc_op *A, int bx, int by, int bz)
{
    return cdiv(A->nx, bx) * cdiv(A->ny, by) * cdiv(A->nz, bz);
}

static long agg_of(const orc_op *A, int bx, int by, int bz, long g)
{
    const long i = g % A->nx, j = (g / A->nx) % A->ny, k = g / (A->nx * A->ny);
    const long ncx = cdiv(A->nx, bx), ncy = cdiv(A->ny, by);
    return i / bx + ncx * (j / by + ncy * (k / bz));
}

/* r_c = P^T r_f: r_c[c] = sum of r_f over the cells of aggregate c, added in
 * ascending fine index */
void orc_coarse_restrict(const orc_op *A, int bx, int by, int bz, const double *rf, double *rc)
{
    const long nf = orc_n(A), nc = orc_coarse_n(A, bx, by, bz);
    for (long c = 0; c < nc; ++c) rc[c] = 0.0;
    for (long g = 0; g < nf; ++g) rc[agg_of(A, bx, by, bz, g)] += rf[g];
}

/* x_f += P y: every fine cell gets the value of its aggregate */
void orc_coarse_prolong_add(const orc_op *A, int bx, int by, int bz, const double *y, double *xf)
{
    const long nf = orc_n(A);
    for (long g = 0; g < nf; ++g) xf[g] += y[agg_of(A, bx, by, bz, g)];
}

/* A_c = P^T A_f P formed column by column, as the definition reads: column c
 * is P^T (A_f p_c), p_c = P e_c the indicator of aggregate c (one full fine
 * operator application and one restriction per column).  Stored as CSR of
 * its rows -- entry (i, c) is the i-th component of column c; the nonzero
 * entries of each row in ascending column order (a row of the CSR is filled
 * by walking the columns in order: data movement only).  rowptr[nc + 1],
 * col / val with room for `cap` entries.  Returns nnz, or -1 if cap is too
 * small.  Cost O(n_c n_f): test sizes only. */
long orc_coarse_galerkin(const orc_op *A, int bx, int by, int bz, long *rowptr, long *col, double *val, long cap)
{
    const long nf = orc_n(A), nc = orc_coarse_n(A, bx, by, bz);
    double *p = (double *)calloc((size_t)nf, sizeof(double));
    double *w = (double *)malloc((size_t)nf * sizeof(double));
    double *t = (double *)malloc((size_t)nc * sizeof(double));
    long *ccol = (long *)malloc((size_t)cap * sizeof(long)), *crow = (long *)malloc((size_t)cap * sizeof(long));
    double *cval = (double *)malloc((size_t)cap * sizeof(double));
    long nnz = 0;
    for (long c = 0; c < nc && nnz >= 0; ++c) {
        for (long g = 0; g < nf; ++g) p[g] = (agg_of(A, bx, by, bz, g) == c) ? 1.0 : 0.0;
        orc_apply(A, p, w);
        orc_coarse_restrict(A, bx, by, bz, w, t);
        for (long i = 0; i < nc; ++i) {
            if (t[i] == 0.0) continue;
            if (nnz == cap) { nnz = -1; break; }
            crow[nnz] = i; ccol[nnz] = c; cval[nnz] = t[i];
            ++nnz;
        }
    }
    if (nnz >= 0) {
        /* CSC (column-major walk) -> CSR: count per row, prefix, fill */
        for (long i = 0; i <= nc; ++i) rowptr[i] = 0;
        for (long q = 0; q < nnz; ++q) rowptr[crow[q] + 1] += 1;
        for (long i = 0; i < nc; ++i) rowptr[i + 1] += rowptr[i];
        long *fill = (long *)malloc((size_t)(nc + 1) * sizeof(long));
        for (long i = 0; i <= nc; ++i) fill[i] = rowptr[i];
        for (long q = 0; q < nnz; ++q) {   /* columns ascending */
            const long d = fill[crow[q]]++;
            col[d] = ccol[q];
            val[d] = cval[q];
        }
        free(fill);
    }
    free(p); free(w); free(t); free(ccol); free(crow); free(cval);
    return nnz;
}

/* Forward Gauss-Seidel on A_c y = r_c ("FGS converges
 * uniformly ... requiring nu = 10-30 iterations"; §8 nu_coarse = 20 at the
 * coarsest level): nu sweeps, each over i = 0 .. n_c-1 in order,
 *     y_i <- (r_i - sum_{j != i} a_ij y_j) / a_ii,
 * the sum over row i's entries in ascending j (the latest y_j: updated for
 * j < i in this sweep).  y holds the initial guess on entry. */
void orc_coarse_fgs(long nc, const long *rowptr, const long *col, const double *val, const double *rc, int nu,
                    double *y)
{
    for (int sweep = 0; sweep < nu; ++sweep)
        for (long i = 0; i < nc; ++i) {
            double acc = rc[i], aii = 0.0;
            for (long q = rowptr[i]; q < rowptr[i + 1]; ++q) {
                if (col[q] == i) aii = val[q];
                else acc -= val[q] * y[col[q]];
            }
            y[i] = acc / aii;
        }
}
