"""Pins for the oracle's Chebyshev basis, Gram assembly
 and Ruhe scaling."""
import math

import numpy as np
import pytest

import inputs
import oracle as orc


def cheb_T(j, x):
    """Chebyshev polynomial of the first kind by its trigonometric closed form."""
    if abs(x) <= 1:
        return math.cos(j * math.acos(x))
    v = math.cosh(j * math.acosh(abs(x)))
    return v if x > 0 or j % 2 == 0 else -v


def diag_csr(vals):
    n = len(vals)
    return orc.csr(np.arange(n + 1), np.arange(n), np.asarray(vals, float))


def test_spec_chebyshev_example(golden):
    g = golden["chebyshev_diag13"]
    A = diag_csr(g["A_diag"])
    P, W = orc.chebyshev_basis(A, np.ones(2), g["lmin"], g["lmax"], g["s"], g["r"])
    assert np.array_equal(P, np.array(g["P"]))
    assert np.array_equal(W, P * np.array(g["A_diag"]))


def test_s1_is_residual():
    A = orc.stencil(orc.KIND_7PT, 4, 4, 4)
    r = np.random.default_rng(0).standard_normal(64)
    P, W = orc.chebyshev_basis(A, orc.diag(A), 0.1, 1.9, 1, r)
    assert np.array_equal(P[0], r)
    assert np.array_equal(W[0], orc.apply(A, r))


@pytest.mark.parametrize("kind,dims,ks,widen", [
    ("7pt", (12, 10, 9), (2, 3, 1), 1.0),
    ("27pt", (9, 8, 10), (1, 4, 2), 1.0),
    ("5pt", (14, 11, 1), (3, 5, 1), 1.0),
    ("7pt", (12, 10, 9), (1, 1, 1), 0.5),   # narrowed interval: |x| > 1, cosh branch
])
def test_single_mode_basis_is_chebyshev_polynomial(kind, dims, ks, widen):
    K = {"5pt": orc.KIND_5PT2D, "7pt": orc.KIND_7PT, "27pt": orc.KIND_27PT}[kind]
    A = orc.stencil(K, *dims)
    D = orc.diag(A)
    lo, hi = inputs.analytic_bounds(kind, *dims)
    mid, half = (lo + hi) / 2, (hi - lo) / 2 * widen
    lmin, lmax = mid - half, mid + half
    d2 = dims[:2] if kind == "5pt" else dims
    k2 = ks[:2] if kind == "5pt" else ks
    lamA = inputs.sine_mode_eig(kind, d2, k2)
    lam = lamA / D[0]
    theta, sigma = 2 / (lmax - lmin), (lmax + lmin) / 2
    xm = theta * (lam - sigma)
    v = inputs.sine_mode(*dims, *ks)
    s = 12
    P, W = orc.chebyshev_basis(A, D, lmin, lmax, s, v)
    for j in range(s):
        T = cheb_T(j, xm)
        scale = max(1.0, abs(T))
        assert np.max(np.abs(P[j] - T * v)) < 1e-12 * scale, j
        assert np.max(np.abs(W[j] - lamA * T * v)) < 1e-11 * scale * max(1, lamA), j


def test_monomial_basis_matches_matrix_powers():
    A = orc.stencil(orc.KIND_7PT, 4, 3, 3)
    M = np.array([orc.apply(A, e) for e in np.eye(A.n)]).T
    r = np.random.default_rng(3).standard_normal(A.n)
    P, _ = orc.monomial_basis(A, orc.diag(A), 5, r)
    v = r.copy()
    for j in range(5):
        assert np.allclose(P[j], v, rtol=1e-13, atol=1e-13)
        v = (M @ v) / 6.0


def test_spec_gram_scaling_example(golden):
    g = golden["gram_scaled_diag13"]
    A = diag_csr([1.0, 3.0])
    P, W = orc.chebyshev_basis(A, np.ones(2), 1.0, 3.0, 2, [1.0, 1.0])
    Ghat, c = orc.gram(P, W)
    assert np.array_equal(Ghat, np.array(g["Ghat"]))
    assert np.array_equal(c, np.array(g["c"]))
    d, G, ct = orc.scale(Ghat, c)
    assert np.array_equal(d, g["d"]) and np.array_equal(G, np.array(g["G"])) and np.array_equal(ct, g["ct"])


@pytest.mark.parametrize("kind,dims", [("7pt", (10, 9, 8)), ("27pt", (8, 9, 7))])
def test_gram_closed_form_multimode(kind, dims):
    """r = sum_m c_m v_m over K >= s sine modes:
    Ghat_ij = sum_m c_m^2 ||v_m||^2 lamA_m T_i(x_m) T_j(x_m),
    c_i    = sum_m c_m^2 ||v_m||^2 T_i(x_m),  ||v_m||^2 = prod_d (N_d+1)/2."""
    K = {"7pt": orc.KIND_7PT, "27pt": orc.KIND_27PT}[kind]
    A = orc.stencil(K, *dims)
    D = orc.diag(A)
    lmin, lmax = inputs.analytic_bounds(kind, *dims)
    theta, sigma = 2 / (lmax - lmin), (lmax + lmin) / 2
    rng = np.random.default_rng(5)
    s, Km = 8, 10
    modes = set()
    while len(modes) < Km:
        modes.add(tuple(int(rng.integers(1, d + 1)) for d in dims))
    modes = sorted(modes)
    coef = rng.standard_normal(Km)
    r = sum(cm * inputs.sine_mode(*dims, *ks) for cm, ks in zip(coef, modes))
    P, W = orc.chebyshev_basis(A, D, lmin, lmax, s, r)
    Ghat, c = orc.gram(P, W)
    nv2 = np.prod([(N + 1) / 2 for N in dims])
    Gcf = np.zeros((s, s)); ccf = np.zeros(s)
    for cm, ks in zip(coef, modes):
        lamA = inputs.sine_mode_eig(kind, dims, ks)
        x = theta * (lamA / D[0] - sigma)
        T = np.array([cheb_T(j, x) for j in range(s)])
        Gcf += cm * cm * nv2 * lamA * np.outer(T, T)
        ccf += cm * cm * nv2 * T
    assert np.max(np.abs(Ghat - Gcf)) < 1e-12 * np.max(np.abs(Gcf))
    assert np.max(np.abs(c - ccf)) < 1e-12 * np.max(np.abs(ccf))
    assert np.array_equal(Ghat, Ghat.T)
    d, G, ct = orc.scale(Ghat, c)
    assert np.all(np.diag(G) == 1.0)
    assert np.max(np.abs(d * d * np.diag(Ghat) - 1.0)) <= 4 * np.finfo(float).eps
    assert np.max(np.abs(G - G.T)) <= 4 * np.finfo(float).eps


def test_gram_scaling_breakdown():
    with pytest.raises(FloatingPointError):
        orc.scale(np.array([[1.0, 0.0], [0.0, 0.0]]), np.array([1.0, 0.0]))
    with pytest.raises(FloatingPointError):
        orc.scale(np.array([[np.nan]]), np.array([1.0]))


def lower_fro(kind, dims, s, seed):
    K = {"1d": orc.KIND_5PT2D, "5pt": orc.KIND_5PT2D}[kind]
    A = orc.stencil(K, *dims)
    if kind == "1d":
        # 1D Laplacian tridiag(-1,2,-1) via CSR (5-point needs ny >= 1 with 2D stencil)
        rp, ci, va = inputs.poisson_csr_1d(dims[0])
        A = orc.csr(rp, ci, va)
        N = dims[0]
        c = math.cos(math.pi / (N + 1))
        lmin, lmax = 1 - c, 1 + c
    else:
        lmin, lmax = inputs.analytic_bounds("5pt", *dims[:2])
    r = np.random.default_rng(seed).uniform(-1, 1, A.n)
    P, W = orc.chebyshev_basis(A, orc.diag(A), lmin, lmax, s, r)
    Ghat, c = orc.gram(P, W)
    _, G, _ = orc.scale(Ghat, c)
    return np.linalg.norm(np.tril(G, -1))


def test_lower_fro_grows_like_sqrt_s_1d():
    """PAPER.md:136-162 (Thm Polynomial Growth, ||L||_F = O(sqrt s)).  On the 1D
    Laplacian with exact bounds, G_{01} -> 1/sqrt2, G_{i,i+1} -> 1/2, so
    ||L||_F -> sqrt(s)/2 (R17)."""
    for s in (4, 8, 16, 32):
        lf = lower_fro("1d", (4096, 1, 1), s, seed=11)
        assert abs(lf / (math.sqrt(s) / 2) - 1) < 0.05, (s, lf)


def test_lower_fro_slope_2d():
    ss = [4, 8, 16, 32]
    lf = [lower_fro("5pt", (64, 64, 1), s, seed=12) for s in ss]
    slope = np.polyfit(np.log(ss), np.log(lf), 1)[0]
    assert 0.4 <= slope <= 0.7, slope


@pytest.mark.parametrize("kind,n,s,nu,it", [("7pt", 40, 16, 25, 0), ("7pt", 48, 16, 25, 25), ("27pt", 28, 16, 30, 10),
                                            ("varcoef7", 20, 16, 20, 30), ("5pt", 64, 8, 20, 50),
                                            ("7pt", 24, 32, 30, 8)])
def test_w_recovered_from_recurrence(kind, n, s, nu, it):
    """W = AP recovered POINTWISE from the Chebyshev recurrence (R23):
      w_0 = M (p_1/theta + sigma p_0),  w_j = M ((p_{j+1} + p_{j-1})/(2 theta) + sigma p_j)
    for j <= s-2 (PAPER.md:36-42 solved for M^{-1} A p_j) equals the SpMV W to a
    few ulps per entry, and so does the Gram block -- also late in the solve,
    where the residual is dominated by the low modes.  (Rebuilding G from
    dot products of P alone, G_ij = p_i^T M p_{j+1}/(2 theta) + ..., would
    cancel large dot products instead; that is not what is done.)"""
    nz = 1 if kind == "5pt" else n
    faces = inputs.lognormal_faces(n, n, nz, seed=42) if kind == "varcoef7" else None
    A = (orc.stencil(orc.KIND_VARCOEF7, n, n, nz, *faces) if faces is not None
         else orc.stencil({"5pt": orc.KIND_5PT2D, "7pt": orc.KIND_7PT, "27pt": orc.KIND_27PT}[kind], n, n, nz))
    b = inputs.rhs_uniform(n, n, nz, seed=42)
    if kind in ("27pt", "varcoef7"):
        lmin, lmax, _ = orc.lanczos_bounds(A, 50, b, 0.05)
    else:
        lmin, lmax = inputs.analytic_bounds(kind, n, n, nz)
    x, tr = orc.sstep_cg(A, lmin, lmax, s, nu, b, rtol=0.0, max_outer=it, dump_iter=it)
    P, W, M = tr.P, tr.W, orc.diag(A)
    th, sg = 2.0 / (lmax - lmin), (lmax + lmin) / 2.0
    Wr = np.empty_like(W)
    Wr[0] = M * (P[1] / th + sg * P[0])
    for j in range(1, s - 1):
        Wr[j] = M * ((P[j + 1] + P[j - 1]) / (2.0 * th) + sg * P[j])
    Wr[s - 1] = W[s - 1]
    for j in range(s - 1):
        assert np.max(np.abs(Wr[j] - W[j])) <= 1e-14 * np.max(np.abs(W[j])), j
    G, _ = orc.gram(P, W)
    Gr, _ = orc.gram(P, Wr)
    assert np.max(np.abs(Gr - G)) <= 1e-14 * np.max(np.abs(G))
    assert np.max(np.abs(np.diag(Gr) - np.diag(G)) / np.diag(G)) <= 1e-13


@pytest.mark.parametrize("s", [2, 9, 16, 24])
def test_gram_space_recurrence_identity(s):
    """The identity the folded Gram pass's Gram-space map rests on (DESIGN.md
    R27): with a constant diagonal M = m I, PAPER.md:36-42 solved for A p_j
    gives A P_{:,0:s} = P_{:,0:s+1} T (T (s+1) x s, m sigma on the diagonal,
    m/theta at (1, 0), m/(2 theta) at (j +- 1, j) otherwise), so Ghat = P^T A P
    = E T with E = P^T P_{:,0:s+1}: checked against the oracle's own Gram of
    its stored W = A P on the s + 1 vectors of its basis."""
    A = orc.stencil(orc.KIND_7PT, 14, 12, 11)
    D = orc.diag(A)
    lo, hi = inputs.analytic_bounds("7pt", 14, 12, 11)
    r = inputs.rhs_uniform(14, 12, 11, seed=4)
    P1, W1 = orc.chebyshev_basis(A, D, lo, hi, s + 1, r)
    Ghat, c = orc.gram(P1[:s], W1[:s])
    theta, sigma, m = 2 / (hi - lo), (hi + lo) / 2, D[0]
    T = np.zeros((s + 1, s))
    for j in range(s):
        T[j, j] = m * sigma
        T[j + 1, j] = m / theta if j == 0 else m / (2 * theta)
        if j > 0:
            T[j - 1, j] = m / (2 * theta)
    E = P1[:s] @ P1.T                       # (s, s+1)
    scale = np.max(np.abs(Ghat))
    assert np.max(np.abs(E @ T - Ghat)) <= 1e-12 * scale
    assert np.max(np.abs(E[:, 0] - c)) <= 1e-13 * np.max(np.abs(c))
    # a wrong coefficient (1/theta at every j, say) is far outside that
    T[2, 1] *= 2
    assert np.max(np.abs(E @ T - Ghat)) > 1e-3 * scale
