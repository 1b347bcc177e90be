"""Pins for the oracle's s-step CG outer iteration (restart form)."""
import math

import numpy as np
import pytest

import inputs
import oracle as orc


def diag_csr(vals):
    n = len(vals)
    return orc.csr(np.arange(n + 1), np.arange(n), np.asarray(vals, float))


def test_worked_example_one_outer(golden):
    g = golden["restart_sstep_diag13"]
    A = diag_csr(g["A_diag"])
    b = np.array(g["b"])
    x1, tr = orc.sstep_cg(A, 1.0, 3.0, 2, 1, b, rtol=0.0, max_outer=1, D=np.ones(2))
    assert np.array_equal(x1, g["x1_nu1"])
    assert np.array_equal(b - A.n * 0 - orc.apply(A, x1), g["r1_nu1"])
    assert np.array_equal(tr.ghat[0], [[4, 2], [2, 4]]) and np.array_equal(tr.c[0], [2, 0])
    assert np.array_equal(tr.alpha_t[0], [1.0, -0.5]) and np.array_equal(tr.alpha[0], [0.5, -0.25])
    x2, _ = orc.sstep_cg(A, 1.0, 3.0, 2, 2, b, rtol=0.0, max_outer=1, D=np.ones(2))
    assert np.array_equal(x2, g["x1_nu2"])


@pytest.mark.parametrize("nu,k", [(1, 1), (1, 3), (2, 2), (3, 4)])
def test_worked_example_closed_form(golden, nu, k):
    """r_k = 4^{-nu k} [1,1],  x_k = (1 - 4^{-nu k}) [1, 1/3]."""
    g = golden["restart_sstep_diag13"]
    A = diag_csr(g["A_diag"])
    b = np.array(g["b"])
    x, tr = orc.sstep_cg(A, 1.0, 3.0, 2, nu, b, rtol=0.0, max_outer=k, D=np.ones(2))
    f = 4.0 ** (-nu * k)
    assert np.allclose(x, (1 - f) * np.array(g["x_limit"]), rtol=1e-15, atol=1e-16)
    assert np.allclose(b - orc.apply(A, x), f * np.ones(2), rtol=1e-12, atol=1e-17)
    assert tr.relres[k] == pytest.approx(f, rel=1e-12)


def test_exact_in_one_outer_with_s_modes():
    """If r has exactly s eigen-modes, an (effectively) exact Gram solve gives
    x_1 = A^{-1} b in one outer iteration (Krylov space contains A^{-1} b)."""
    dims = (9, 8, 7)
    A = orc.stencil(orc.KIND_7PT, *dims)
    s = 4
    modes = [(1, 1, 1), (2, 3, 1), (5, 2, 4), (8, 7, 6)]
    coef = [1.0, -0.5, 0.25, 0.8]
    b = sum(c * inputs.sine_mode(*dims, *m) for c, m in zip(coef, modes))
    xstar = sum(c / inputs.sine_mode_eig("7pt", dims, m) * inputs.sine_mode(*dims, *m) for c, m in zip(coef, modes))
    lmin, lmax = inputs.analytic_bounds("7pt", *dims)
    x, tr = orc.sstep_cg(A, lmin, lmax, s, 4000, b, rtol=0.0, max_outer=1)
    assert np.linalg.norm(x - xstar) <= 1e-8 * np.linalg.norm(xstar)


@pytest.mark.parametrize("nu", [1, 2, 3, 5])
def test_worked_example_delta(golden, nu):
    """delta_k = ||c~ - G a~|| / ||c~|| on the worked example,
    by hand: G = [[1, 1/2], [1/2, 1]], c~ = [1, 0] at every outer iteration
    (r_k is a multiple of [1, 1]); each FGS sweep maps the error of a~ to a
    quarter of itself and leaves the residual c~ - G a~ = [4^-nu, 0], so
    delta_k = 4^-nu exactly (pins the normalisation and the square root)."""
    g = golden["restart_sstep_diag13"]
    A = diag_csr(g["A_diag"])
    b = np.array(g["b"])
    x, tr = orc.sstep_cg(A, 1.0, 3.0, 2, nu, b, rtol=0.0, max_outer=3, D=np.ones(2))
    for k in range(3):
        assert tr.delta[k] == pytest.approx(4.0 ** (-nu), rel=1e-13), (k, tr.delta[k])
    # and a non-trivial case: delta equals the definition evaluated by numpy on
    # the oracle's own G, c~, a~ of a 2D Laplacian outer iteration
    A2 = orc.stencil(orc.KIND_5PT2D, 12, 11, 1)
    b2 = inputs.rhs_uniform(12, 11, 1, seed=5)
    lmin, lmax = inputs.analytic_bounds("5pt", 12, 11)
    _, t2 = orc.sstep_cg(A2, lmin, lmax, 5, nu, b2, rtol=0.0, max_outer=2, dump_iter=1)
    for k in range(2):
        d = 1.0 / np.sqrt(np.diag(t2.ghat[k]))
        G = d[:, None] * t2.ghat[k] * d[None, :]
        np.fill_diagonal(G, 1.0)
        ct = d * t2.c[k]
        res = ct - G @ t2.alpha_t[k]
        assert t2.delta[k] == pytest.approx(np.linalg.norm(res) / np.linalg.norm(ct), rel=1e-10)
        assert t2.delta[k] > 0.0


@pytest.mark.parametrize("nu", [1, 3, 20])
def test_energy_identity(nu):
    """||e_k||_A^2 - ||e_{k+1}||_A^2 = 2 a~^T c~ - a~^T G a~ > 0 (each unit-
    diagonal GS coordinate step is an exact line minimisation of the energy)."""
    dims = (10, 9, 1)
    A = orc.stencil(orc.KIND_5PT2D, *dims)
    b = inputs.rhs_uniform(10, 9, 1, seed=3)
    lmin, lmax = inputs.analytic_bounds("5pt", 10, 9)
    K = 6
    xs = [np.zeros(A.n)]
    for k in range(1, K + 1):
        x, tr = orc.sstep_cg(A, lmin, lmax, 4, nu, b, rtol=0.0, max_outer=k)
        xs.append(x)
    f = [-0.5 * x @ (b + (b - orc.apply(A, x))) for x in xs]     # f(x) = 1/2 x'Ax - b'x
    for k in range(K):
        drop = 2 * (f[k] - f[k + 1])
        assert drop > 0
        assert abs(drop - tr.energy[k]) <= 1e-12 * max(1.0, abs(drop)) + 1e-13 * abs(f[0])


def test_cfg1_matches_dense_direct_solve():
    """BASELINE cfg 1 (2D 5-pt 64x64, s=8, nu=20, rtol 1e-8) vs a dense direct
    solve: ||x - x*|| / ||x*|| <= kappa(M^-1 A) * rtol and the true residual
    ||b - Ax|| <= rtol ||b|| (1 + 1e-6)."""
    nx = ny = 64
    A = orc.stencil(orc.KIND_5PT2D, nx, ny, 1)
    b = inputs.rhs_uniform(nx, ny, 1, seed=42)
    lmin, lmax = inputs.analytic_bounds("5pt", nx, ny)
    x, tr = orc.sstep_cg(A, lmin, lmax, 8, 20, b, rtol=1e-8, max_outer=1000)
    assert tr.converged and not tr.breakdown
    T = 2 * np.eye(nx) - np.eye(nx, k=1) - np.eye(nx, k=-1)
    M = np.kron(np.eye(ny), T) + np.kron(T, np.eye(nx))
    xstar = np.linalg.solve(M, b)
    kappa = lmax / lmin
    assert np.linalg.norm(x - xstar) <= kappa * 1e-8 * np.linalg.norm(xstar)
    assert np.linalg.norm(b - M @ x) <= 1e-8 * np.linalg.norm(b) * (1 + 1e-6)
    # recurrence residual vs true residual
    assert abs(tr.relres[tr.outer] - np.linalg.norm(b - M @ x) / np.linalg.norm(b)) < 1e-12
    assert 40 <= tr.outer <= 300


def test_zero_rhs_converges_immediately():
    A = orc.stencil(orc.KIND_7PT, 4, 4, 4)
    x, tr = orc.sstep_cg(A, 0.1, 1.9, 4, 5, np.zeros(64), rtol=1e-8, max_outer=10)
    assert tr.converged and tr.outer == 0 and np.all(x == 0)


def test_nonzero_x0_restart_equivalence():
    """Resuming from x_k reproduces the uninterrupted run (restart form is
    memoryless except for x), up to recomputing r = b - A x_k."""
    dims = (8, 8, 8)
    A = orc.stencil(orc.KIND_7PT, *dims)
    b = inputs.rhs_uniform(*dims, seed=9)
    lmin, lmax = inputs.analytic_bounds("7pt", *dims)
    x6, _ = orc.sstep_cg(A, lmin, lmax, 5, 10, b, rtol=0.0, max_outer=6)
    x3, _ = orc.sstep_cg(A, lmin, lmax, 5, 10, b, rtol=0.0, max_outer=3)
    x6b, _ = orc.sstep_cg(A, lmin, lmax, 5, 10, b, x0=x3, rtol=0.0, max_outer=3)
    assert np.linalg.norm(x6b - x6) <= 1e-10 * np.linalg.norm(x6)


def test_classical_pcg_reference():
    dims = (16, 16, 1)
    A = orc.stencil(orc.KIND_5PT2D, *dims)
    b = inputs.rhs_uniform(*dims, seed=1)
    x, it = orc.pcg(A, b, rtol=1e-10)
    assert np.linalg.norm(b - orc.apply(A, x)) <= 1e-10 * np.linalg.norm(b) * 1.0001
    assert it <= 16 * 16


# ---------------------------------------------------------------------------
# NEXT-2 variants on the same boundary: exact Cholesky Gram
# solve and the monomial basis

def test_cholesky_worked_example(golden):
    """With the exact Gram solve one restart step on A = diag(1,3), s = n = 2
    reaches the nu -> infinity limit of the worked example, x_1 = [1, 1/3]."""
    g = golden["restart_sstep_diag13"]
    A = diag_csr(g["A_diag"])
    b = np.array(g["b"])
    x, tr = orc.sstep_cg(A, 1.0, 3.0, 2, 1, b, rtol=0.0, max_outer=1, D=np.ones(2), gram_solver="cholesky")
    assert np.allclose(x, g["x_limit"], rtol=1e-15, atol=0)
    # alpha~ solves G a~ = c~ with G = [[1, 1/2], [1/2, 1]], c~ = [1, 0]: a~ = [4/3, -2/3]
    assert np.allclose(tr.alpha_t[0], [4.0 / 3.0, -2.0 / 3.0], rtol=1e-15)
    assert tr.delta[0] <= 1e-15


def _dense(A):
    n = A.n
    return np.column_stack([orc.apply(A, e) for e in np.eye(n)])


def test_monomial_basis_is_matrix_powers():
    """p_j = (M^{-1}A)^j r, by the definition (dense matrix powers, n = 60)."""
    A = orc.stencil(orc.KIND_5PT2D, 6, 10)
    D = orc.diag(A)
    r = inputs.rhs_uniform(6, 10, 1, seed=3)
    P, W = orc.monomial_basis(A, D, 5, r)
    Md = _dense(A) / D[:, None]
    for j in range(5):
        ref = np.linalg.matrix_power(Md, j) @ r
        assert np.allclose(P[j], ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())
        assert np.allclose(W[j], _dense(A) @ ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("basis", ["chebyshev", "monomial"])
def test_full_krylov_space_exact(basis):
    """s = n with the exact Gram solve: the basis spans R^n, so one outer step
    gives A^{-1} b (dense direct solve), for either basis.  The tolerance is
    kappa(G) eps: the monomial Gram matrix is far worse conditioned
    (PAPER.md:31 kappa(G) = O(kappa(M^{-1}A)^{s-1})), the Chebyshev one is not."""
    A = orc.stencil(orc.KIND_5PT2D, 3, 2)      # n = 6
    b = inputs.rhs_uniform(3, 2, 1, seed=11)
    lmin, lmax = inputs.analytic_bounds("5pt", 3, 2, 1)
    x, tr = orc.sstep_cg(A, lmin, lmax, 6, 1, b, rtol=0.0, max_outer=1, gram_solver="cholesky", basis=basis)
    xs = np.linalg.solve(_dense(A), b)
    tol = 1e-12 if basis == "chebyshev" else 1e-7
    assert np.linalg.norm(x - xs) <= tol * np.linalg.norm(xs)


def test_fgs_many_sweeps_equals_cholesky_mode():
    """nu_infinity FGS sweeps (R20) and the Cholesky mode give the same outer
    iterates when kappa(G) is small (s = 4 on a 2D 16^2 Laplacian)."""
    A = orc.stencil(orc.KIND_5PT2D, 16, 16)
    b = inputs.rhs_uniform(16, 16, 1, seed=42)
    lmin, lmax = inputs.analytic_bounds("5pt", 16, 16, 1)
    x1, t1 = orc.sstep_cg(A, lmin, lmax, 4, 400, b, rtol=0.0, max_outer=5)
    x2, t2 = orc.sstep_cg(A, lmin, lmax, 4, 1, b, rtol=0.0, max_outer=5, gram_solver="cholesky")
    assert np.linalg.norm(x1 - x2) <= 1e-10 * np.linalg.norm(x2)
    assert np.max(np.abs(t1.alpha[:5] - t2.alpha[:5])) <= 1e-9 * np.max(np.abs(t2.alpha[:5]))


def test_cfg2_count_sensitivity():
    """BASELINE cfg 2 (128^3 7-point, s = 16, nu = 25, rtol 1e-8): perturbing b
    by one ulp (relative 2.2e-16, random signs) changes the oracle's own outer
    count by more than 1 -- the residual history oscillates near rtol and
    rounding differences grow ~1e3x per 20 outer iterations.  This pins the
    reading R22: the north_star 'outer count +-1' binds only where
    the iteration is not chaotic (cfg 1 and the reduced shapes, which the GPU
    tests hold to +-1), not at cfg 2 full size."""
    n, s, nu = 128, 16, 25
    A = orc.stencil(orc.KIND_7PT, n, n, n)
    b = inputs.rhs_uniform(n, n, n, seed=42)
    lmin, lmax = inputs.analytic_bounds("7pt", n, n, n)
    _, t0 = orc.sstep_cg(A, lmin, lmax, s, nu, b, rtol=1e-8, max_outer=3000)
    rng = np.random.default_rng(0)
    bp = b * (1 + 2.2e-16 * rng.choice([-1.0, 1.0], size=b.size))
    _, t1 = orc.sstep_cg(A, lmin, lmax, s, nu, bp, rtol=1e-8, max_outer=3000)
    assert t0.converged and t1.converged
    assert abs(t0.outer - t1.outer) > 1, (t0.outer, t1.outer)
    # and the residual histories agree early, then separate
    k = min(t0.outer, t1.outer)
    assert abs(t0.relres[10] - t1.relres[10]) <= 1e-10 * t0.relres[10]
    assert np.max(np.abs(t0.relres[k - 10:k] - t1.relres[k - 10:k]) / t0.relres[k - 10:k]) > 1e-3


def test_restart_from_recurrence_residual_is_outer_k():
    """b := r_k (the oracle's recurrence residual after k outer iterations),
    x_0 = 0 makes outer 0 of the restart bitwise identical to outer k of the
    original solve (basis, Gram block, alpha): the GPU deep-parity tests
    (tests/test_gpu_deep_parity.py) rely on this to give both sides
    identical inputs at any depth."""
    A = orc.stencil(orc.KIND_7PT, 13, 11, 9)
    b = inputs.rhs_uniform(13, 11, 9, seed=42)
    lmin, lmax = inputs.analytic_bounds("7pt", 13, 11, 9)
    s, nu, k = 6, 10, 7
    _, trk = orc.sstep_cg(A, lmin, lmax, s, nu, b, rtol=0.0, max_outer=k + 1, dump_iter=k)
    rk = trk.P[0].copy()
    _, tr1 = orc.sstep_cg(A, lmin, lmax, s, nu, rk, rtol=0.0, max_outer=1, dump_iter=0)
    assert np.array_equal(tr1.P, trk.P) and np.array_equal(tr1.W, trk.W)
    assert np.array_equal(tr1.ghat[0], trk.ghat[k]) and np.array_equal(tr1.c[0], trk.c[k])
    assert np.array_equal(tr1.alpha_t[0], trk.alpha_t[k]) and np.array_equal(tr1.alpha[0], trk.alpha[k])
    assert tr1.delta[0] == trk.delta[k]
