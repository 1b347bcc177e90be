"""Pins for the oracle's FGS inner solve (§3) and its
equivalence with A-norm MGS (§5 Thm Algebraic Equivalence)."""
import math

import numpy as np
import pytest

import inputs
import oracle as orc

EPS = np.finfo(float).eps


def rand_unit_spd(s, rng, cond_target=None):
    Q, _ = np.linalg.qr(rng.standard_normal((s, s)))
    lam = np.exp(rng.uniform(0, math.log(cond_target or 100.0), s))
    M = (Q * lam) @ Q.T
    d = 1 / np.sqrt(np.diag(M))
    G = d[:, None] * M * d[None, :]
    np.fill_diagonal(G, 1.0)
    return (G + G.T) / 2


def test_spec_fgs_examples(golden):
    g = golden["fgs_2x2"]
    G, rhs = np.array(g["G"]), np.array(g["rhs"])
    a1, h = orc.fgs(G, rhs, 1, hist=True)
    assert np.array_equal(a1, g["sweep1"])
    assert np.array_equal(rhs - G @ a1, g["residual1"])
    assert np.array_equal(orc.fgs(G, rhs, 2), g["sweep2"])
    assert np.allclose(orc.fgs(G, rhs, 60), g["limit"], rtol=0, atol=1e-15)
    assert h[0] == pytest.approx(math.sqrt(2)) and h[1] == pytest.approx(0.25)


def test_identity_gram_one_sweep_exact():
    rhs = np.arange(1.0, 6.0)
    assert np.array_equal(orc.fgs(np.eye(5), rhs, 1), rhs)


@pytest.mark.parametrize("s", [3, 8, 16, 32])
def test_residual_structure(s):
    """PAPER.md:64-71 (Prop. FGS Residual Structure):
    r^(1) = -L^T alpha^(1);  r^(v+1) = -L^T alpha^(v+1) + L^T alpha^(v)."""
    rng = np.random.default_rng(s)
    G = rand_unit_spd(s, rng)
    rhs = rng.standard_normal(s)
    U = np.triu(G, 1)       # L^T
    a = [np.zeros(s)] + [orc.fgs(G, rhs, v) for v in range(1, 6)]
    scale = np.abs(rhs).max() + np.abs(G).max() * max(np.abs(x).max() for x in a)
    assert np.max(np.abs((rhs - G @ a[1]) + U @ a[1])) < 1e-13 * scale
    for v in range(1, 5):
        r = rhs - G @ a[v + 1]
        assert np.max(np.abs(r - (-U @ a[v + 1] + U @ a[v]))) < 1e-13 * scale


@pytest.mark.parametrize("s", [4, 10, 20])
def test_fgs_converges_to_cholesky(s):
    """nu -> inf FGS equals the dense Cholesky solve (north_star; R20: nu_inf =
    ceil(ln 1e-14 / ln rho(T)), kappa(G) <= 1e4)."""
    rng = np.random.default_rng(100 + s)
    G = rand_unit_spd(s, rng, cond_target=1e3)
    rhs = rng.standard_normal(s)
    xs = orc.cholesky_solve(G, rhs)
    assert np.allclose(xs, np.linalg.solve(G, rhs), rtol=1e-10, atol=0)   # pins Cholesky itself
    L = np.tril(G, -1)
    T = -np.linalg.solve(np.eye(s) + L, L.T)
    rho = max(abs(np.linalg.eigvals(T)))
    nu = int(math.ceil(math.log(1e-14) / math.log(rho))) + 50
    a = orc.fgs(G, rhs, nu)
    assert np.max(np.abs(a - xs)) <= 1e-10 * np.max(np.abs(xs))


@pytest.mark.parametrize("seed", range(6))
def test_error_contraction_forms(seed):
    """Corrected Lemma (R16): the *error* obeys
    ||e^(v)||_2 <= ||T||_2^v ||e^(0)||_2 and ||e^(v)||_G strictly decreases."""
    rng = np.random.default_rng(seed)
    s = 12
    G = rand_unit_spd(s, rng, cond_target=50.0)
    rhs = rng.standard_normal(s)
    xs = np.linalg.solve(G, rhs)
    L = np.tril(G, -1)
    T = -np.linalg.solve(np.eye(s) + L, L.T)
    nT = np.linalg.norm(T, 2)
    e0 = np.linalg.norm(xs)
    prevG = math.inf
    for v in range(1, 15):
        e = xs - orc.fgs(G, rhs, v)
        assert np.linalg.norm(e) <= nT ** v * e0 * (1 + 1e-10) + 1e-13
        eG = math.sqrt(e @ G @ e)
        assert eG < prevG or eG < 1e-13
        prevG = eG


@pytest.mark.parametrize("s", [5, 16, 20])
def test_backward_stability_one_sweep(s):
    """PAPER.md:82-105 (Thm Backward Stability): the computed sweep satisfies
    (D+L) a~ = rhs - L^T a_prev + dr with ||dr|| <= eps C(s) (||rhs|| + ||D+L|| ||a~||),
    C(s) = O(s); we assert C(s) = 8 s."""
    rng = np.random.default_rng(s)
    G = rand_unit_spd(s, rng, cond_target=1e3)
    rhs = rng.standard_normal(s)
    a1 = orc.fgs(G, rhs, 1)
    DL = np.tril(G)
    dr = DL @ a1 - rhs
    bound = EPS * 8 * s * (np.linalg.norm(rhs) + np.linalg.norm(DL, 2) * np.linalg.norm(a1))
    assert np.linalg.norm(dr) <= bound


@pytest.mark.parametrize("kind,dims,s,seed", [("7pt", (8, 7, 6), 6, 0), ("7pt", (6, 6, 6), 10, 1),
                                              ("27pt", (6, 5, 7), 8, 2), ("5pt", (16, 12, 1), 8, 3)])
def test_one_sweep_equals_mgs(kind, dims, s, seed):
    """PAPER.md:172-223 (Thm Algebraic Equivalence): one FGS sweep on
    G a = P~^T A v with G = P~^T A P~, a^(0) = 0, equals MGS of v against P~
    in the A-inner product (R18: rhs uses A v)."""
    K = {"5pt": orc.KIND_5PT2D, "7pt": orc.KIND_7PT, "27pt": orc.KIND_27PT}[kind]
    A = orc.stencil(K, *dims)
    rng = np.random.default_rng(seed)
    r = rng.uniform(-1, 1, A.n)
    lmin, lmax = inputs.analytic_bounds(kind, *dims)
    P, W = orc.chebyshev_basis(A, orc.diag(A), lmin, lmax, s, r)
    Ghat, c = orc.gram(P, W)
    d, G, _ = orc.scale(Ghat, c)
    Pt = P * d[:, None]
    v = rng.uniform(-1, 1, A.n)
    Av = orc.apply(A, v)
    rhs = np.array([orc.dot(Pt[j], Av) for j in range(s)])
    a1 = orc.fgs(G, rhs, 1)
    gamma, _ = orc.mgs_anorm(A, Pt, v)
    assert np.max(np.abs(a1 - gamma)) <= 1e-12 * max(1.0, np.max(np.abs(gamma)))
