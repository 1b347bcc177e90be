"""Pins for the oracle's block-conjugate s-step CG (
SPEC.md:349, 358; R24): each outer block Q_k = P_k - Q_{k-1} B_k is
made A-conjugate to the previous one, B_k = G_{k-1}^{-1} (A Q_{k-1})^T P_k.

What fixes it independently of its own formulas:
  * outer 0 has no previous block: identical to the restart form;
  * with exact Gram solves the blocks span K_{Ks}(A, r_0) and the iterate is
    the A-norm-optimal one there -- i.e. classical CG after K*s iterations
    (a constant Jacobi diagonal does not change the Krylov space); s = 1 is CG
    step by step;
  * G_k = Q_k^T A Q_k and c_k = Q_k^T r_k (checked against the explicitly
    formed block) and Q_k is A-orthogonal to Q_{k-1};
  * s = n: one outer iteration with an exact solve is a direct solve."""
import numpy as np
import pytest

import inputs
import oracle as orc


def _cg(A, b, iters):
    """Unpreconditioned CG after `iters` iterations (orc_pcg with D = 1)."""
    x, _ = orc.pcg(A, b, rtol=0.0, max_iter=iters, D=np.ones(A.n))
    return x


def test_outer0_equals_restart():
    A = orc.stencil(orc.KIND_7PT, 11, 9, 8)
    b = inputs.rhs_uniform(11, 9, 8, seed=42)
    lmin, lmax = inputs.analytic_bounds("7pt", 11, 9, 8)
    for gs in ("fgs", "cholesky"):
        x1, t1 = orc.sstep_cg(A, lmin, lmax, 6, 10, b, rtol=0.0, max_outer=1, gram_solver=gs)
        x2, t2 = orc.sstep_cg(A, lmin, lmax, 6, 10, b, rtol=0.0, max_outer=1, gram_solver=gs, block=True)
        assert np.array_equal(x1, x2)
        assert np.array_equal(t1.alpha[0], t2.alpha[0]) and np.array_equal(t2.gconj[0], t2.ghat[0])


@pytest.mark.parametrize("s,K", [(1, 12), (2, 6), (4, 4)])
def test_exact_block_cg_is_cg(s, K):
    """Exact solves: K outer iterations of block-conjugate s-step CG = K*s
    iterations of classical CG (2D Laplacian, constant Jacobi diagonal)."""
    A = orc.stencil(orc.KIND_5PT2D, 12, 11, 1)
    b = inputs.rhs_uniform(12, 11, 1, seed=7)
    lmin, lmax = inputs.analytic_bounds("5pt", 12, 11)
    xb, tr = orc.sstep_cg(A, lmin, lmax, s, 1, b, rtol=0.0, max_outer=K, gram_solver="cholesky", block=True)
    xc = _cg(A, b, K * s)
    assert not tr.breakdown
    assert np.linalg.norm(xb - xc) <= 1e-9 * np.linalg.norm(xc), np.linalg.norm(xb - xc) / np.linalg.norm(xc)
    # and the restart form is NOT CG beyond its first outer iteration (the pin discriminates)
    if K > 1:
        xr, _ = orc.sstep_cg(A, lmin, lmax, s, 1, b, rtol=0.0, max_outer=K, gram_solver="cholesky")
        assert np.linalg.norm(xr - xc) > 1e-6 * np.linalg.norm(xc)


def test_conjugated_system_is_the_block_gram():
    """G_k, c_k of the trace = Q_k^T A Q_k, Q_k^T r_k of the explicitly formed
    block (numpy here, from the raw bases the oracle dumps), and Q_k is
    A-orthogonal to Q_{k-1} (exact solves)."""
    A = orc.stencil(orc.KIND_7PT, 9, 8, 7)
    b = inputs.rhs_uniform(9, 8, 7, seed=3)
    lmin, lmax = inputs.analytic_bounds("7pt", 9, 8, 7)
    s = 4
    x0, t0 = orc.sstep_cg(A, lmin, lmax, s, 1, b, rtol=0.0, max_outer=1, gram_solver="cholesky", block=True,
                          dump_iter=0)
    Q0, Z0 = t0.P.T, t0.W.T                               # outer 0: Q = P
    x1, t1 = orc.sstep_cg(A, lmin, lmax, s, 1, b, rtol=0.0, max_outer=1, gram_solver="cholesky", block=True,
                          dump_iter=1)
    _, tb = orc.sstep_cg(A, lmin, lmax, s, 1, b, rtol=0.0, max_outer=2, gram_solver="cholesky", block=True,
                         dump_iter=1)
    P1, W1 = tb.P.T, tb.W.T                               # raw basis of r_1
    r1 = b - orc.apply(A, x0)
    B = np.linalg.solve(Q0.T @ Z0, Z0.T @ P1)
    Q1, Z1 = P1 - Q0 @ B, W1 - Z0 @ B
    G1 = Q1.T @ Z1
    assert np.max(np.abs(tb.gconj[1] - G1)) <= 1e-10 * np.max(np.abs(G1))
    assert np.max(np.abs(tb.cconj[1] - Q1.T @ r1)) <= 1e-10 * np.max(np.abs(Q1.T @ r1))
    assert np.max(np.abs(Q0.T @ Z1)) <= 1e-10 * np.max(np.abs(G1))   # A-conjugate blocks


def test_s_equals_n_direct_solve():
    n = 6
    A = orc.stencil(orc.KIND_5PT2D, 3, 2, 1)
    b = inputs.rhs_uniform(3, 2, 1, seed=1)
    lmin, lmax = inputs.analytic_bounds("5pt", 3, 2)
    x, tr = orc.sstep_cg(A, lmin, lmax, n, 1, b, rtol=0.0, max_outer=1, gram_solver="cholesky", block=True)
    assert not tr.breakdown
    Ad = np.array([orc.apply(A, e) for e in np.eye(n)]).T
    xs = np.linalg.solve(Ad, b)
    assert np.linalg.norm(x - xs) <= 1e-6 * np.linalg.norm(xs)


def test_block_converges_in_fewer_outers_with_exact_solves():
    """Context for DESIGN.md R24: with exact (Cholesky) Gram solves the
    block-conjugate form needs far fewer outer iterations than the restart
    form; with nu FGS sweeps (inexact alpha, so r_k is not orthogonal to
    Q_{k-1}) it is the restart form that converges faster -- the paper's
    choice."""
    A = orc.stencil(orc.KIND_7PT, 24, 24, 24)
    b = inputs.rhs_uniform(24, 24, 24, seed=42)
    lmin, lmax = inputs.analytic_bounds("7pt", 24, 24, 24)
    out = {}
    for gs in ("cholesky", "fgs"):
        for blk in (False, True):
            _, tr = orc.sstep_cg(A, lmin, lmax, 8, 20, b, rtol=1e-8, max_outer=2000, gram_solver=gs, block=blk)
            assert tr.converged
            out[(gs, blk)] = tr.outer
    assert out[("cholesky", True)] * 2 <= out[("cholesky", False)], out
    assert out[("fgs", False)] < out[("fgs", True)], out
