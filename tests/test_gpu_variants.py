"""GPU parity of the SURVEY §8(f) NEXT-1/NEXT-2 rows against the CPU oracle:
Lanczos spectral bounds, the exact Cholesky Gram solve
 and the monomial basis, all through the
C ABI on the same seeded inputs."""
import numpy as np
import pytest

import inputs
import oracle as orc
from gpu_cases import TOL_ALPHA, TOL_ALPHA_DRIFT, TOL_GRAM, TOL_GRAM_DRIFT, TOL_X10, Problem, assert_alpha, assert_gram

pytestmark = pytest.mark.gpu


LZ_CASES = [("7pt", 24, 20, 18, 1), ("27pt", 20, 18, 16, 1), ("varcoef7", 18, 16, 14, 1), ("7pt", 21, 19, 17, 3),
            ("varcoef7", 16, 14, 13, 4), ("5pt", 64, 64, 1, 1)]


@pytest.mark.parametrize("kind,nx,ny,nz,slabs", LZ_CASES, ids=lambda v: str(v))
def test_lanczos_bounds(kind, nx, ny, nz, slabs):
    """The first Lanczos coefficients agree with the oracle's to rounding
    (later ones drift: no reorthogonalisation amplifies rounding), and the
    widened extreme Ritz values of 50 steps agree to 1e-9 relative (converged
    extreme eigenvalues are insensitive to that drift)."""
    import torch
    P = Problem(kind, nx, ny, nz, 4, 5, bounds=(0.1, 1.9))
    lo, hi, m, al, be = orc.lanczos_bounds(P.A, 50, P.b, 0.05, tridiag=True)
    with P.gpu_solver(slabs=slabs) as S:
        glo, ghi, gal, gbe = S.estimate_bounds(torch.from_numpy(P.b).cuda(), 50, 0.05, tridiag=True)
    assert m == 50
    assert np.max(np.abs(gal[:8] - al[:8])) <= 1e-12 * np.max(np.abs(al))
    assert np.max(np.abs(gbe[:7] - be[:7])) <= 1e-12 * np.max(np.abs(be))
    assert abs(glo - lo) <= 1e-9 * lo and abs(ghi - hi) <= 1e-9 * hi
    if kind in ("7pt", "5pt"):   # inside the analytic interval after widening inward (Ritz values interlace)
        a_lo, a_hi = inputs.analytic_bounds(kind, nx, ny, nz)
        assert glo / 0.95 >= a_lo * (1 - 1e-12) and ghi / 1.05 <= a_hi * (1 + 1e-12)


def test_lanczos_then_solve_cfg3_shape():
    """Bounds from the GPU Lanczos, set on a context created without bounds,
    give the same solve as the oracle with the oracle's bounds (BASELINE cfg 3
    recipe at reduced size: 27-point, Lanczos-50 + 5 %, s = 16, nu = 30)."""
    import torch

    import paper_2512_09642_b200 as sscg
    nx, ny, nz, s, nu = 26, 24, 22, 16, 30
    P = Problem("27pt", nx, ny, nz, s, nu, lanczos=True)
    with sscg.Solver(sscg.Stencil("27pt", nx, ny, nz), 0.0, 0.0, s, nu) as S:
        with pytest.raises(sscg.SSCGError):
            S.solve(P.b_gpu(), rtol=0.0, max_outer=1)      # no bounds yet
        lo, hi = S.estimate_bounds(P.b_gpu(), 50, 0.05)
        assert abs(lo - P.lmin) <= 1e-9 * P.lmin and abs(hi - P.lmax) <= 1e-9 * P.lmax
        S.set_bounds(P.lmin, P.lmax)                        # identical inputs on both sides
        x = S.solve(P.b_gpu(), rtol=0.0, max_outer=10).cpu().numpy()
        x_or, tr = P.oracle(max_outer=10, dump_iter=10)
        assert_gram(S, tr, 0)
        assert_alpha(S, tr, 0)
    assert np.linalg.norm(x - x_or) <= TOL_X10 * np.linalg.norm(x_or)


@pytest.mark.parametrize("kind,nx,ny,nz,s", [("7pt", 30, 28, 26, 8), ("27pt", 20, 18, 17, 12), ("5pt", 64, 64, 1, 8),
                                             ("varcoef7", 18, 16, 15, 6)])
def test_cholesky_gram_solver(kind, nx, ny, nz, s):
    P = Problem(kind, nx, ny, nz, s, 1, lanczos=(kind in ("27pt", "varcoef7")))
    x_or, tr = P.oracle_ex(max_outer=8, gram_solver="cholesky")
    with P.gpu_solver(gram_solver="cholesky") as S:
        x = S.solve(P.b_gpu(), rtol=0.0, max_outer=8).cpu().numpy()
        assert_gram(S, tr, 0)
        assert_alpha(S, tr, 0)
        for k in range(1, 8):
            assert_gram(S, tr, k, tol=TOL_GRAM_DRIFT)
            assert_alpha(S, tr, k, tol=TOL_ALPHA_DRIFT)
        import paper_2512_09642_b200 as sscg
        assert S.inspect(sscg.INSPECT_DELTA, 0)[0] <= 1e-10    # exact solve: tiny Gram residual
    assert np.linalg.norm(x - x_or) <= TOL_X10 * np.linalg.norm(x_or)


def test_cholesky_worked_example(golden):
    """diag(1,3), s = n = 2: one exact step reaches x = [1, 1/3] (tests/golden)."""
    import torch

    import paper_2512_09642_b200 as sscg
    g = golden["restart_sstep_diag13"]
    dev = torch.device("cuda")
    op = sscg.CSR(torch.tensor([0, 1, 2], dtype=torch.int64, device=dev),
                  torch.tensor([0, 1], dtype=torch.int32, device=dev),
                  torch.tensor(g["A_diag"], dtype=torch.float64, device=dev))
    ones = torch.ones(2, dtype=torch.float64, device=dev)
    with sscg.Solver(op, g["lmin"], g["lmax"], 2, 1, diag_M=ones, gram_solver="cholesky") as S:
        x = S.solve(torch.tensor(g["b"], dtype=torch.float64, device=dev), rtol=0.0, max_outer=1)
        assert np.allclose(x.cpu().numpy(), g["x_limit"], rtol=1e-15, atol=0)


@pytest.mark.parametrize("kind,nx,ny,nz,s,solver", [("7pt", 24, 22, 20, 4, "fgs"), ("7pt", 24, 22, 20, 4, "cholesky"),
                                                    ("27pt", 16, 15, 14, 3, "fgs"), ("5pt", 40, 36, 1, 4, "cholesky")])
def test_monomial_basis(kind, nx, ny, nz, s, solver):
    P = Problem(kind, nx, ny, nz, s, 10, bounds=(0.1, 1.9))
    x_or, tr = P.oracle_ex(max_outer=6, dump_iter=0, gram_solver=solver, basis="monomial")
    with P.gpu_solver(gram_solver=solver, basis="monomial") as S:
        x = S.solve(P.b_gpu(), rtol=0.0, max_outer=6).cpu().numpy()
        assert_gram(S, tr, 0)
        assert_alpha(S, tr, 0, tol=TOL_ALPHA)
        for k in range(1, 6):
            assert_gram(S, tr, k, tol=TOL_GRAM_DRIFT)
    assert np.linalg.norm(x - x_or) <= TOL_X10 * np.linalg.norm(x_or)


def test_option_errors():
    import paper_2512_09642_b200 as sscg
    with sscg.Solver(sscg.Stencil("7pt", 8, 8, 8), 0.1, 1.9, 4, 4) as S:
        for key, val in ((sscg.OPT_GRAM_SOLVER, 7), (sscg.OPT_BASIS, -1), (9, 0)):
            with pytest.raises(sscg.SSCGError) as e:
                S.set_option(key, val)
            assert e.value.code == sscg.ERR_INVALID
        for lo, hi in ((0.0, 1.0), (1.0, 1.0), (2.0, 1.0)):
            with pytest.raises(sscg.SSCGError):
                S.set_bounds(lo, hi)


@pytest.mark.parametrize("kind,nx,ny,nz,s,solver", [("7pt", 30, 28, 26, 16, "fgs"), ("5pt", 64, 64, 1, 8, "fgs"),
                                                    ("7pt", 12, 12, 12, 40, "fgs"), ("27pt", 20, 18, 17, 12, "cholesky")])
def test_diagnostics_lnorm_delta(kind, nx, ny, nz, s, solver):
    """Per-outer diagnostics recorded by K4/K4C: ||L||_F of the scaled Gram
    matrix G = I + L + L^T (the quantity FGS convergence depends on,
    PAPER.md:24-25) and delta_k = ||c~ - G a~|| / ||c~||,
    against the same quantities from the oracle's Gram trace at outer 0."""
    import paper_2512_09642_b200 as sscg
    bounds = (0.02, 2.2) if s == 40 else None
    P = Problem(kind, nx, ny, nz, s, 25, bounds=bounds, lanczos=(kind == "27pt"))
    x_or, tr = P.oracle_ex(max_outer=3, gram_solver=solver)
    with P.gpu_solver(gram_solver=solver) as S:
        S.solve(P.b_gpu(), rtol=0.0, max_outer=3)
        d, G, ct = orc.scale(tr.ghat[0], tr.c[0])
        ln_or = np.linalg.norm(np.tril(G, -1))
        ln = S.inspect(sscg.INSPECT_LNORM, 0)[0]
        assert abs(ln - ln_or) <= 1e-12 * ln_or
        de = S.inspect(sscg.INSPECT_DELTA, 0)[0]
        if solver == "fgs":
            assert abs(de - tr.delta[0]) <= 1e-6 * tr.delta[0]
        else:
            assert de <= 1e-10 and tr.delta[0] <= 1e-10
        st = S.stats()
        assert np.allclose(st.delta_history[:3], [S.inspect(sscg.INSPECT_DELTA, k)[0] for k in range(3)], rtol=0)


@pytest.mark.parametrize("kind,nx,ny,nz,s", [("7pt", 30, 28, 26, 16), ("5pt", 64, 64, 1, 8), ("7pt", 24, 20, 18, 24),
                                             ("27pt", 20, 18, 17, 5)])
def test_diagnostics_kappa(kind, nx, ny, nz, s):
    """kappa(G) of the Ruhe-scaled Gram matrix per outer (SSCG_OPT_DIAGNOSTICS),
    against numpy's condition number of the oracle's scaled G at outer 0."""
    import paper_2512_09642_b200 as sscg
    P = Problem(kind, nx, ny, nz, s, 20, lanczos=(kind == "27pt"))
    x_or, tr = P.oracle(max_outer=2, dump_iter=0)
    with P.gpu_solver() as S:
        S.set_option(sscg.OPT_DIAGNOSTICS, 1)
        S.solve(P.b_gpu(), rtol=0.0, max_outer=2)
        # ||P_0||_F and the budget term delta_0 ||A|| ||P_0||_F, ||A|| = Gershgorin
        # bound = 2 x centre for these graph-Laplacian stencils
        pf = np.sqrt(sum(np.dot(p, p) for p in tr.P))
        assert abs(S.inspect(sscg.INSPECT_PNORM, 0)[0] - pf) <= 1e-12 * pf
        anorm = 2.0 * {"5pt": 4.0, "7pt": 6.0, "27pt": 26.0}[kind]
        b0 = tr.delta[0] * anorm * pf
        assert abs(S.inspect(sscg.INSPECT_BUDGET, 0)[0] - b0) <= 1e-6 * b0
        st = S.stats()
        assert st.budget == pytest.approx(S.inspect(sscg.INSPECT_BUDGET, 0)[0] + S.inspect(sscg.INSPECT_BUDGET, 1)[0],
                                          rel=1e-14)
        d, G, ct = orc.scale(tr.ghat[0], tr.c[0])
        ev = np.linalg.eigvalsh(G)
        assert ev[0] > 0
        k_ref = ev[-1] / ev[0]
        k_gpu = S.inspect(sscg.INSPECT_KAPPA, 0)[0]
        # eigenvalues of G are perturbed by ~eps ||G|| (Weyl): relative accuracy of kappa ~ eps kappa
        assert abs(k_gpu - k_ref) <= max(1e-10, 1e-14 * k_ref) * k_ref, (k_gpu, k_ref)
        assert S.inspect(sscg.INSPECT_KAPPA, 1)[0] > 1.0
