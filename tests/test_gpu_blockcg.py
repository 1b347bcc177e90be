"""GPU parity of the block-conjugate s-step CG mode (SSCG_OPT_BLOCKCG; SURVEY
§8(f) NEXT-2, R24) against the oracle's block mode (pinned in
tests/test_oracle_blockcg.py): outer 0 at the north_star tolerances (no
previous block: the restart step), the conjugated Gram systems of later outer
iterations within the drift budget (each side carries its own Q_{k-1}),
x after 10 outer iterations to 1e-8, full solves to the oracle's count +-1,
and the decomposition paths (in-process slabs, the one-rank NCCL mode)."""
import numpy as np
import pytest

import oracle as orc
from gpu_cases import (TOL_ALPHA, TOL_ALPHA_DRIFT, TOL_GRAM, TOL_GRAM_DRIFT, TOL_X10, Problem, rel_inf)

pytestmark = pytest.mark.gpu

CASES = [("7pt", 40, 36, 33, 8, 20, "cholesky"), ("7pt", 40, 36, 33, 16, 25, "cholesky"),
         ("7pt", 33, 17, 19, 5, 10, "fgs"), ("27pt", 24, 22, 20, 8, 30, "cholesky"),
         ("varcoef7", 24, 22, 20, 8, 20, "cholesky"), ("5pt", 64, 64, 1, 8, 20, "cholesky"),
         ("7pt", 26, 18, 21, 12, 20, "cholesky")]   # W-free with three 8-row blocks (2s = 24)


def _ids(c):
    return "-".join(map(str, c))


def _oracle(P, gs, max_outer, rtol=0.0):
    return orc.sstep_cg(P.A, P.lmin, P.lmax, P.s, P.nu, P.b, rtol=rtol, max_outer=max_outer, gram_solver=gs,
                        block=True)


@pytest.mark.parametrize("wfree", ["1", "0"], ids=["wfree", "storedW"])
@pytest.mark.parametrize("case", CASES, ids=_ids)
def test_block_ten_outer(case, wfree, monkeypatch):
    """With W_k recovered (the default for constant diagonals: the 2s-row Gram
    pass K2R BLK and K5B recover W_k from P_k, Z' stays stored) and with the
    stored W."""
    import paper_2512_09642_b200 as sscg
    monkeypatch.setenv("SSCG_WFREE", wfree)
    kind, nx, ny, nz, s, nu, gs = case
    P = Problem(kind, nx, ny, nz, s, nu, lanczos=(kind in ("27pt", "varcoef7")))
    x_or, tr = _oracle(P, gs, 10)
    with P.gpu_solver(gram_solver=gs, block=True) as S:
        w_free = wfree == "1" and kind in ("7pt", "27pt") and s <= 16 and nx % 2 == 0   # (K1T stencils)
        assert S.query(sscg.QUERY_GRAM_VECTORS) == (3 * s + 1 if w_free else 4 * s)
        assert S.query(sscg.QUERY_UPDATE_VECTORS) == (5 * s + 4 if w_free else 6 * s + 3)
        x = S.solve(P.b_gpu(), rtol=0.0, max_outer=10).cpu().numpy()
        st = S.stats()
        assert st.outer_iterations == 10
        # each side carries its own Q_{k-1}: with inexact FGS solves e = Q'^T r_k is
        # O(delta) instead of 0 and B = G'^{-1} C amplifies the two sides' rounding
        # differences by kappa(G'), so the drift budget binds over the first outer
        # iterations only (R24); x after 10 outer is held to 1e-8 either way
        kmax = 10 if gs == "cholesky" else 5
        for k in range(kmax):
            g = S.inspect(sscg.INSPECT_GRAM, k)
            G, c = g[: s * s].reshape(s, s), g[s * s:]
            tol = TOL_GRAM if k == 0 else TOL_GRAM_DRIFT
            eg = np.max(np.abs(G - tr.gconj[k])) / np.max(np.abs(tr.gconj[k]))
            ec = np.max(np.abs(c - tr.cconj[k])) / np.max(np.abs(tr.cconj[k]))
            assert eg <= tol and ec <= tol, (k, eg, ec)
            al = S.inspect(sscg.INSPECT_ALPHA, k)
            assert rel_inf(al, tr.alpha[k]) <= (TOL_ALPHA if k == 0 else TOL_ALPHA_DRIFT), (k, rel_inf(al, tr.alpha[k]))
        assert np.allclose(st.relres_history, tr.relres[:11], rtol=1e-7, atol=0)
    ex = np.linalg.norm(x - x_or) / np.linalg.norm(x_or)
    assert ex <= TOL_X10, ex


@pytest.mark.parametrize("case", [("7pt", 40, 36, 33, 16, 25), ("5pt", 64, 64, 1, 8, 20), ("27pt", 24, 24, 24, 16, 30)],
                         ids=_ids)
def test_block_full_solve(case):
    """Full solve with exact (Cholesky) Gram solves: outer count equal to the
    oracle's +-1, true residual <= rtol, and well below the restart form's count."""
    kind, nx, ny, nz, s, nu = case
    P = Problem(kind, nx, ny, nz, s, nu, lanczos=(kind == "27pt"))
    _, tr = _oracle(P, "cholesky", 2000, rtol=1e-8)
    assert tr.converged
    with P.gpu_solver(gram_solver="cholesky", block=True) as S:
        x = S.solve(P.b_gpu(), rtol=1e-8, max_outer=2000).cpu().numpy()
        st = S.stats()
    assert st.converged and abs(st.outer_iterations - tr.outer) <= 1, (st.outer_iterations, tr.outer)
    res = np.linalg.norm(P.b - orc.apply(P.A, x)) / np.linalg.norm(P.b)
    assert res <= 1e-8 * (1 + 1e-6), res
    with P.gpu_solver(gram_solver="cholesky") as S:
        S.solve(P.b_gpu(), rtol=1e-8, max_outer=2000)
        restart = S.stats().outer_iterations
    assert st.outer_iterations < restart, (st.outer_iterations, restart)
    if restart >= 10:   # long enough a solve for the Krylov advantage to show
        assert 2 * st.outer_iterations <= restart, (st.outer_iterations, restart)


@pytest.mark.parametrize("env", [{}, {"SSCG_NCCL_SELF": "1"}, {"SSCG_K1_MP3": "1"}], ids=["slabs", "nccl_self", "mp3"])
def test_block_slabs(env, monkeypatch):
    """Three in-process slabs (per-slab [P | Q'], one summed 2s-row block), also
    through the one-rank NCCL mode (one allreduce per outer) and with K1M
    triples: equal to the one-slab block solve to rounding."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    P = Problem("7pt", 40, 36, 33, 8, 20)
    with P.gpu_solver(gram_solver="cholesky", block=True) as S1:
        x1 = S1.solve(P.b_gpu(), rtol=0.0, max_outer=6).cpu().numpy()
    with P.gpu_solver(slabs=3, gram_solver="cholesky", block=True) as S:
        x = S.solve(P.b_gpu(), rtol=0.0, max_outer=6).cpu().numpy()
        st = S.stats()
    assert np.linalg.norm(x - x1) <= 1e-10 * np.linalg.norm(x1)
    if env.get("SSCG_NCCL_SELF") == "1":
        assert st.allreduces == 7


def test_block_option_toggle():
    """Switching the mode off again restores the restart form exactly."""
    import paper_2512_09642_b200 as sscg
    P = Problem("7pt", 33, 17, 19, 5, 10)
    with P.gpu_solver() as S0:
        x0 = S0.solve(P.b_gpu(), rtol=0.0, max_outer=5).cpu().numpy()
    with P.gpu_solver(block=True) as S:
        xb = S.solve(P.b_gpu(), rtol=0.0, max_outer=5).cpu().numpy()
        S.set_option(sscg.OPT_BLOCKCG, 0)
        x = S.solve(P.b_gpu(), rtol=0.0, max_outer=5).cpu().numpy()
    assert np.array_equal(x, x0)
    assert not np.array_equal(xb, x0)
