"""GPU parity deep in the solve, at the north_star tolerances.

Both sides get IDENTICAL inputs at outer iteration k: the oracle runs k outer
iterations on the seeded b and returns its recurrence residual r_k (the p_0 of
its outer iteration k); then the oracle and the CUDA path each
start from b := r_k, x_0 = 0.  The basis, Gram block and alpha of that outer
iteration are then the ones of outer k of the original solve, computed from
the same input on both sides, so the strict tolerances of BASELINE.json's
north_star bind (R15): basis p_j / w_j 1e-12 (normwise inf,
relative), Gram 1e-11 of max|Ghat| (and c likewise), alpha~ / alpha 1e-10.
The update is checked too: x_1 of the restart (= x_{k+1} - x_k of the solve)
to 1e-10 relative.

k runs over {10, 50, a few iterations before convergence} and every operator
kind, under the default schedule and with each schedule switch forced both
ways (triples K1M, pairs K1F/K1FV, single steps K1T, the stored-W Gram K2/K2D
vs the W-free K2R/K2S, the recurrence vs stored-W update).  Under the W-free
schedule the product path never stores w_j (j < s-1): K2R recovers it per
point inside the Gram pass and the Gram block checks that; the w_j read back
here for j < s-1 come from the inspect hook's recovery kernel (k_wrec, the
same per-point formula); w_{s-1} is the stored SpMV output, or, under the
w_{s-1} fold (7-point default: K2R and K5 form it from p_{s-1}), the inspect
hook's single step over p_{s-1}."""
import numpy as np
import pytest

import inputs
import oracle as orc
from gpu_cases import TOL_ALPHA, TOL_BASIS, TOL_GRAM, Problem, assert_alpha, assert_basis, assert_gram, rel_inf

pytestmark = pytest.mark.gpu

# kind, nx, ny, nz, s, nu  (reduced BASELINE shapes with ragged tiles; cfg 1 at full size)
SHAPES = {
    "cfg1": ("5pt", 64, 64, 1, 8, 20),
    "7pt": ("7pt", 40, 36, 33, 16, 25),
    "7pt_mid": ("7pt", 88, 72, 66, 16, 25),       # long enough a solve for k = 50
    "cfg2": ("7pt", 128, 128, 128, 16, 25),       # BASELINE cfg 2 at full size
    "27pt": ("27pt", 30, 28, 26, 16, 30),
    "varcoef7": ("varcoef7", 24, 22, 20, 8, 20),
    "7pt_odd": ("7pt", 33, 17, 19, 5, 10),
}

# schedule switches forced per operator kind; {} = the default schedule
SWITCHES = {
    "7pt": [{}, {"SSCG_WL_FOLD": "0"}, {"SSCG_K1_MP3": "1"}, {"SSCG_K1_MP3": "0", "SSCG_K1_FUSE": "1"}, {"SSCG_K1_FUSE": "0"},
            {"SSCG_WFREE": "0"}, {"SSCG_WFREE": "0", "SSCG_K2_DMMA": "1"}, {"SSCG_K5_RECUR": "0"},
            {"SSCG_K1_TMA": "0", "SSCG_K1_FUSE": "0"}, {"SSCG_PDL": "0"}],
    "7pt_mid": [{}, {"SSCG_K1_MP3": "1"}, {"SSCG_K1_MP3": "0", "SSCG_K1_FUSE": "1"}, {"SSCG_WFREE": "0"},
                {"SSCG_WL_FOLD": "0"}],
    "cfg2": [{}, {"SSCG_K1_MP3": "1"}, {"SSCG_K5_RECUR": "0"}, {"SSCG_WFREE": "0"}, {"SSCG_WL_FOLD": "0"}],
    "27pt": [{}, {"SSCG_K1_FUSE": "1"}, {"SSCG_WFREE": "0"}, {"SSCG_WFREE": "0", "SSCG_K2_DMMA": "1"},
             {"SSCG_K5_RECUR": "0"}],
    "varcoef7": [{}, {"SSCG_K1_FUSE_VC": "1"}, {"SSCG_K1_FUSE_VC": "0"}, {"SSCG_K2S": "0"}, {"SSCG_WFREE": "0"},
                 {"SSCG_K5_RECUR": "0"}, {"SSCG_FACES_TMA": "0"}],
    # cfg 1 runs the single-CTA outer iteration (KS) by default; SSCG_SMALL=0 the multi-kernel path
    "cfg1": [{}, {"SSCG_SMALL": "0"}, {"SSCG_SMALL": "0", "SSCG_K5_RECUR": "0"}],
    # odd nx: padded row pitch, so the stored-W schedule and the stored-W update always
    "7pt_odd": [{}, {"SSCG_K1_FUSE": "1"}, {"SSCG_K1_TMA": "0", "SSCG_K1_FUSE": "0"}, {"SSCG_SMALL": "1"}],
}

_problems = {}
_states = {}


def _problem(name):
    if name not in _problems:
        kind, nx, ny, nz, s, nu = SHAPES[name]
        _problems[name] = Problem(kind, nx, ny, nz, s, nu, lanczos=(kind == "27pt"))
    return _problems[name]


_depth_cache = {}


def _depths(P):
    """{10, 50, a few before convergence} (clipped to the solve's length)."""
    if id(P) not in _depth_cache:
        _, tr = P.oracle(max_outer=5000, rtol=1e-8)
        K = tr.outer
        _depth_cache[id(P)] = sorted({min(10, K - 1), min(50, K - 1), max(1, K - 3)})
    return _depth_cache[id(P)]


def _state(name, k):
    """(oracle r_k, oracle trace of one outer iteration from b := r_k, x_1)."""
    key = (name, k)
    if key not in _states:
        P = _problem(name)
        _, tr = P.oracle(max_outer=k, dump_iter=k)
        rk = tr.P[0].copy()
        x1, tr1 = orc.sstep_cg(P.A, P.lmin, P.lmax, P.s, P.nu, rk, rtol=0.0, max_outer=1, dump_iter=0)
        _states[key] = (rk, tr1, x1)
    return _states[key]


def _cases():
    out = []
    for name in SHAPES:
        for env in SWITCHES[name]:
            tag = ",".join(f"{k[5:]}={v}" for k, v in env.items()) or "default"
            out.append(pytest.param(name, env, id=f"{name}-{tag}"))
    return out


@pytest.mark.parametrize("name,env", _cases())
def test_identical_inputs_deep(name, env, monkeypatch):
    import torch
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    P = _problem(name)
    for k in _depths(P):
        rk, tr1, x1_or = _state(name, k)
        with P.gpu_solver() as S:
            b = torch.from_numpy(rk).cuda()
            S.solve(b, rtol=0.0, max_outer=0)          # basis + Gram of outer k (stop test only)
            assert_basis(S, tr1, P.s, tol=TOL_BASIS)
            assert_gram(S, tr1, 0, tol=TOL_GRAM)
            x1 = S.solve(b, rtol=0.0, max_outer=1).cpu().numpy()
            assert_gram(S, tr1, 0, tol=TOL_GRAM)
            assert_alpha(S, tr1, 0, tol=TOL_ALPHA)
            ex = np.linalg.norm(x1 - x1_or) / np.linalg.norm(x1_or)
            assert ex <= TOL_ALPHA, (k, ex)
            d = S.inspect(__import__("paper_2512_09642_b200").INSPECT_DELTA, 0)[0]
            assert abs(d - tr1.delta[0]) <= 1e-8 * tr1.delta[0] + 1e-15, (k, d, tr1.delta[0])


def test_depths_cover_late_solve():
    """The depths really reach deep into the solve (not only k = 0)."""
    P = _problem("7pt_mid")
    ds = _depths(P)
    assert max(ds) >= 50 and len(ds) == 3
