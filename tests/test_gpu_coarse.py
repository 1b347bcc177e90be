"""GPU parity of the AMG coarse-grid FGS (PAPER.md:225-246
§6, 347-354 §8; R25) against the CPU oracle, through the C ABI
(sscg_coarse_*), on seeded inputs: the coarse operator's entries, restriction,
prolongation and nu forward Gauss-Seidel sweeps -- bitwise, in both the
streaming mode (A_c never stored: each row recomputed from the fine operator
at every visit) and the assembled mode.  The oracle forms A_c column by column
from its definition P^T A_f P and runs textbook Gauss-Seidel."""
import functools

import numpy as np
import pytest

import inputs
import oracle as orc
from gpu_cases import KIND_ORC

pytestmark = pytest.mark.gpu

# (kind, fine dims, aggregate b): ragged last aggregates, anisotropic b, P = I,
# and the paper's coarsest-level size n_c ~ 5000 (34^3 fine cells, 2x2x2 -> 17^3)
CASES = [("7pt", (21, 18, 13), (2, 2, 2)), ("7pt", (20, 16, 12), (3, 2, 4)), ("7pt", (12, 10, 8), (1, 1, 1)),
         ("varcoef7", (23, 19, 17), (2, 2, 2)), ("varcoef7", (16, 20, 9), (3, 3, 2)),
         ("5pt", (70, 50, 1), (2, 2, 1)), ("5pt", (33, 31, 1), (3, 2, 1)), ("varcoef7", (34, 34, 34), (2, 2, 2))]
IDS = ["%s-%dx%dx%d-b%d%d%d" % (k, *d, *b) for k, d, b in CASES]


@functools.lru_cache(maxsize=None)
def oracle_case(kind, dims, b):
    faces = inputs.lognormal_faces(*dims, seed=17) if kind == "varcoef7" else (None, None, None)
    A = orc.stencil(KIND_ORC[kind], *dims, *faces)
    Ac = orc.coarse_galerkin(A, b)
    return A, faces, Ac


def gpu_coarse(kind, dims, b, mode, faces):
    import torch

    import paper_2512_09642_b200 as sscg
    if kind == "varcoef7":
        f = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in faces]
        op = sscg.Stencil("varcoef7", *dims, *f)
    else:
        op = sscg.Stencil(kind, *dims)
    return sscg.CoarseFGS(op, b, mode)


def expected_entries(Ac, dims_c):
    """(7, n_c) from the oracle's CSR rows: neighbours z-1, y-1, x-1, itself, x+1, y+1, z+1"""
    ncx, ncy, ncz = dims_c
    E = np.zeros((7, Ac.n))
    for c in range(Ac.n):
        I, J, K = c % ncx, (c // ncx) % ncy, c // (ncx * ncy)
        nb = [c - ncx * ncy if K > 0 else -1, c - ncx if J > 0 else -1, c - 1 if I > 0 else -1, c,
              c + 1 if I + 1 < ncx else -1, c + ncx if J + 1 < ncy else -1, c + ncx * ncy if K + 1 < ncz else -1]
        row = dict(zip(Ac.col[Ac.rowptr[c]:Ac.rowptr[c + 1]].tolist(), Ac.val[Ac.rowptr[c]:Ac.rowptr[c + 1]].tolist()))
        for d, j in enumerate(nb):
            if j >= 0:
                E[d, c] = row.pop(j, 0.0)
        assert not row, "A_c couples a non-neighbour aggregate"
    return E


@pytest.mark.parametrize("mode", ["streaming", "assembled"])
@pytest.mark.parametrize("kind,dims,b", CASES, ids=IDS)
def test_coarse_parity_bitwise(kind, dims, b, mode):
    import torch
    A, faces, Ac = oracle_case(kind, dims, b)
    with gpu_coarse(kind, dims, b, mode, faces) as G:
        assert G.n == Ac.n and G.dims == orc.coarse_dims(A, b)
        assert G.query(5) == (0 if mode == "streaming" else 8 * Ac.n * 8)   # COARSE_QUERY_MATRIX_BYTES (7 entries + pad)
        # entries of A_c
        assert np.array_equal(G.entries().cpu().numpy(), expected_entries(Ac, G.dims))
        # restriction of a fine residual, prolongation of a coarse vector
        rf = inputs.rhs_uniform(*dims, seed=5)
        rc = orc.coarse_restrict(A, rf, b)
        rc_g = G.restrict(torch.from_numpy(rf).cuda())
        assert np.array_equal(rc_g.cpu().numpy(), rc)
        yv = inputs.rhs_uniform(*G.dims, seed=6)
        xf = inputs.rhs_uniform(*dims, seed=7)
        xg = torch.from_numpy(xf).cuda()
        G.prolong_add(torch.from_numpy(yv).cuda(), xg)
        assert np.array_equal(xg.cpu().numpy(), orc.coarse_prolong_add(A, yv, xf, b))
        # nu sweeps from zero and from a nonzero initial guess
        for nu in (1, 2, 7, 20):
            y = G.fgs(rc_g, nu).cpu().numpy()
            assert np.array_equal(y, orc.coarse_fgs(Ac, rc, nu)), nu
        y0 = inputs.rhs_uniform(*G.dims, seed=8)
        yg = torch.from_numpy(y0).cuda()
        G.fgs(rc_g, 20, yg)
        assert np.array_equal(yg.cpu().numpy(), orc.coarse_fgs(Ac, rc, 20, y0))
        yg0 = torch.from_numpy(y0).cuda()
        G.fgs(rc_g, 0, yg0)   # nu = 0 leaves y alone
        assert np.array_equal(yg0.cpu().numpy(), y0)


def test_coarse_many_sweeps_reach_direct_solve():
    """Enough sweeps on the paper-size coarse level (n_c = 4913) reach the
    dense direct solution (numpy): the GPU iteration is the oracle's, which
    converges (rho_FGS < 1).  This A_c is a coarse Laplacian
    of 17^3 points, rho_FGS ~ cos^2(pi/18) ~ 0.97 (pinned on the oracle for
    the model problem), so 2000 sweeps for 1e-9."""
    import torch
    kind, dims, b = "varcoef7", (34, 34, 34), (2, 2, 2)
    A, faces, Ac = oracle_case(kind, dims, b)
    rc = orc.coarse_restrict(A, inputs.rhs_uniform(*dims, seed=9), b)
    y_star = np.linalg.solve(Ac.dense(), rc)
    with gpu_coarse(kind, dims, b, "assembled", faces) as G:
        y = G.fgs(torch.from_numpy(rc).cuda(), 2000).cpu().numpy()
    assert np.linalg.norm(y - y_star) <= 1e-9 * np.linalg.norm(y_star)


def test_coarse_errors():
    import torch

    import paper_2512_09642_b200 as sscg
    with pytest.raises(sscg.SSCGError) as e:
        sscg.CoarseFGS(sscg.Stencil("27pt", 8, 8, 8))
    assert e.value.code == sscg.ERR_UNSUPPORTED
    with pytest.raises(sscg.SSCGError) as e:
        sscg.CoarseFGS(sscg.Stencil("7pt", 64, 64, 64))   # n_c = 32768 > SSCG_COARSE_MAX_N
    assert e.value.code == sscg.ERR_UNSUPPORTED
    with pytest.raises(sscg.SSCGError) as e:
        sscg.CoarseFGS(sscg.Stencil("5pt", 16, 16, 1), (2, 2, 2))
    assert e.value.code == sscg.ERR_INVALID
    with sscg.CoarseFGS(sscg.Stencil("7pt", 8, 8, 8)) as G:
        rc = torch.zeros(G.n, dtype=torch.float64, device="cuda")
        with pytest.raises(sscg.SSCGError) as e:
            G.fgs(rc, -1)
        assert e.value.code == sscg.ERR_INVALID
        with pytest.raises(ValueError):
            G.fgs(torch.zeros(G.n + 1, dtype=torch.float64, device="cuda"), 1)


def _random_coarse(n=36, seed=5):
    rng = np.random.default_rng(seed)
    out = []
    for it in range(n):
        kind = ["5pt", "7pt", "varcoef7"][it % 3]
        if kind == "5pt":
            dims = (int(rng.integers(2, 90)), int(rng.integers(2, 90)), 1)
            b = (int(rng.integers(1, 5)), int(rng.integers(1, 5)), 1)
        else:
            dims = tuple(int(v) for v in rng.integers(2, 30, 3))
            b = tuple(int(v) for v in rng.integers(1, 5, 3))
        out.append((kind, dims, b, int(rng.integers(1, 25))))
    return out


@pytest.mark.parametrize("case", _random_coarse(), ids=lambda c: "%s-%dx%dx%d-b%d%d%d-nu%d" % (c[0], *c[1], *c[2], c[3]))
def test_coarse_random_shapes_bitwise(case):
    """Seeded random fine grids, aggregate sizes (ragged last aggregates,
    anisotropic, P = I) and sweep counts: nu sweeps bitwise equal to the
    oracle in both modes (row-padded shared layout, closed-form / face-loaded
    streaming entries, prefetched assembled entries)."""
    import torch
    kind, dims, b, nu = case
    A, faces, Ac = oracle_case(kind, dims, b)
    rf = inputs.rhs_uniform(*dims, seed=3)
    rc = orc.coarse_restrict(A, rf, b)
    ref = orc.coarse_fgs(Ac, rc, nu)
    for mode in ("streaming", "assembled"):
        with gpu_coarse(kind, dims, b, mode, faces) as G:
            y = G.fgs(G.restrict(torch.from_numpy(rf).cuda()), nu).cpu().numpy()
        assert np.array_equal(y, ref), mode
