"""Pins for the oracle's Lanczos bounds and the seeded input
generators (inputs/, shared by both sides, no method arithmetic)."""
import numpy as np
import pytest

import inputs
import oracle as orc


def diag_csr(vals):
    n = len(vals)
    return orc.csr(np.arange(n + 1), np.arange(n), np.asarray(vals, float))


def test_spec_lanczos_examples(golden):
    g = golden["lanczos_diag123"]
    A = diag_csr(g["A_diag"])
    lo, hi, m = orc.lanczos_bounds(A, g["iters"], np.ones(3), 0.0, D=np.ones(3))
    assert (lo, hi) == pytest.approx(tuple(g["bounds_m0"]), abs=1e-12)
    lo, hi, _ = orc.lanczos_bounds(A, g["iters"], np.ones(3), 0.1, D=np.ones(3))
    assert (lo, hi) == pytest.approx(tuple(g["bounds_m01"]), abs=1e-12)
    lo, hi, m = orc.lanczos_bounds(diag_csr(np.ones(5)), 1, np.arange(1.0, 6.0), 0.0, D=np.ones(5))
    assert (lo, hi) == pytest.approx((1.0, 1.0), abs=1e-14)


def test_tridiag_eig_matches_eigvalsh():
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal(12), rng.standard_normal(11)
    T = np.diag(a) + np.diag(b, 1) + np.diag(b, -1)
    ev = np.linalg.eigvalsh(T)
    for k in (0, 5, 11):
        assert orc.tridiag_eig(a, b, k) == pytest.approx(ev[k], abs=1e-12)


def test_lanczos_full_depth_brackets_spectrum():
    dims = (5, 5, 6)
    A = orc.stencil(orc.KIND_27PT, *dims)
    lo_ex, hi_ex = inputs.analytic_bounds("27pt", *dims)
    lo, hi, m = orc.lanczos_bounds(A, 150, inputs.rhs_uniform(*dims, seed=4), 0.0)
    assert abs(lo - lo_ex) <= 1e-8 * hi_ex and abs(hi - hi_ex) <= 1e-8 * hi_ex


def test_analytic_bounds_against_dense_eigs():
    for kind, K, dims in (("5pt", orc.KIND_5PT2D, (7, 6, 1)), ("7pt", orc.KIND_7PT, (5, 4, 6)),
                          ("27pt", orc.KIND_27PT, (4, 5, 6))):
        A = orc.stencil(K, *dims)
        M = np.array([orc.apply(A, e) for e in np.eye(A.n)]).T
        ev = np.linalg.eigvalsh(M) / M[0, 0]
        lo, hi = inputs.analytic_bounds(kind, *dims)
        assert lo == pytest.approx(ev[0], rel=1e-12) and hi == pytest.approx(ev[-1], rel=1e-12)


def test_splitmix64_reference(golden):
    outs = [int(h) for h in inputs._mix(np.array([0x9E3779B97F4A7C15 * k % 2**64 for k in (1, 2, 3)],
                                                   dtype=np.uint64))]
    assert [f"{o:016x}" for o in outs] == golden["splitmix64_seed0"]["outputs_hex"]


def test_rhs_partition_invariant_and_range():
    nx, ny, nz = 6, 5, 8
    full = inputs.rhs_uniform(nx, ny, nz, seed=42)
    parts = [inputs.rhs_uniform(nx, ny, nz, seed=42, z0=z0, nzl=2) for z0 in range(0, 8, 2)]
    assert np.array_equal(np.concatenate(parts), full)
    assert full.min() >= -1 and full.max() < 1
    pts = inputs.rhs_at(nx, ny, [0, 5, 3], [0, 4, 2], [0, 7, 1], seed=42)
    assert np.array_equal(pts, full.reshape(nz, ny, nx)[[0, 7, 1], [0, 4, 2], [0, 5, 3]])
    big = inputs.rhs_uniform(64, 64, 16, seed=1)
    assert abs(big.mean()) < 0.01 and abs(big.var() - 1 / 3) < 0.01
    assert not np.array_equal(big, inputs.rhs_uniform(64, 64, 16, seed=2))


def test_lognormal_faces_moments():
    kx, ky, kz = inputs.lognormal_faces(40, 40, 40, seed=42)
    assert kx.shape == (40, 40, 41) and ky.shape == (40, 41, 40) and kz.shape == (41, 40, 40)
    z = np.log(np.concatenate([kx.ravel(), ky.ravel(), kz.ravel()]))
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01
