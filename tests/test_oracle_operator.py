"""Pins for the oracle's operators, preconditioner diagonal and dot product.

Each check is fixed by mathematics independent of the oracle's own code:
closed-form eigenpairs, Kronecker-sum assembly, the finite-volume energy
identity, exactly-summed reference sums.
"""
import math

import numpy as np
import pytest

import inputs
import oracle as orc

pytestmark = pytest.mark.filterwarnings("ignore")


def dense(A):
    n = A.n
    M = np.zeros((n, n))
    for i in range(n):
        e = np.zeros(n); e[i] = 1.0
        M[:, i] = orc.apply(A, e)
    return M


def tridiag(N):
    return 2 * np.eye(N) - np.eye(N, k=1) - np.eye(N, k=-1)


def test_27pt_2cube(golden):
    g = golden["poisson27_2cube"]
    A = orc.stencil(orc.KIND_27PT, 2, 2, 2)
    M = dense(A)
    assert np.allclose(np.diag(M), 26.0)
    assert all((M[i] == -1).sum() == 7 for i in range(8))
    assert np.allclose(np.sort(np.linalg.eigvalsh(M)), g["eigs"], atol=1e-12)
    assert np.allclose(orc.apply(A, np.ones(8)), g["A_ones"])


def test_27pt_interior_rows_sum_zero():
    # corrected SPEC.md:47: points with all 26 neighbours inside have row sum 0
    A = orc.stencil(orc.KIND_27PT, 4, 4, 4)
    y = orc.apply(A, np.ones(64)).reshape(4, 4, 4)
    assert np.all(y[1:3, 1:3, 1:3] == 0.0)
    assert np.all(y[0] > 0)


@pytest.mark.parametrize("kind,dims", [("5pt", (7, 5, 1)), ("7pt", (6, 5, 4)), ("27pt", (5, 6, 4))])
def test_sine_modes_are_eigenvectors(kind, dims):
    K = {"5pt": orc.KIND_5PT2D, "7pt": orc.KIND_7PT, "27pt": orc.KIND_27PT}[kind]
    A = orc.stencil(K, *dims)
    rng = np.random.default_rng(0)
    for _ in range(4):
        ks = [int(rng.integers(1, d + 1)) for d in dims]
        if kind == "5pt":
            ks[2] = 1
        v = inputs.sine_mode(*dims, *ks)
        lam = inputs.sine_mode_eig(kind, dims[:2] if kind == "5pt" else dims, ks[:2] if kind == "5pt" else ks)
        assert np.max(np.abs(orc.apply(A, v) - lam * v)) < 1e-13 * max(1, abs(lam))


def test_7pt_equals_kronecker_sum():
    nx, ny, nz = 5, 4, 3
    A = dense(orc.stencil(orc.KIND_7PT, nx, ny, nz))
    I = np.eye
    K = (np.kron(I(nz), np.kron(I(ny), tridiag(nx))) + np.kron(I(nz), np.kron(tridiag(ny), I(nx)))
         + np.kron(tridiag(nz), np.kron(I(ny), I(nx))))
    assert np.array_equal(A, K)


def test_5pt_equals_kronecker_sum():
    nx, ny = 6, 5
    A = dense(orc.stencil(orc.KIND_5PT2D, nx, ny, 1))
    K = np.kron(np.eye(ny), tridiag(nx)) + np.kron(tridiag(ny), np.eye(nx))
    assert np.array_equal(A, K)


def test_27pt_equals_27I_minus_box():
    nx, ny, nz = 4, 3, 5
    A = dense(orc.stencil(orc.KIND_27PT, nx, ny, nz))
    B1 = lambda N: np.eye(N) + np.eye(N, k=1) + np.eye(N, k=-1)
    box = np.kron(B1(nz), np.kron(B1(ny), B1(nx)))
    assert np.array_equal(A, 27 * np.eye(nx * ny * nz) - box)


def test_varcoef_energy_identity_and_symmetry():
    nx, ny, nz = 5, 4, 3
    kx, ky, kz = inputs.lognormal_faces(nx, ny, nz, seed=7)
    A = orc.stencil(orc.KIND_VARCOEF7, nx, ny, nz, kx, ky, kz)
    M = dense(A)
    assert np.allclose(M, M.T, rtol=0, atol=1e-14)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(nx * ny * nz)
    X = np.zeros((nz + 2, ny + 2, nx + 2))
    X[1:-1, 1:-1, 1:-1] = x.reshape(nz, ny, nx)
    # x^T A x = sum_faces k_f (x_a - x_b)^2 with x = 0 outside (FV energy)
    E = (kx * (X[1:-1, 1:-1, 1:] - X[1:-1, 1:-1, :-1]) ** 2).sum()
    E += (ky * (X[1:-1, 1:, 1:-1] - X[1:-1, :-1, 1:-1]) ** 2).sum()
    E += (kz * (X[1:, 1:-1, 1:-1] - X[:-1, 1:-1, 1:-1]) ** 2).sum()
    assert abs(x @ orc.apply(A, x) - E) < 1e-12 * E
    # unit coefficients reduce to the 7-point Laplacian
    one = [np.ones_like(k) for k in (kx, ky, kz)]
    A1 = orc.stencil(orc.KIND_VARCOEF7, nx, ny, nz, *one)
    assert np.array_equal(dense(A1), dense(orc.stencil(orc.KIND_7PT, nx, ny, nz)))
    assert np.allclose(orc.diag(A), np.diag(M), rtol=0, atol=0)


def test_csr_matches_stencil_and_dense():
    for kind, K, dims in (("5pt", orc.KIND_5PT2D, (6, 4, 1)), ("7pt", orc.KIND_7PT, (4, 3, 5))):
        rp, ci, va = inputs.stencil_csr(kind, *dims)
        Acsr = orc.csr(rp, ci, va)
        D = np.zeros((Acsr.n, Acsr.n))
        for i in range(Acsr.n):
            D[i, ci[rp[i]:rp[i + 1]]] = va[rp[i]:rp[i + 1]]
        x = np.random.default_rng(2).standard_normal(Acsr.n)
        assert np.allclose(orc.apply(Acsr, x), D @ x, rtol=0, atol=1e-13)
        assert np.allclose(orc.apply(orc.stencil(K, *dims), x), D @ x, rtol=0, atol=1e-13)
        assert np.array_equal(orc.diag(Acsr), np.diag(D))


def test_diag_constant_stencils():
    assert np.all(orc.diag(orc.stencil(orc.KIND_5PT2D, 3, 3, 1)) == 4)
    assert np.all(orc.diag(orc.stencil(orc.KIND_7PT, 3, 3, 3)) == 6)
    assert np.all(orc.diag(orc.stencil(orc.KIND_27PT, 3, 3, 3)) == 26)


@pytest.mark.parametrize("n", [1, 7, 1000, (1 << 16) + 123, 3 * (1 << 16) - 1])
def test_dot_accuracy(n):
    rng = np.random.default_rng(n)
    x, y = rng.standard_normal(n), rng.standard_normal(n)
    exact = math.fsum((x * y).tolist())
    scale = np.abs(x * y).sum()
    assert abs(orc.dot(x, y) - exact) <= 1e-14 * scale + 1e-300
