"""Pins for the oracle's AMG coarse-grid routines (§6,
347-354 §8; R25): the Galerkin operator A_c = P^T A_f P of the
piecewise-constant aggregation, restriction / prolongation, and Forward
Gauss-Seidel on A_c.

Each check is fixed by mathematics independent of the oracle's code: the
surface-area / face-sum closed forms of P^T A P for a finite-volume operator
(p^T A p = sum over faces k_f (p_a - p_b)^2, Dirichlet faces with p_b = 0),
P = I, the adjoint identity, Gauss-Seidel on a 2 x 2 system written out, the
limit of many sweeps (a dense direct solve), and the textbook asymptotic rate
rho_GS = rho_J^2 of lexicographic Gauss-Seidel on the model Laplacian.
"""
import itertools
import math

import numpy as np
import pytest

import inputs
import oracle as orc

pytestmark = pytest.mark.filterwarnings("ignore")


def boxes(n, b):
    """aggregate index ranges along one axis"""
    return [(s, min(s + b, n)) for s in range(0, n, b)]


def closed_form_ac(kind, dims, b, faces=None):
    """A_c from the face sums: entry (I, J) = -sum of the coefficients of the
    fine faces between aggregates I and J, entry (I, I) = sum over every face
    of aggregate I's surface (shared or Dirichlet).  Constant stencils have
    unit face coefficients (5-/7-point Laplacian)."""
    nx, ny, nz = dims
    bx, by, bz = b
    X, Y, Z = boxes(nx, bx), boxes(ny, by), boxes(nz, bz)
    ncx, ncy, ncz = len(X), len(Y), len(Z)
    nc = ncx * ncy * ncz
    M = np.zeros((nc, nc))
    if faces is None:
        kx = np.ones((nz, ny, nx + 1)); ky = np.ones((nz, ny + 1, nx)); kz = np.ones((nz + 1, ny, nx))
    else:
        kx = faces[0].reshape(nz, ny, nx + 1); ky = faces[1].reshape(nz, ny + 1, nx)
        kz = faces[2].reshape(nz + 1, ny, nx)
    agg = lambda x, y, z: x // bx + ncx * (y // by + ncy * (z // bz))   # noqa: E731
    # every fine face: between cells a, b (or a and the Dirichlet boundary)
    for z, y, f in itertools.product(range(nz), range(ny), range(nx + 1)):
        lo = agg(f - 1, y, z) if f > 0 else None
        hi = agg(f, y, z) if f < nx else None
        add_face(M, lo, hi, kx[z, y, f])
    for z, f, x in itertools.product(range(nz), range(ny + 1), range(nx)):
        lo = agg(x, f - 1, z) if f > 0 else None
        hi = agg(x, f, z) if f < ny else None
        add_face(M, lo, hi, ky[z, f, x])
    if kind != orc.KIND_5PT2D:   # the 2D operator has no z faces
        for f, y, x in itertools.product(range(nz + 1), range(ny), range(nx)):
            lo = agg(x, y, f - 1) if f > 0 else None
            hi = agg(x, y, f) if f < nz else None
            add_face(M, lo, hi, kz[f, y, x])
    return M


def add_face(M, a, b, k):
    # energy k (p_a - p_b)^2 of one face, with p = indicator of an aggregate
    if a is not None and b is not None and a == b:
        return   # face inside one aggregate: p_a - p_b = 0 for every indicator
    if a is not None:
        M[a, a] += k
    if b is not None:
        M[b, b] += k
    if a is not None and b is not None:
        M[a, b] -= k
        M[b, a] -= k


CASES = [(orc.KIND_7PT, (8, 6, 4), (2, 2, 2)), (orc.KIND_7PT, (9, 7, 5), (2, 2, 2)),
         (orc.KIND_7PT, (7, 5, 6), (3, 2, 4)), (orc.KIND_7PT, (5, 4, 3), (1, 1, 1)),
         (orc.KIND_5PT2D, (11, 9, 1), (2, 2, 1)), (orc.KIND_5PT2D, (10, 7, 1), (3, 4, 1))]


@pytest.mark.parametrize("kind,dims,b", CASES)
def test_galerkin_constant_stencil_surface_areas(kind, dims, b):
    """Constant 5/7-point Laplacian: A_c(I, I) = surface area of the aggregate
    box (2(sx sy + sy sz + sz sx) cells' faces), A_c(I, J) = -(shared face
    area); exactly, as integers."""
    A = orc.stencil(kind, *dims)
    Ac = orc.coarse_galerkin(A, b)
    ref = closed_form_ac(kind, dims, b)
    assert Ac.n == ref.shape[0] == int(np.prod(orc.coarse_dims(A, b)))
    assert np.array_equal(Ac.dense(), ref)


def test_galerkin_even_grid_is_scaled_coarse_laplacian():
    """2x2x2 aggregates of the 7-point Laplacian on an even grid: A_c = 4 x
    the 7-point Laplacian of the coarse grid (centre 24, neighbours -4)."""
    A = orc.stencil(orc.KIND_7PT, 8, 6, 4)
    Ac = orc.coarse_galerkin(A).dense()
    L = orc.stencil(orc.KIND_7PT, 4, 3, 2)
    n = L.n
    Ld = np.zeros((n, n))
    for i in range(n):
        e = np.zeros(n); e[i] = 1.0
        Ld[:, i] = orc.apply(L, e)
    assert np.array_equal(Ac, 4.0 * Ld)


@pytest.mark.parametrize("dims,b", [((7, 6, 5), (2, 2, 2)), ((6, 9, 4), (3, 2, 2)), ((5, 5, 7), (2, 3, 1))])
def test_galerkin_varcoef_face_sums(dims, b):
    """Variable-coefficient FV operator: the same face-sum closed form with the
    lognormal face coefficients (to rounding: the oracle sums in its own order)."""
    faces = inputs.lognormal_faces(*dims, seed=7)
    A = orc.stencil(orc.KIND_VARCOEF7, *dims, *faces)
    Ac = orc.coarse_galerkin(A, b).dense()
    ref = closed_form_ac(orc.KIND_VARCOEF7, dims, b, faces)
    assert np.allclose(Ac, ref, rtol=1e-14, atol=1e-14 * np.abs(ref).max())
    assert np.array_equal(Ac != 0.0, ref != 0.0)       # the same sparsity
    assert np.array_equal(Ac, Ac.T)                     # symmetric bitwise (R25)
    assert np.all(np.linalg.eigvalsh(Ac) > 0.0)         # SPD


def test_galerkin_identity_aggregation():
    """b = (1, 1, 1): P = I, A_c = A_f (each column one operator application)."""
    faces = inputs.lognormal_faces(4, 3, 3, seed=3)
    A = orc.stencil(orc.KIND_VARCOEF7, 4, 3, 3, *faces)
    Ac = orc.coarse_galerkin(A, (1, 1, 1)).dense()
    n = A.n
    for i in range(n):
        e = np.zeros(n); e[i] = 1.0
        assert np.array_equal(Ac[:, i], orc.apply(A, e))


def test_restrict_prolong():
    """P 1_c = 1_f, P^T 1_f = aggregate sizes, <P^T r, y> = <r, P y>."""
    A = orc.stencil(orc.KIND_7PT, 9, 7, 5)
    b = (2, 3, 2)
    nc = int(np.prod(orc.coarse_dims(A, b)))
    assert np.array_equal(orc.coarse_prolong_add(A, np.ones(nc), np.zeros(A.n), b), np.ones(A.n))
    sizes = np.array([(x1 - x0) * (y1 - y0) * (z1 - z0)
                      for (z0, z1) in boxes(5, 2) for (y0, y1) in boxes(7, 3) for (x0, x1) in boxes(9, 2)], float)
    assert np.array_equal(orc.coarse_restrict(A, np.ones(A.n), b), sizes)
    rng = np.random.default_rng(1)
    r, y = rng.standard_normal(A.n), rng.standard_normal(nc)
    lhs = np.dot(orc.coarse_restrict(A, r, b), y)
    rhs = np.dot(r, orc.coarse_prolong_add(A, y, np.zeros(A.n), b))
    assert abs(lhs - rhs) <= 1e-13 * np.abs(r).sum() * np.abs(y).max()


def test_fgs_two_by_two_written_out():
    """One and two sweeps on a 2 x 2 system, Gauss-Seidel written out."""
    a11, a12, a22 = 4.0, -1.5, 3.0
    M = orc.CoarseMatrix(2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([a11, a12, a12, a22]))
    r = np.array([1.0, 2.0])
    y0 = np.array([0.25, -0.5])
    x1 = (r[0] - a12 * y0[1]) / a11
    x2 = (r[1] - a12 * x1) / a22
    assert np.array_equal(orc.coarse_fgs(M, r, 1, y0), [x1, x2])
    x1b = (r[0] - a12 * x2) / a11
    x2b = (r[1] - a12 * x1b) / a22
    assert np.array_equal(orc.coarse_fgs(M, r, 2, y0), [x1b, x2b])
    assert np.array_equal(orc.coarse_fgs(M, r, 0, y0), y0)


@pytest.mark.parametrize("kind,dims,b", [(orc.KIND_7PT, (10, 8, 6), (2, 2, 2)),
                                         (orc.KIND_VARCOEF7, (9, 7, 6), (2, 2, 2)),
                                         (orc.KIND_5PT2D, (13, 11, 1), (2, 2, 1))])
def test_fgs_converges_to_direct_solve(kind, dims, b):
    """Many sweeps reach the dense direct solution of A_c y = r_c."""
    faces = inputs.lognormal_faces(*dims, seed=5) if kind == orc.KIND_VARCOEF7 else (None, None, None)
    A = orc.stencil(kind, *dims, *faces)
    Ac = orc.coarse_galerkin(A, b)
    rc = orc.coarse_restrict(A, inputs.rhs_uniform(*dims, seed=11), b)
    y_star = np.linalg.solve(Ac.dense(), rc)
    y = orc.coarse_fgs(Ac, rc, 600)
    assert np.linalg.norm(y - y_star) <= 1e-12 * np.linalg.norm(y_star)


def test_fgs_asymptotic_rate_model_problem():
    """Lexicographic Gauss-Seidel on the (scaled) 7-point Laplacian of an
    mx x my x mz grid contracts the error asymptotically by rho_J^2 per sweep,
    rho_J = (cos(pi/(mx+1)) + cos(pi/(my+1)) + cos(pi/(mz+1))) / 3 (the
    consistently ordered case of Young's theory).  A_c of 2x2x2 aggregates of
    an even grid is 4 x that Laplacian (pinned above), so the rate is the same."""
    dims = (12, 10, 8)
    A = orc.stencil(orc.KIND_7PT, *dims)
    Ac = orc.coarse_galerkin(A)
    mx, my, mz = orc.coarse_dims(A)
    rho = ((math.cos(math.pi / (mx + 1)) + math.cos(math.pi / (my + 1)) + math.cos(math.pi / (mz + 1))) / 3) ** 2
    rc = np.zeros(Ac.n)   # y* = 0: the iterate is the error
    y = orc.coarse_fgs(Ac, rc, 1, inputs.rhs_uniform(mx, my, mz, seed=2))
    for _ in range(150):
        y = orc.coarse_fgs(Ac, rc, 1, y)
    e0 = np.linalg.norm(y)
    y = orc.coarse_fgs(Ac, rc, 20, y)
    ratio = (np.linalg.norm(y) / e0) ** (1 / 20)
    assert abs(ratio - rho) <= 2e-3 * rho, (ratio, rho)
