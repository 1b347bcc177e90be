"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds none of the method's arithmetic: only the problem
description (right-hand sides, face coefficients, closed-form spectra of the
model problems) that both sides consume.  Recipe:

* b ~ U[-1, 1] from a counter-based SplitMix64 hash of the *global* linear
  grid index g = x + nx*(y + ny*z), so every z-slab partition sees the same
  values (R14).  u = (h >> 11) * 2^-53,  b = 2u - 1.
* variable coefficients: k = exp(N(0,1)) per face (lognormal mu=0, sigma=1),
  N(0,1) by Box-Muller from two hash streams; generated once on the host and
  the same bits go to both sides.
* analytic spectral bounds of M^{-1}A for the constant-coefficient Laplacians
  with Jacobi M (R13).
"""
from __future__ import annotations

import math

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def _key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        return _mix(np.array([(seed & (2**64 - 1)) ^ ((stream * 0xD1B54A32D192ED03) & (2**64 - 1))],
                             dtype=np.uint64))[0]


def hash_u64(g: np.ndarray, seed: int = 42, stream: int = 0) -> np.ndarray:
    """SplitMix64 output number g+1 of the generator keyed by (seed, stream)."""
    g = np.asarray(g, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix(_key(seed, stream) + (g + np.uint64(1)) * _GOLDEN)


def uniform01(g, seed=42, stream=0) -> np.ndarray:
    """u in [0, 1) with 53 random bits."""
    return (hash_u64(g, seed, stream) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def rhs_uniform(nx: int, ny: int, nz: int, seed: int = 42, z0: int = 0, nzl: int | None = None,
                chunk: int = 1 << 24) -> np.ndarray:
    """b ~ U[-1,1] on planes [z0, z0+nzl) of the global nx*ny*nz grid, flat
    x-fastest.  Values depend only on the global index (partition invariant)."""
    if nzl is None:
        nzl = nz - z0
    n = nx * ny * nzl
    base = nx * ny * z0
    out = np.empty(n, dtype=np.float64)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        g = np.arange(base + lo, base + hi, dtype=np.uint64)
        out[lo:hi] = 2.0 * uniform01(g, seed, 0) - 1.0
    return out


def rhs_at(nx: int, ny: int, xs, ys, zs, seed: int = 42) -> np.ndarray:
    """b at arbitrary global points (for sampled full-size parity)."""
    g = np.asarray(xs, np.uint64) + np.uint64(nx) * (np.asarray(ys, np.uint64)
                                                     + np.uint64(ny) * np.asarray(zs, np.uint64))
    return 2.0 * uniform01(g, seed, 0) - 1.0


def lognormal_faces(nx: int, ny: int, nz: int, seed: int = 42):
    """Face coefficients k = exp(N(0,1)) for the variable-coefficient 7-point
    operator (R12): kx (nz, ny, nx+1), ky (nz, ny+1, nx), kz (nz+1, ny, nx),
    each from its own pair of hash streams (1,2), (3,4), (5,6)."""
    def gen(shape, s1, s2):
        g = np.arange(int(np.prod(shape)), dtype=np.uint64)
        u1 = 1.0 - uniform01(g, seed, s1)            # (0, 1]
        u2 = uniform01(g, seed, s2)
        z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
        return np.exp(z).reshape(shape)
    return (gen((nz, ny, nx + 1), 1, 2), gen((nz, ny + 1, nx), 3, 4), gen((nz + 1, ny, nx), 5, 6))


def analytic_bounds(kind: str, nx: int, ny: int = 1, nz: int = 1):
    """Exact extreme eigenvalues of M^{-1}A, M = diag(A), for the constant-
    coefficient Dirichlet Laplacians on an nx*ny*nz interior grid (R13).
    kind: '5pt' (2D, nz ignored), '7pt', '27pt'."""
    if kind in ("5pt", "7pt"):
        dims = [nx, ny] if kind == "5pt" else [nx, ny, nz]
        cs = sum(math.cos(math.pi / (N + 1)) for N in dims)
        dim = len(dims)
        return 1.0 - cs / dim, 1.0 + cs / dim
    if kind == "27pt":
        c = [math.cos(math.pi / (N + 1)) for N in (nx, ny, nz)]
        # eigenvalues of A = 27 I - box: 27 - prod_d (1 + 2 cos(k_d pi/(N_d+1)))
        lam_min = (27.0 - (1 + 2 * c[0]) * (1 + 2 * c[1]) * (1 + 2 * c[2])) / 26.0
        # max: make the product as negative as possible: one factor at its most
        # negative value (1 - 2 c_d), the other two at their largest (1 + 2 c)
        prods = []
        for d in range(3):
            p = 1.0 - 2.0 * c[d]
            for e in range(3):
                if e != d:
                    p *= 1.0 + 2.0 * c[e]
            prods.append(p)
        return lam_min, (27.0 - min(prods)) / 26.0
    raise ValueError(kind)


def sine_mode(nx: int, ny: int, nz: int, kx: int, ky: int, kz: int) -> np.ndarray:
    """v(x,y,z) = prod_d sin(k_d pi (x_d+1)/(N_d+1)): an eigenvector of every
    constant-coefficient Dirichlet stencil above (flat, x fastest)."""
    sx = np.sin(kx * np.pi * np.arange(1, nx + 1) / (nx + 1))
    sy = np.sin(ky * np.pi * np.arange(1, ny + 1) / (ny + 1))
    sz = np.sin(kz * np.pi * np.arange(1, nz + 1) / (nz + 1))
    return (sz[:, None, None] * sy[None, :, None] * sx[None, None, :]).ravel()


def sine_mode_eig(kind: str, dims, ks) -> float:
    """Eigenvalue of A (not M^{-1}A) for sine mode ks on grid dims."""
    cs = [math.cos(k * math.pi / (N + 1)) for k, N in zip(ks, dims)]
    if kind == "5pt":
        return 4.0 - 2.0 * (cs[0] + cs[1])
    if kind == "7pt":
        return 6.0 - 2.0 * sum(cs)
    if kind == "27pt":
        p = 1.0
        for c in cs:
            p *= 1.0 + 2.0 * c
        return 27.0 - p
    raise ValueError(kind)


def poisson_csr_1d(n: int):
    """1D Dirichlet Laplacian tridiag(-1, 2, -1) as CSR (rowptr, colind, val)."""
    rows, cols, vals = [], [], []
    rowptr = [0]
    for i in range(n):
        for j, v in ((i - 1, -1.0), (i, 2.0), (i + 1, -1.0)):
            if 0 <= j < n:
                cols.append(j); vals.append(v)
        rowptr.append(len(cols))
    return np.array(rowptr, np.int64), np.array(cols, np.int32), np.array(vals, np.float64)


def stencil7_csr_fast(nx: int, ny: int, nz: int):
    """The 7-point graph Laplacian (6 / -1, Dirichlet) of an nx x ny x nz grid as
    CSR with ascending columns (z-1, y-1, x-1, itself, x+1, y+1, z+1), built
    vectorised for large grids (bench.py's CSR workload); the same matrix as
    stencil_csr("7pt", ...)."""
    n = nx * ny * nz
    g = np.arange(n, dtype=np.int64)
    x, y, z = g % nx, (g // nx) % ny, g // (nx * ny)
    offs = [(-nx * ny, z > 0), (-nx, y > 0), (-1, x > 0), (0, np.ones(n, bool)), (1, x < nx - 1),
            (nx, y < ny - 1), (nx * ny, z < nz - 1)]
    valid = np.stack([m for _, m in offs], axis=1)                    # [n, 7]
    cols = g[:, None] + np.array([o for o, _ in offs], np.int64)[None, :]
    vals = np.where(np.arange(7)[None, :] == 3, 6.0, -1.0) * np.ones((n, 1))
    rowptr = np.zeros(n + 1, np.int64)
    rowptr[1:] = np.cumsum(valid.sum(axis=1))
    return rowptr, cols[valid].astype(np.int32), vals[valid]


def stencil_csr(kind: str, nx: int, ny: int, nz: int = 1, faces=None):
    """Assemble a stencil operator as CSR (sorted columns) for CSR-path tests."""
    n = nx * ny * nz
    rowptr = np.zeros(n + 1, np.int64)
    cols, vals = [], []
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                ent = []
                if kind == "5pt":
                    ent.append((x + nx * y, 4.0))
                    for dx, dy in ((0, -1), (-1, 0), (1, 0), (0, 1)):
                        if 0 <= x + dx < nx and 0 <= y + dy < ny:
                            ent.append((x + dx + nx * (y + dy), -1.0))
                elif kind == "7pt":
                    ent.append((x + nx * (y + ny * z), 6.0))
                    for dx, dy, dz in ((0, 0, -1), (0, -1, 0), (-1, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)):
                        if 0 <= x + dx < nx and 0 <= y + dy < ny and 0 <= z + dz < nz:
                            ent.append((x + dx + nx * (y + dy + ny * (z + dz)), -1.0))
                else:
                    raise ValueError(kind)
                ent.sort()
                i = x + nx * (y + ny * z)
                for c, v in ent:
                    cols.append(c); vals.append(v)
                rowptr[i + 1] = len(cols)
    return rowptr, np.array(cols, np.int32), np.array(vals, np.float64)
