"""CPU FP64 oracle for Chebyshev s-step PCG with nu-sweep FGS Gram solves
(Thomas & D'Ambra, arxiv 2512.09642).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` leg may import this
package.  It shares no code with the CUDA product path
(``paper_2512_09642_b200``), and never imports it.

The arithmetic lives in ``sscg_oracle.c`` (plain C, ``-ffp-contract=off``);
this module only marshals numpy arrays through ctypes.  Every C routine cites
the PAPER.md passage it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sscg_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

KIND_5PT2D, KIND_7PT, KIND_27PT, KIND_VARCOEF7, KIND_CSR = 0, 1, 2, 3, 4


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, FP64, no FMA contraction, OpenMP rows)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Op(C.Structure):
    _fields_ = [("kind", C.c_int), ("nx", C.c_long), ("ny", C.c_long), ("nz", C.c_long),
                ("kx", C.c_void_p), ("ky", C.c_void_p), ("kz", C.c_void_p),
                ("n", C.c_long), ("rowptr", C.c_void_p), ("colind", C.c_void_p), ("val", C.c_void_p)]


class _Trace(C.Structure):
    _fields_ = [("outer", C.c_int), ("converged", C.c_int), ("breakdown", C.c_int),
                ("r0norm", C.c_double),
                ("relres", C.c_void_p), ("ghat", C.c_void_p), ("c", C.c_void_p), ("d", C.c_void_p),
                ("alpha_t", C.c_void_p), ("alpha", C.c_void_p), ("delta", C.c_void_p),
                ("energy", C.c_void_p), ("dump_iter", C.c_int), ("P_dump", C.c_void_p),
                ("W_dump", C.c_void_p), ("gconj", C.c_void_p), ("cconj", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        vp, d, i, l = C.c_void_p, C.c_double, C.c_int, C.c_long
        L.orc_n.argtypes = [vp]; L.orc_n.restype = l
        L.orc_apply.argtypes = [vp, vp, vp]
        L.orc_diag.argtypes = [vp, vp]
        L.orc_dot.argtypes = [l, vp, vp]; L.orc_dot.restype = d
        L.orc_chebyshev_basis.argtypes = [vp, vp, d, d, i, vp, vp, vp]
        L.orc_monomial_basis.argtypes = [vp, vp, i, vp, vp, vp]
        L.orc_gram.argtypes = [l, i, vp, vp, vp, vp]
        L.orc_scale.argtypes = [i, vp, vp, vp, vp, vp]; L.orc_scale.restype = i
        L.orc_fgs.argtypes = [i, vp, vp, i, vp, vp]
        L.orc_cholesky_solve.argtypes = [i, vp, vp, vp]; L.orc_cholesky_solve.restype = i
        L.orc_mgs_anorm.argtypes = [vp, i, vp, vp, vp, vp]
        L.orc_sstep_cg.argtypes = [vp, vp, d, d, i, i, vp, vp, d, i, vp]; L.orc_sstep_cg.restype = i
        L.orc_sstep_cg_ex.argtypes = [vp, vp, d, d, i, i, vp, vp, d, i, vp, i]; L.orc_sstep_cg_ex.restype = i
        L.orc_pcg.argtypes = [vp, vp, vp, vp, d, i]; L.orc_pcg.restype = i
        L.orc_tridiag_eig.argtypes = [i, vp, vp, i]; L.orc_tridiag_eig.restype = d
        L.orc_lanczos_bounds.argtypes = [vp, vp, i, vp, d, vp, vp]; L.orc_lanczos_bounds.restype = i
        L.orc_lanczos_bounds_tri.argtypes = [vp, vp, i, vp, d, vp, vp, vp, vp]
        L.orc_lanczos_bounds_tri.restype = i
        L.orc_coarse_n.argtypes = [vp, i, i, i]; L.orc_coarse_n.restype = l
        L.orc_coarse_restrict.argtypes = [vp, i, i, i, vp, vp]
        L.orc_coarse_prolong_add.argtypes = [vp, i, i, i, vp, vp]
        L.orc_coarse_galerkin.argtypes = [vp, i, i, i, vp, vp, vp, l]; L.orc_coarse_galerkin.restype = l
        L.orc_coarse_fgs.argtypes = [l, vp, vp, vp, vp, i, vp]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class Operator:
    """Operator description.  Grid functions are flat arrays indexed
    g = x + nx*(y + ny*z).  ``keep`` pins the numpy buffers the C struct
    points into."""
    kind: int
    nx: int = 0
    ny: int = 1
    nz: int = 1
    kx: np.ndarray | None = None
    ky: np.ndarray | None = None
    kz: np.ndarray | None = None
    rowptr: np.ndarray | None = None
    colind: np.ndarray | None = None
    val: np.ndarray | None = None

    def __post_init__(self):
        if self.kind == KIND_VARCOEF7:
            self.kx, self.ky, self.kz = _f64(self.kx), _f64(self.ky), _f64(self.kz)
            assert self.kx.size == self.nz * self.ny * (self.nx + 1)
            assert self.ky.size == self.nz * (self.ny + 1) * self.nx
            assert self.kz.size == (self.nz + 1) * self.ny * self.nx
        if self.kind == KIND_CSR:
            self.rowptr = np.ascontiguousarray(self.rowptr, dtype=np.int64)
            self.colind = np.ascontiguousarray(self.colind, dtype=np.int32)
            self.val = _f64(self.val)
        n = (len(self.rowptr) - 1) if self.kind == KIND_CSR else 0
        self._s = _Op(self.kind, self.nx, self.ny, self.nz, _p(self.kx), _p(self.ky), _p(self.kz),
                      n, _p(self.rowptr), _p(self.colind), _p(self.val))

    @property
    def n(self) -> int:
        return lib().orc_n(C.byref(self._s))

    @property
    def ref(self):
        return C.byref(self._s)


def stencil(kind: int, nx: int, ny: int = 1, nz: int = 1, kx=None, ky=None, kz=None) -> Operator:
    return Operator(kind, nx, ny, nz, kx, ky, kz)


def csr(rowptr, colind, val) -> Operator:
    return Operator(KIND_CSR, rowptr=rowptr, colind=colind, val=val)


def apply(A: Operator, x) -> np.ndarray:
    x = _f64(x)
    y = np.empty(A.n)
    lib().orc_apply(A.ref, _p(x), _p(y))
    return y


def diag(A: Operator) -> np.ndarray:
    d = np.empty(A.n)
    lib().orc_diag(A.ref, _p(d))
    return d


def dot(x, y) -> float:
    x, y = _f64(x), _f64(y)
    return lib().orc_dot(x.size, _p(x), _p(y))


def chebyshev_basis(A: Operator, D, lmin, lmax, s, r):
    """Returns (P, W) as (s, n) arrays: P[j] = p_j, W[j] = A p_j."""
    D, r = _f64(D), _f64(r)
    P = np.empty((s, A.n)); W = np.empty((s, A.n))
    lib().orc_chebyshev_basis(A.ref, _p(D), lmin, lmax, s, _p(r), _p(P), _p(W))
    return P, W


def monomial_basis(A: Operator, D, s, r):
    D, r = _f64(D), _f64(r)
    P = np.empty((s, A.n)); W = np.empty((s, A.n))
    lib().orc_monomial_basis(A.ref, _p(D), s, _p(r), _p(P), _p(W))
    return P, W


def gram(P, W):
    """Ghat = P^T W (s x s), c = P^T p_0, with P, W given as (s, n) arrays."""
    P, W = _f64(P), _f64(W)
    s, n = P.shape
    G = np.empty((s, s)); c = np.empty(s)
    lib().orc_gram(n, s, _p(P), _p(W), _p(G), _p(c))
    return G, c


def scale(Ghat, c):
    """Ruhe scaling -> (d, G, c~); raises on breakdown."""
    Ghat, c = _f64(Ghat), _f64(c)
    s = c.size
    d = np.empty(s); G = np.empty((s, s)); ct = np.empty(s)
    rc = lib().orc_scale(s, _p(Ghat), _p(c), _p(d), _p(G), _p(ct))
    if rc:
        raise FloatingPointError(f"Gram breakdown at column {rc - 1}")
    return d, G, ct


def fgs(G, rhs, nu, hist=False):
    G, rhs = _f64(G), _f64(rhs)
    s = rhs.size
    a = np.empty(s)
    h = np.empty(nu + 1) if hist else None
    lib().orc_fgs(s, _p(G), _p(rhs), nu, _p(a), _p(h))
    return (a, h) if hist else a


def cholesky_solve(G, rhs):
    G, rhs = _f64(G), _f64(rhs)
    x = np.empty(rhs.size)
    rc = lib().orc_cholesky_solve(rhs.size, _p(G), _p(rhs), _p(x))
    if rc:
        raise np.linalg.LinAlgError(f"non-positive pivot {rc - 1}")
    return x


def mgs_anorm(A: Operator, Pt, v):
    """Pt: (s, n) scaled basis rows.  Returns (gamma, w_s)."""
    Pt, v = _f64(Pt), _f64(v)
    s = Pt.shape[0]
    g = np.empty(s); w = np.empty(A.n)
    lib().orc_mgs_anorm(A.ref, s, _p(Pt), _p(v), _p(g), _p(w))
    return g, w


@dataclass
class Trace:
    outer: int
    converged: bool
    breakdown: bool
    r0norm: float
    relres: np.ndarray
    ghat: np.ndarray
    c: np.ndarray
    d: np.ndarray
    alpha_t: np.ndarray
    alpha: np.ndarray
    delta: np.ndarray
    energy: np.ndarray
    P: np.ndarray | None = None
    W: np.ndarray | None = None
    gconj: np.ndarray | None = None   # block-conjugate mode: G_k = Q_k^T A Q_k
    cconj: np.ndarray | None = None   # and c_k = Q_k^T r_k


OPT_CHOLESKY, OPT_MONOMIAL, OPT_BLOCKCG = 1, 2, 4


def sstep_cg(A: Operator, lmin, lmax, s, nu, b, x0=None, rtol=1e-8, max_outer=1000, D=None,
             dump_iter=-1, gram_solver="fgs", basis="chebyshev", block=False) -> tuple[np.ndarray, Trace]:
    """Run the oracle s-step CG; returns (x, Trace).  Trace arrays are indexed
    by outer iteration k (only the first ``outer`` (+1 for ghat/c/relres)
    entries are meaningful).  gram_solver 'fgs' (nu sweeps) or
    'cholesky' (exact); basis 'chebyshev' or
    'monomial'; block=True: block-conjugate s-step CG
    (sscg_oracle.c ORC_OPT_BLOCKCG, R24) instead of the restart form
    (the basis dump holds the raw basis P_k, W_k before the conjugation)."""
    opts = (OPT_CHOLESKY if gram_solver == "cholesky" else 0) | (OPT_MONOMIAL if basis == "monomial" else 0)
    opts |= OPT_BLOCKCG if block else 0
    assert gram_solver in ("fgs", "cholesky") and basis in ("chebyshev", "monomial")
    b = _f64(b)
    n = A.n
    x = np.zeros(n) if x0 is None else _f64(x0).copy()
    K = max_outer + 1
    relres = np.zeros(K); ghat = np.zeros((K, s, s)); c = np.zeros((K, s)); d = np.zeros((K, s))
    at = np.zeros((K, s)); al = np.zeros((K, s)); de = np.zeros(K); en = np.zeros(K)
    Pd = np.zeros((s, n)) if dump_iter >= 0 else None
    Wd = np.zeros((s, n)) if dump_iter >= 0 else None
    gq = np.zeros((K, s, s)) if block else None
    cq = np.zeros((K, s)) if block else None
    tr = _Trace(0, 0, 0, 0.0, _p(relres), _p(ghat), _p(c), _p(d), _p(at), _p(al), _p(de), _p(en),
                dump_iter, _p(Pd), _p(Wd), _p(gq), _p(cq))
    Dm = None if D is None else _f64(D)
    lib().orc_sstep_cg_ex(A.ref, _p(Dm), lmin, lmax, s, nu, _p(b), _p(x), rtol, max_outer, C.byref(tr), opts)
    return x, Trace(tr.outer, bool(tr.converged), bool(tr.breakdown), tr.r0norm, relres, ghat, c, d,
                    at, al, de, en, Pd, Wd, gq, cq)


def pcg(A: Operator, b, rtol=1e-8, max_iter=100000, D=None):
    b = _f64(b)
    x = np.zeros(A.n)
    Dm = None if D is None else _f64(D)
    it = lib().orc_pcg(A.ref, _p(Dm), _p(b), _p(x), rtol, max_iter)
    return x, it


def tridiag_eig(a, b, k):
    a, b = _f64(a), _f64(b)
    return lib().orc_tridiag_eig(a.size, _p(a), _p(b), k)


def lanczos_bounds(A: Operator, iters, v0, margin, D=None, tridiag=False):
    """(lmin, lmax, m) -- with tridiag=True also the Lanczos coefficients
    (alpha[:m], beta[:m-1])."""
    v0 = _f64(v0)
    lo, hi = C.c_double(), C.c_double()
    Dm = None if D is None else _f64(D)
    al, be = np.zeros(iters), np.zeros(iters)
    m = lib().orc_lanczos_bounds_tri(A.ref, _p(Dm), iters, _p(v0), margin, C.byref(lo), C.byref(hi), _p(al), _p(be))
    if tridiag:
        return lo.value, hi.value, m, al[:m], be[:max(m - 1, 0)]
    return lo.value, hi.value, m


# --------------------------------------------------------------------------
# AMG coarse grid (R25): aggregates of
# b = (bx, by, bz) fine cells, A_c = P^T A_f P, Forward Gauss-Seidel on A_c
# --------------------------------------------------------------------------

def coarse_dims(A: Operator, b=(2, 2, 2)):
    bx, by, bz = b
    return (-(-A.nx // bx), -(-A.ny // by), -(-A.nz // bz))


def coarse_restrict(A: Operator, rf, b=(2, 2, 2)) -> np.ndarray:
    """r_c = P^T r_f."""
    rf = _f64(rf)
    rc = np.empty(int(np.prod(coarse_dims(A, b))))
    lib().orc_coarse_restrict(A.ref, *b, _p(rf), _p(rc))
    return rc


def coarse_prolong_add(A: Operator, y, xf, b=(2, 2, 2)) -> np.ndarray:
    """Returns x_f + P y (xf is not modified)."""
    y = _f64(y)
    out = _f64(xf).copy()
    lib().orc_coarse_prolong_add(A.ref, *b, _p(y), _p(out))
    return out


@dataclass
class CoarseMatrix:
    n: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    def dense(self) -> np.ndarray:
        M = np.zeros((self.n, self.n))
        for i in range(self.n):
            for q in range(self.rowptr[i], self.rowptr[i + 1]):
                M[i, self.col[q]] = self.val[q]
        return M


def coarse_galerkin(A: Operator, b=(2, 2, 2)) -> CoarseMatrix:
    """A_c = P^T A_f P, column by column (sscg_oracle.c orc_coarse_galerkin)."""
    nc = lib().orc_coarse_n(A.ref, *b)
    cap = 27 * nc + 64
    rowptr = np.zeros(nc + 1, dtype=np.int64)
    col = np.zeros(cap, dtype=np.int64)
    val = np.zeros(cap)
    nnz = lib().orc_coarse_galerkin(A.ref, *b, _p(rowptr), _p(col), _p(val), cap)
    assert nnz >= 0
    return CoarseMatrix(nc, rowptr, col[:nnz].copy(), val[:nnz].copy())


def coarse_fgs(Ac: CoarseMatrix, rc, nu, y0=None) -> np.ndarray:
    """nu Forward Gauss-Seidel sweeps on A_c y = r_c from y0 (default 0)."""
    rc = _f64(rc)
    y = np.zeros(Ac.n) if y0 is None else _f64(y0).copy()
    lib().orc_coarse_fgs(Ac.n, _p(Ac.rowptr), _p(Ac.col), _p(Ac.val), _p(rc), nu, _p(y))
    return y
