"""B200-native Chebyshev-basis s-step PCG with nu-sweep Forward Gauss-Seidel
Gram solves (Thomas & D'Ambra, arxiv 2512.09642).

Thin Python binding of ``libsscg.so`` (C ABI in ``include/sscg.h``): this
module only marshals arguments (torch tensors / numpy arrays -> pointers);
every step of the solve runs in the library's sm_100a kernels.  There is no
CPU fallback: if the library cannot be loaded, every call raises.

    import paper_2512_09642_b200 as sscg
    op = sscg.Stencil("7pt", nx, ny, nz)
    with sscg.Solver(op, lmin, lmax, s=16, nu=25) as S:
        x = S.solve(b, rtol=1e-8, max_outer=1000)      # b: cuda float64 tensor
        print(S.stats())
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SSCG_LIB selects another in-tree build of the same library (variant builds
# from `python -m paper_2512_09642_b200.build --variant NAME -D...`, for sweeps)
LIB_PATH = os.environ.get("SSCG_LIB") or os.path.join(_HERE, "libsscg.so")

OK, ERR_INVALID, ERR_CUDA, ERR_NCCL, ERR_OOM, ERR_BREAKDOWN, ERR_NONFINITE, ERR_UNSUPPORTED = range(8)
OP_STENCIL5_2D, OP_STENCIL7, OP_STENCIL27, OP_VARCOEF7, OP_CSR = range(5)
(INSPECT_P, INSPECT_W, INSPECT_GRAM, INSPECT_D, INSPECT_ALPHA_T, INSPECT_ALPHA, INSPECT_DELTA, INSPECT_LNORM,
 INSPECT_KAPPA, INSPECT_PNORM, INSPECT_BUDGET) = range(11)
SOLVE_X0_ZERO = 1
OPT_GRAM_SOLVER, OPT_BASIS, OPT_DIAGNOSTICS, OPT_BLOCKCG = 0, 1, 2, 3
GRAM_FGS, GRAM_CHOLESKY = 0, 1
BASIS_CHEBYSHEV, BASIS_MONOMIAL = 0, 1
(QUERY_BASIS_FUSED, QUERY_BASIS_VECTORS, QUERY_UPDATE_VECTORS, QUERY_GRAM_VECTORS, QUERY_BASIS_SINGLE_VECTORS,
 QUERY_PEER_HALO) = 0, 1, 2, 3, 4, 5

EXPORTS = ["sscg_partition", "sscg_halo_plan", "sscg_nccl_unique_id", "sscg_setup", "sscg_solve", "sscg_solve_host", "sscg_iterate",
           "sscg_set_profiling", "sscg_profile", "sscg_stats", "sscg_inspect", "sscg_local_shape", "sscg_destroy",
           "sscg_last_error", "sscg_version", "sscg_set_bounds", "sscg_set_option", "sscg_estimate_bounds", "sscg_query",
           "sscg_coarse_create", "sscg_coarse_restrict", "sscg_coarse_prolong_add", "sscg_coarse_fgs",
           "sscg_coarse_entries", "sscg_coarse_query", "sscg_coarse_destroy"]
COARSE_STREAMING, COARSE_ASSEMBLED = 0, 1
(COARSE_QUERY_N, COARSE_QUERY_NCX, COARSE_QUERY_NCY, COARSE_QUERY_NCZ, COARSE_QUERY_WAVEFRONTS,
 COARSE_QUERY_MATRIX_BYTES) = range(6)
PROF_NAMES = ["basis", "gram", "allreduce", "fgs", "update", "halo", "basis_single"]


class SSCGError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"sscg error {code}: {msg}")
        self.code = code


class _Operator(C.Structure):
    _fields_ = [("kind", C.c_int32), ("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("kx", C.c_void_p), ("ky", C.c_void_p), ("kz", C.c_void_p), ("n", C.c_int64),
                ("rowptr", C.c_void_p), ("colind", C.c_void_p), ("val", C.c_void_p)]


class _Comm(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("slabs_per_rank", C.c_int32),
                ("nccl_id", C.c_void_p)]


class _Stats(C.Structure):
    _fields_ = [("outer_iterations", C.c_int32), ("converged", C.c_int32), ("breakdown", C.c_int32),
                ("nonfinite", C.c_int32), ("r0_norm", C.c_double), ("relres_final", C.c_double),
                ("history_len", C.c_int32), ("relres_history", C.POINTER(C.c_double)),
                ("delta_history", C.POINTER(C.c_double)), ("ms_total", C.c_double),
                ("kernel_launches", C.c_int64), ("allreduces", C.c_int64), ("budget", C.c_double)]


class _Profile(C.Structure):
    _fields_ = [("ms", C.c_double * 7), ("launches", C.c_int64 * 7)]


_lib = None


def load(path: str = LIB_PATH):
    """Load libsscg.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run `python -m paper_2512_09642_b200.build`")
    L = C.CDLL(path)
    vp, i32, i64, d, u32 = C.c_void_p, C.c_int32, C.c_int64, C.c_double, C.c_uint32
    L.sscg_partition.argtypes = [i64, i32, i32, i32, C.POINTER(i64), C.POINTER(i64)]
    L.sscg_halo_plan.argtypes = [i64, i32, i32, i32, i32, C.POINTER(i64)]
    L.sscg_halo_plan.restype = C.c_int
    L.sscg_nccl_unique_id.argtypes = [vp]
    L.sscg_setup.argtypes = [C.POINTER(_Operator), vp, d, d, i32, i32, C.POINTER(_Comm), vp, C.POINTER(vp)]
    L.sscg_solve.argtypes = [vp, vp, vp, d, i32, u32]
    L.sscg_solve_host.argtypes = [vp, vp, vp, d, i32, u32]
    L.sscg_iterate.argtypes = [vp, vp, i32]
    L.sscg_set_profiling.argtypes = [vp, i32]
    L.sscg_profile.argtypes = [vp, C.POINTER(_Profile)]
    L.sscg_stats.argtypes = [vp, C.POINTER(_Stats)]
    L.sscg_inspect.argtypes = [vp, i32, i32, vp, i64]
    L.sscg_local_shape.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]
    L.sscg_set_bounds.argtypes = [vp, d, d]
    L.sscg_set_option.argtypes = [vp, i32, i32]
    L.sscg_estimate_bounds.argtypes = [vp, vp, i32, d, C.POINTER(d), C.POINTER(d), vp, vp]
    L.sscg_query.argtypes = [vp, i32, C.POINTER(i64)]
    L.sscg_destroy.argtypes = [vp]
    L.sscg_destroy.restype = None
    L.sscg_coarse_create.argtypes = [C.POINTER(_Operator), i32, i32, i32, i32, C.POINTER(vp)]
    L.sscg_coarse_restrict.argtypes = [vp, vp, vp, vp]
    L.sscg_coarse_prolong_add.argtypes = [vp, vp, vp, vp]
    L.sscg_coarse_fgs.argtypes = [vp, vp, vp, i32, vp]
    L.sscg_coarse_entries.argtypes = [vp, vp, vp]
    L.sscg_coarse_query.argtypes = [vp, i32, C.POINTER(i64)]
    L.sscg_coarse_destroy.argtypes = [vp]
    L.sscg_coarse_destroy.restype = None
    L.sscg_last_error.restype = C.c_char_p
    L.sscg_version.restype = C.c_char_p
    for name in ("sscg_partition", "sscg_nccl_unique_id", "sscg_setup", "sscg_solve", "sscg_solve_host",
                 "sscg_iterate", "sscg_set_profiling", "sscg_profile", "sscg_stats", "sscg_inspect",
                 "sscg_local_shape", "sscg_set_bounds", "sscg_set_option", "sscg_estimate_bounds", "sscg_query",
                 "sscg_coarse_create", "sscg_coarse_restrict", "sscg_coarse_prolong_add", "sscg_coarse_fgs",
                 "sscg_coarse_entries", "sscg_coarse_query"):
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


def _check(code):
    if code != OK:
        raise SSCGError(code, load().sscg_last_error().decode())


def partition(nz: int, nranks: int, slabs_per_rank: int, rank: int) -> tuple[int, int]:
    """Planes (z0, nzl) of process `rank` (sscg_partition; host only)."""
    z0, nzl = C.c_int64(), C.c_int64()
    _check(load().sscg_partition(nz, nranks, slabs_per_rank, rank, C.byref(z0), C.byref(nzl)))
    return z0.value, nzl.value


def halo_plan(nz: int, nranks: int, slabs_per_rank: int, rank: int, slab: int = 0) -> dict:
    """sscg_halo_plan: neighbour processes and global plane indices of one
    local slab's halo exchange (host only)."""
    out = (C.c_int64 * 6)()
    _check(load().sscg_halo_plan(nz, nranks, slabs_per_rank, rank, slab, out))
    return {"peer_lo": out[0], "send_lo_z": out[1], "recv_lo_z": out[2],
            "peer_hi": out[3], "send_hi_z": out[4], "recv_hi_z": out[5]}


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(load().sscg_nccl_unique_id(buf))
    return buf.raw


def _check_dev(name, t, n):
    """A process-local float64 CUDA vector of n elements (ValueError otherwise:
    the library writes n doubles through the raw pointer)."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
            and t.numel() == n):
        raise ValueError(f"{name}: need a contiguous float64 CUDA tensor of {n} elements")


def _check_host(name, a, n):
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous and a.size == n):
        raise ValueError(f"{name}: need a C-contiguous float64 numpy array of {n} elements")


def _ptr(t):
    """Device/host pointer of a torch tensor or numpy array (no copies)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


@dataclass
class Stencil:
    """Constant/variable-coefficient stencil on the GLOBAL nx*ny*nz grid.
    kind: '5pt' (2D), '7pt', '27pt', 'varcoef7' (faces kx, ky, kz: device
    float64 tensors covering this process's planes, see include/sscg.h)."""
    kind: str
    nx: int
    ny: int
    nz: int = 1
    kx: object = None
    ky: object = None
    kz: object = None

    def _struct(self):
        k = {"5pt": OP_STENCIL5_2D, "7pt": OP_STENCIL7, "27pt": OP_STENCIL27, "varcoef7": OP_VARCOEF7}[self.kind]
        return _Operator(k, self.nx, self.ny, self.nz, _ptr(self.kx), _ptr(self.ky), _ptr(self.kz), 0, None, None, None)


@dataclass
class CSR:
    """General symmetric CSR (device tensors: int64 rowptr, int32 colind,
    float64 val), single process."""
    rowptr: object
    colind: object
    val: object

    def _struct(self):
        n = int(self.rowptr.shape[0]) - 1
        return _Operator(OP_CSR, 0, 0, 0, None, None, None, n, _ptr(self.rowptr), _ptr(self.colind), _ptr(self.val))


@dataclass
class Stats:
    outer_iterations: int
    converged: bool
    breakdown: bool
    nonfinite: bool
    r0_norm: float
    relres_final: float
    relres_history: np.ndarray
    delta_history: np.ndarray
    ms_total: float
    kernel_launches: int
    allreduces: int
    budget: float


class Solver:
    """One sscg context (sscg_setup ... sscg_destroy)."""

    def __init__(self, op, lmin: float, lmax: float, s: int, nu: int, diag_M=None, rank: int = 0,
                 nranks: int = 1, slabs_per_rank: int = 1, nccl_id: bytes | None = None, stream=None,
                 gram_solver: str = "fgs", basis: str = "chebyshev", block: bool = False):
        """lmin = lmax = 0 creates the context without spectral bounds (set
        them with set_bounds, e.g. from estimate_bounds)."""
        L = load()
        self._op = op
        self._opst = op._struct()
        self.s, self.nu = s, nu
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        comm = _Comm(rank, nranks, slabs_per_rank, C.cast(idbuf, C.c_void_p) if idbuf is not None else None)
        h = C.c_void_p()
        strm = None if stream is None else (stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
        _check(L.sscg_setup(C.byref(self._opst), _ptr(diag_M), lmin, lmax, s, nu, C.byref(comm), strm,
                            C.byref(h)))
        self._h = h
        z0, nzp, nloc = C.c_int64(), C.c_int64(), C.c_int64()
        _check(L.sscg_local_shape(h, C.byref(z0), C.byref(nzp), C.byref(nloc)))
        self.z0, self.nz_local, self.n_local = z0.value, nzp.value, nloc.value
        if gram_solver != "fgs":
            self.set_option(OPT_GRAM_SOLVER, {"fgs": GRAM_FGS, "cholesky": GRAM_CHOLESKY}[gram_solver])
        if basis != "chebyshev":
            self.set_option(OPT_BASIS, {"chebyshev": BASIS_CHEBYSHEV, "monomial": BASIS_MONOMIAL}[basis])
        if block:
            self.set_option(OPT_BLOCKCG, 1)

    def query(self, what: int) -> int:
        v = C.c_int64()
        _check(load().sscg_query(self._h, what, C.byref(v)))
        return v.value

    def set_bounds(self, lmin: float, lmax: float):
        _check(load().sscg_set_bounds(self._h, lmin, lmax))

    def set_option(self, key: int, value: int):
        _check(load().sscg_set_option(self._h, key, value))

    def estimate_bounds(self, v0, iters: int = 50, margin: float = 0.05, tridiag: bool = False):
        """Lanczos bounds of M^{-1}A from v0 (cuda float64, process-local);
        returns (lmin, lmax) or, with tridiag=True, (lmin, lmax, alpha, beta)."""
        import torch
        _check_dev("v0", v0, self.n_local)
        cur = torch.cuda.current_stream()
        if cur.cuda_stream != 0:
            cur.synchronize()
        lo, hi = C.c_double(), C.c_double()
        al, be = np.zeros(iters), np.zeros(iters)
        _check(load().sscg_estimate_bounds(self._h, _ptr(v0), iters, margin, C.byref(lo), C.byref(hi),
                                           al.ctypes.data, be.ctypes.data))
        return (lo.value, hi.value, al, be) if tridiag else (lo.value, hi.value)

    def close(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.sscg_destroy(h)
        self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def solve(self, b, x=None, rtol: float = 1e-8, max_outer: int = 1000, raise_on_breakdown: bool = True):
        """b, x: float64 CUDA tensors (process-local).  x=None => x_0 = 0 and a
        new tensor is returned; otherwise x is updated in place."""
        import torch
        _check_dev("b", b, self.n_local)
        flags = 0
        if x is None:
            x = torch.empty_like(b)
            flags = SOLVE_X0_ZERO
        _check_dev("x", x, self.n_local)
        if x.device != b.device:
            raise ValueError("b and x must be on the same device")
        cur = torch.cuda.current_stream()
        if cur.cuda_stream != 0:      # the library stream orders only after the legacy default stream
            cur.synchronize()
        code = load().sscg_solve(self._h, _ptr(b), _ptr(x), rtol, max_outer, flags)
        if code in (ERR_BREAKDOWN, ERR_NONFINITE) and not raise_on_breakdown:
            return x
        _check(code)
        return x

    def solve_host(self, b: np.ndarray, x: np.ndarray | None = None, rtol: float = 1e-8, max_outer: int = 1000):
        """End-to-end call with host buffers (copies are inside the call)."""
        _check_host("b", b, self.n_local)
        flags = 0
        if x is None:
            x = np.empty_like(b)
            flags = SOLVE_X0_ZERO
        _check_host("x", x, self.n_local)
        _check(load().sscg_solve_host(self._h, _ptr(b), _ptr(x), rtol, max_outer, flags))
        return x

    def iterate(self, x, nsteps: int):
        """Exactly nsteps more outer iterations from the last solve's state."""
        _check_dev("x", x, self.n_local)
        _check(load().sscg_iterate(self._h, _ptr(x), nsteps))
        return x

    def set_profiling(self, on: bool = True):
        _check(load().sscg_set_profiling(self._h, 1 if on else 0))

    def profile(self) -> dict:
        """{category: (ms, launches)} accumulated since set_profiling."""
        p = _Profile()
        _check(load().sscg_profile(self._h, C.byref(p)))
        return {n: (p.ms[i], int(p.launches[i])) for i, n in enumerate(PROF_NAMES)}

    def stats(self) -> Stats:
        st = _Stats()
        _check(load().sscg_stats(self._h, C.byref(st)))
        rh = (np.ctypeslib.as_array(st.relres_history, (st.history_len,)).copy()
              if st.history_len and bool(st.relres_history) else np.zeros(0))
        nd = max(st.history_len - 1, 0)
        dh = np.ctypeslib.as_array(st.delta_history, (nd,)).copy() if nd and bool(st.delta_history) else np.zeros(0)
        return Stats(st.outer_iterations, bool(st.converged), bool(st.breakdown), bool(st.nonfinite), st.r0_norm,
                     st.relres_final, rh, dh, st.ms_total, st.kernel_launches, st.allreduces, st.budget)

    def inspect(self, what: int, index: int) -> np.ndarray:
        n = {INSPECT_P: self.n_local, INSPECT_W: self.n_local, INSPECT_GRAM: self.s * self.s + self.s,
             INSPECT_D: self.s, INSPECT_ALPHA_T: self.s, INSPECT_ALPHA: self.s, INSPECT_DELTA: 1,
             INSPECT_LNORM: 1, INSPECT_KAPPA: 1, INSPECT_PNORM: 1, INSPECT_BUDGET: 1}[what]
        out = np.empty(n, dtype=np.float64)
        _check(load().sscg_inspect(self._h, what, index, out.ctypes.data, out.nbytes))
        return out

    def basis(self, j: int):
        return self.inspect(INSPECT_P, j), self.inspect(INSPECT_W, j)

    def gram(self, k: int):
        g = self.inspect(INSPECT_GRAM, k)
        s = self.s
        return g[: s * s].reshape(s, s), g[s * s:]


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class CoarseFGS:
    """AMG coarse-grid Forward Gauss-Seidel (sscg_coarse_*; PAPER.md:225-246,
    347-354; R25): one coarse level of b = (bx, by, bz) aggregates of
    the fine operator ``op`` (Stencil '5pt', '7pt' or 'varcoef7'), A_c = P^T A_f P
    never stored (mode 'streaming') or formed once ('assembled').  Vectors are
    float64 CUDA tensors; calls run on torch's current stream."""

    def __init__(self, op: Stencil, b=(2, 2, 2), mode: str = "streaming"):
        L = load()
        self.op = op   # keeps the face tensors alive
        m = {"streaming": COARSE_STREAMING, "assembled": COARSE_ASSEMBLED}[mode]
        h = C.c_void_p()
        _check(L.sscg_coarse_create(C.byref(op._struct()), b[0], b[1], b[2], m, C.byref(h)))
        self._h = h
        self.b = tuple(b)
        self.n_fine = op.nx * op.ny * op.nz
        self.n = self.query(COARSE_QUERY_N)
        self.dims = (self.query(COARSE_QUERY_NCX), self.query(COARSE_QUERY_NCY), self.query(COARSE_QUERY_NCZ))

    def query(self, what: int) -> int:
        v = C.c_int64()
        _check(load().sscg_coarse_query(self._h, what, C.byref(v)))
        return v.value

    def restrict(self, rf, rc=None):
        """r_c = P^T r_f"""
        import torch
        _check_dev("rf", rf, self.n_fine)
        rc = torch.empty(self.n, dtype=torch.float64, device=rf.device) if rc is None else rc
        _check_dev("rc", rc, self.n)
        _check(load().sscg_coarse_restrict(self._h, _ptr(rf), _ptr(rc), _stream()))
        return rc

    def prolong_add(self, y, xf):
        """x_f += P y (in place)"""
        _check_dev("y", y, self.n)
        _check_dev("xf", xf, self.n_fine)
        _check(load().sscg_coarse_prolong_add(self._h, _ptr(y), _ptr(xf), _stream()))
        return xf

    def fgs(self, rc, nu: int, y=None):
        """nu forward Gauss-Seidel sweeps on A_c y = r_c from y (zero if None);
        y is updated in place and returned"""
        import torch
        _check_dev("rc", rc, self.n)
        y = torch.zeros(self.n, dtype=torch.float64, device=rc.device) if y is None else y
        _check_dev("y", y, self.n)
        _check(load().sscg_coarse_fgs(self._h, _ptr(rc), _ptr(y), int(nu), _stream()))
        return y

    def entries(self):
        """(7, n_c) row entries: neighbours z-1, y-1, x-1, itself, x+1, y+1, z+1"""
        import torch
        out = torch.empty(7 * self.n, dtype=torch.float64, device="cuda")
        _check(load().sscg_coarse_entries(self._h, _ptr(out), _stream()))
        return out.view(7, self.n)

    def close(self):
        if getattr(self, "_h", None):
            load().sscg_coarse_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
