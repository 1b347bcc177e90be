"""Shared helpers for the GPU parity tests: build the same seeded problem for
the CUDA path (through the C ABI) and for the CPU oracle, and compare them
with the north_star tolerances."""
from __future__ import annotations

import numpy as np

import inputs
import oracle as orc

KIND_ORC = {"5pt": orc.KIND_5PT2D, "7pt": orc.KIND_7PT, "27pt": orc.KIND_27PT, "varcoef7": orc.KIND_VARCOEF7}

# north_star tolerances (BASELINE.json) -- DESIGN.md R15
TOL_BASIS = 1e-12     # ||dp_j||inf / ||p_j||inf and same for w_j
TOL_GRAM = 1e-11      # max|dGhat| / max|Ghat|
TOL_ALPHA = 1e-10     # ||d alpha||inf / ||alpha||inf
TOL_X10 = 1e-8        # ||dx||_2 / ||x||_2 after 10 outer iterations
# k >= 1 without a restart: each side iterates on its own r_k; rounding
# differences propagate through the (ill-conditioned) Gram solves (R15)
TOL_GRAM_DRIFT = 1e-9
TOL_ALPHA_DRIFT = 1e-8
TOL_BASIS_DRIFT = 1e-9


class Problem:
    """A seeded model problem: operator, rhs, bounds (all from inputs/ or the
    oracle -- never from the CUDA path)."""

    def __init__(self, kind, nx, ny, nz, s, nu, seed=42, bounds=None, lanczos=False):
        self.kind, self.nx, self.ny, self.nz, self.s, self.nu, self.seed = kind, nx, ny, nz, s, nu, seed
        self.faces = inputs.lognormal_faces(nx, ny, nz, seed=seed) if kind == "varcoef7" else None
        if kind == "varcoef7":
            self.A = orc.stencil(orc.KIND_VARCOEF7, nx, ny, nz, *self.faces)
        else:
            self.A = orc.stencil(KIND_ORC[kind], nx, ny, nz)
        self.b = inputs.rhs_uniform(nx, ny, nz, seed=seed)
        if bounds is not None:
            self.lmin, self.lmax = bounds
        elif lanczos or kind == "varcoef7":
            lo, hi, _ = orc.lanczos_bounds(self.A, 50, self.b, 0.05)
            self.lmin, self.lmax = lo, hi
        else:
            self.lmin, self.lmax = inputs.analytic_bounds(kind, nx, ny, nz)

    def gpu_solver(self, slabs=1, **kw):
        import torch

        import paper_2512_09642_b200 as sscg
        dev = torch.device("cuda")
        self._keep = []
        if self.kind == "varcoef7":
            kx, ky, kz = (torch.from_numpy(np.ascontiguousarray(f)).to(dev) for f in self.faces)
            self._keep = [kx, ky, kz]
            op = sscg.Stencil("varcoef7", self.nx, self.ny, self.nz, kx, ky, kz)
        else:
            op = sscg.Stencil(self.kind, self.nx, self.ny, self.nz)
        return sscg.Solver(op, self.lmin, self.lmax, self.s, self.nu, slabs_per_rank=slabs, **kw)

    def b_gpu(self):
        import torch
        return torch.from_numpy(self.b).cuda()

    def oracle(self, max_outer, rtol=0.0, dump_iter=-1):
        return orc.sstep_cg(self.A, self.lmin, self.lmax, self.s, self.nu, self.b, rtol=rtol,
                            max_outer=max_outer, dump_iter=dump_iter)

    def oracle_ex(self, max_outer, rtol=0.0, dump_iter=-1, gram_solver="fgs", basis="chebyshev"):
        return orc.sstep_cg(self.A, self.lmin, self.lmax, self.s, self.nu, self.b, rtol=rtol,
                            max_outer=max_outer, dump_iter=dump_iter, gram_solver=gram_solver, basis=basis)


def rel_inf(a, ref):
    return float(np.max(np.abs(a - ref)) / max(np.max(np.abs(ref)), 1e-300))


def assert_basis(S, tr, s, tol=TOL_BASIS):
    for j in range(s):
        p, w = S.basis(j)
        ep, ew = rel_inf(p, tr.P[j]), rel_inf(w, tr.W[j])
        assert ep <= tol, f"p_{j}: {ep:.3e}"
        assert ew <= tol, f"w_{j}: {ew:.3e}"


def assert_gram(S, tr, k, tol=TOL_GRAM):
    G, c = S.gram(k)
    scale = np.max(np.abs(tr.ghat[k]))
    eg = np.max(np.abs(G - tr.ghat[k])) / scale
    ec = np.max(np.abs(c - tr.c[k])) / max(np.max(np.abs(tr.c[k])), 1e-300)
    assert eg <= tol, f"Gram[{k}]: {eg:.3e}"
    assert ec <= tol, f"c[{k}]: {ec:.3e}"


def assert_alpha(S, tr, k, tol=TOL_ALPHA):
    import paper_2512_09642_b200 as sscg
    at = S.inspect(sscg.INSPECT_ALPHA_T, k)
    al = S.inspect(sscg.INSPECT_ALPHA, k)
    assert rel_inf(at, tr.alpha_t[k]) <= tol, f"alpha~[{k}]: {rel_inf(at, tr.alpha_t[k]):.3e}"
    assert rel_inf(al, tr.alpha[k]) <= tol, f"alpha[{k}]: {rel_inf(al, tr.alpha[k]):.3e}"
