"""The inexact Gram solve in the restart form (FGS with
nu sweeps instead of the exact factorisation): outer iterations to rtol 1e-8,
device time per full solve and the true residual ||b - A x|| / ||b||, for
nu in {1, 2, 5, 10, 20, 30} and the exact (Cholesky) solve, 7-point Poisson on
one GPU.  usage: python tools/nu_sweep.py [n] [s]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import inputs  # noqa: E402
import paper_2512_09642_b200 as sscg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
s = int(sys.argv[2]) if len(sys.argv) > 2 else 16
b = torch.from_numpy(inputs.rhs_uniform(n, n, n, seed=42)).cuda()
lmin, lmax = inputs.analytic_bounds("7pt", n, n, n)


def true_relres(x):
    # ||b - A x|| / ||b|| for the 7-point operator (6 / -1, Dirichlet), in torch on the GPU
    v = x.view(n, n, n)
    ax = 6.0 * v
    ax[1:] -= v[:-1]
    ax[:-1] -= v[1:]
    ax[:, 1:] -= v[:, :-1]
    ax[:, :-1] -= v[:, 1:]
    ax[:, :, 1:] -= v[:, :, :-1]
    ax[:, :, :-1] -= v[:, :, 1:]
    return float(torch.linalg.norm(b - ax.reshape(-1)) / torch.linalg.norm(b))


out = {"n": n, "s": s, "rtol": 1e-8, "runs": {}}
for nu, gs in [(1, "fgs"), (2, "fgs"), (5, "fgs"), (10, "fgs"), (20, "fgs"), (30, "fgs"), (30, "cholesky")]:
    with sscg.Solver(sscg.Stencil("7pt", n, n, n), lmin, lmax, s, nu, gram_solver=gs) as S:
        S.solve(b, rtol=1e-8, max_outer=20000)   # warm-up (graph capture)
        x = S.solve(b, rtol=1e-8, max_outer=20000)
        st = S.stats()
        key = "cholesky" if gs == "cholesky" else "fgs_nu%d" % nu
        out["runs"][key] = {"outer": st.outer_iterations, "converged": bool(st.converged), "ms_total": st.ms_total,
                            "ms_per_outer": st.ms_total / max(st.outer_iterations, 1),
                            "true_relres": true_relres(x)}
        print(key, out["runs"][key], flush=True)
print(json.dumps(out))
