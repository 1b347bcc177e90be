"""Restart vs block-conjugate s-step CG (R24) on one GPU: outer
iterations to rtol 1e-8 and device time per full solve, FGS (nu sweeps) and
exact (Cholesky) Gram solves.  usage: python tools/blockcg_compare.py [n] [s] [nu]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import inputs  # noqa: E402
import paper_2512_09642_b200 as sscg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
s = int(sys.argv[2]) if len(sys.argv) > 2 else 16
nu = int(sys.argv[3]) if len(sys.argv) > 3 else 25
b = torch.from_numpy(inputs.rhs_uniform(n, n, n, seed=42)).cuda()
lmin, lmax = inputs.analytic_bounds("7pt", n, n, n)
out = {"n": n, "s": s, "nu": nu, "runs": {}}
for block in (False, True):
    for gs in ("fgs", "cholesky"):
        with sscg.Solver(sscg.Stencil("7pt", n, n, n), lmin, lmax, s, nu, gram_solver=gs, block=block) as S:
            S.solve(b, rtol=1e-8, max_outer=5000)   # warm-up (graph capture)
            S.solve(b, rtol=1e-8, max_outer=5000)
            st = S.stats()
            out["runs"][("block" if block else "restart") + "_" + gs] = {
                "outer": st.outer_iterations, "converged": st.converged, "ms_total": st.ms_total,
                "ms_per_outer": st.ms_total / max(st.outer_iterations, 1)}
print(json.dumps(out))
