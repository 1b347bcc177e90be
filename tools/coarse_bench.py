"""AMG coarse-grid FGS on one B200 (
DESIGN.md R25): the paper's coarsest-level size n_c ~ 5000 (34^3 fine cells,
2x2x2 aggregates -> 17^3 = 4913), nu_coarse = 20.

Per operator and mode (streaming: A_c never stored; assembled: 7 n_c
entries), the device time of one sscg_coarse_fgs call (CUDA events on the
launching stream, mean over `reps` calls after warm-up) and its pipelined
barrier steps T + 2(nu - 1).  Context (library code, not this framework's
kernels): the dense direct solve the paper compares against, here cuSOLVER
Cholesky through torch on the GPU (factorisation once, then one solve per
call) and the bytes each variant keeps for A_c.  Accuracy: the A_c-norm error
of nu sweeps against the direct solution (nu = 10-30).
usage: python tools/coarse_bench.py [n_fine] [reps]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import inputs  # noqa: E402
import paper_2512_09642_b200 as sscg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 34
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
nu = 20
dev = torch.device("cuda")


def timed(fn, reps):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {"n_fine": n, "b": [2, 2, 2], "nu": nu, "reps": reps, "runs": {}}
for kind in ("7pt", "varcoef7"):
    keep = []
    if kind == "varcoef7":
        keep = [torch.from_numpy(np.ascontiguousarray(f)).to(dev) for f in inputs.lognormal_faces(n, n, n, seed=17)]
        op = sscg.Stencil("varcoef7", n, n, n, *keep)
    else:
        op = sscg.Stencil("7pt", n, n, n)
    rf = torch.from_numpy(inputs.rhs_uniform(n, n, n, seed=9)).to(dev)
    res = {}
    for mode in ("streaming", "assembled"):
        with sscg.CoarseFGS(op, (2, 2, 2), mode) as G:
            rc = G.restrict(rf)
            y = torch.zeros(G.n, dtype=torch.float64, device=dev)
            ms = timed(lambda: G.fgs(rc, nu, y.zero_()), reps)
            T = G.query(sscg.COARSE_QUERY_WAVEFRONTS)
            steps = T + 2 * (nu - 1)
            res[mode] = {"n_c": G.n, "ms_per_fgs": ms, "steps": steps, "us_per_step": 1e3 * ms / steps,
                         "sequential_steps_unpipelined": nu * T,
                         "matrix_bytes": G.query(sscg.COARSE_QUERY_MATRIX_BYTES),
                         "ms_restrict": timed(lambda: G.restrict(rf, rc), reps),
                         "ms_prolong_add": timed(lambda: G.prolong_add(y, rf), reps)}
            if mode == "assembled":
                E = G.entries()
                ncx, ncy, ncz = G.dims
                nc = G.n
                idx = torch.arange(nc, device=dev)
                Ad = torch.zeros(nc, nc, dtype=torch.float64, device=dev)
                offs = [-ncx * ncy, -ncx, -1, 0, 1, ncx, ncx * ncy]
                for d, o in enumerate(offs):
                    m = E[d] != 0
                    Ad[idx[m], idx[m] + o] = E[d][m]
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                Lc = torch.linalg.cholesky(Ad)
                e1.record()
                torch.cuda.synchronize()
                y_star = torch.cholesky_solve(rc.view(-1, 1), Lc).view(-1)
                res["direct_dense_cholesky"] = {
                    "ms_factor": e0.elapsed_time(e1),
                    "ms_per_solve": timed(lambda: torch.cholesky_solve(rc.view(-1, 1), Lc), reps),
                    "matrix_bytes": nc * nc * 8, "library": "cuSOLVER via torch.linalg (context only)"}
                acc = {}
                en = lambda v: float(torch.sqrt(v @ (Ad @ v)))   # noqa: E731
                for k in (5, 10, 20, 30, 60):
                    yk = G.fgs(rc, k)
                    acc[str(k)] = en(yk - y_star) / en(y_star)
                res["anorm_error_vs_nu"] = acc
    out["runs"][kind] = res
print(json.dumps(out))
