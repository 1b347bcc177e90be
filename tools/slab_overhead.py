"""Cost of the halo schedule on one GPU: cfg 5 (448^3, s = 16, nu = 30) split
into 1, 2, 4 in-process z-slabs (boundary planes first, device-to-device halo
copies overlapped with the interior, fixed-order block sum) -- a proxy for the
per-rank overhead of the multi-GPU schedule (the NCCL transfers themselves
are not in it).  usage: python tools/slab_overhead.py [n] [steps]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import inputs  # noqa: E402
import paper_2512_09642_b200 as sscg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 448
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
b = torch.from_numpy(inputs.rhs_uniform(n, n, n, seed=42)).cuda()
lmin, lmax = inputs.analytic_bounds("7pt", n, n, n)
res = {}
for slabs in (1, 2, 4):
    with sscg.Solver(sscg.Stencil("7pt", n, n, n), lmin, lmax, 16, 30, slabs_per_rank=slabs) as S:
        x = S.solve(b, rtol=0.0, max_outer=0)
        S.iterate(x, 3)
        S.iterate(x, steps)
        ms = S.stats().ms_total / steps
        res[slabs] = {"ms_per_outer": ms, "fused": S.query(sscg.QUERY_BASIS_FUSED)}
        del x
    torch.cuda.empty_cache()
for k, v in res.items():
    v["relative_to_1"] = res[1]["ms_per_outer"] / v["ms_per_outer"]
print(json.dumps({"n": n, "steps": steps, "slabs": res}))
