"""Per-rank cost of the multi-GPU halo schedule, measured on one GPU: cfg 5
(n^3 per slab, s = 16, nu = 30) as 1, 2, 4 in-process z-slabs of n planes
EACH (the weak-scaling per-rank size), stacked in z -- boundary planes first,
device-to-device halo copies overlapped with the interior, fixed-order block
sum.  One GPU runs the slabs one after the other, so the time per outer
iteration divided by the slab count is the per-rank time with the halo
schedule's extra launches and copies; relative_to_1 = t(1 slab) / that.  The
NCCL transfers themselves are not in it (the copies are device-to-device).

Schedules with several slabs: "deep" (the default: each K1M triple in one
launch storing the planes its neighbours need straight into their ghost
planes -- peer-store halos, no exchange after the triple), "deep_copies"
(SSCG_PEER_HALO=0: the triple, then one 3 + 2-plane exchange by copies), "deep_overlap" (SSCG_DEEP_OVERLAP=1:
the planes the exchange sends computed first, the exchange overlapped with
the rest of the triple), "plane1" (SSCG_DEEP_HALO=0: single steps on the
boundary planes around three 1-plane exchanges per triple).  usage: python tools/slab_overhead.py [n] [steps]"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import inputs  # noqa: E402
import paper_2512_09642_b200 as sscg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 448
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
MODES = {"deep": {"SSCG_DEEP_HALO": "1", "SSCG_DEEP_OVERLAP": "0", "SSCG_NO_OVERLAP": "0", "SSCG_PEER_HALO": "1"},
         "deep_copies": {"SSCG_DEEP_HALO": "1", "SSCG_DEEP_OVERLAP": "0", "SSCG_NO_OVERLAP": "0", "SSCG_PEER_HALO": "0"},
         "deep_overlap": {"SSCG_DEEP_HALO": "1", "SSCG_DEEP_OVERLAP": "1", "SSCG_NO_OVERLAP": "0"},
         "plane1": {"SSCG_DEEP_HALO": "0", "SSCG_DEEP_OVERLAP": "0", "SSCG_NO_OVERLAP": "0"}}
runs = [(1, "deep")] + [(sl, m) for sl in (2, 4) for m in MODES]
res = {}
for slabs, mode in runs:
    os.environ.update(MODES[mode])   # read at setup
    nz = n * slabs
    b = torch.from_numpy(inputs.rhs_uniform(n, n, nz, seed=42)).cuda()
    lmin, lmax = inputs.analytic_bounds("7pt", n, n, nz)
    with sscg.Solver(sscg.Stencil("7pt", n, n, nz), lmin, lmax, 16, 30, slabs_per_rank=slabs) as S:
        x = S.solve(b, rtol=0.0, max_outer=0)
        S.iterate(x, 3)
        S.iterate(x, steps)
        st = S.stats()
        key = "1" if slabs == 1 else "%d_%s" % (slabs, mode)
        res[key] = {"ms_per_outer_per_slab": st.ms_total / steps / slabs, "fused": S.query(sscg.QUERY_BASIS_FUSED),
                    "launches_per_outer": st.kernel_launches / steps}
        # the same steps with every launch group bracketed by events (eager launches):
        # where the extra time goes, per category and slab
        S.set_profiling(True)
        S.iterate(x, steps)
        prof = S.profile()
        S.set_profiling(False)
        res[key]["profiled_ms_per_outer_per_slab"] = {k: round(v[0] / steps / slabs, 4) for k, v in prof.items()}
        del x
    del b
    torch.cuda.empty_cache()
for k, v in res.items():
    v["relative_to_1"] = res["1"]["ms_per_outer_per_slab"] / v["ms_per_outer_per_slab"]
print(json.dumps({"n": n, "steps": steps, "per_slab_planes": n, "slabs": res}))
