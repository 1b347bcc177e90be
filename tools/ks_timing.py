"""cfg 1 through the single-CTA-cluster outer iteration with a KS_TIMING build
(python -m paper_2512_09642_b200.build --variant kst -DKS_TIMING; run with
SSCG_LIB=.../libsscg_kst.so): per-phase device ns of a few outer iterations."""
import sys

import torch

sys.path.insert(0, ".")
import inputs  # noqa: E402
import paper_2512_09642_b200 as sscg  # noqa: E402

b = torch.from_numpy(inputs.rhs_uniform(64, 64, 1, seed=42)).cuda()
with sscg.Solver(sscg.Stencil("5pt", 64, 64, 1), *inputs.analytic_bounds("5pt", 64, 64), 8, 20) as S:
    S.solve(b, rtol=0.0, max_outer=4)
    torch.cuda.synchronize()
