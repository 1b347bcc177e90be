import os, sys
sys.path.insert(0, '.')
os.environ['SSCG_DEBUG'] = '1'
import torch, numpy as np, inputs, paper_2512_09642_b200 as sscg
n = 32
kx, ky, kz = [torch.from_numpy(np.ascontiguousarray(f)).cuda() for f in inputs.lognormal_faces(n, n, n)]
S = sscg.Solver(sscg.Stencil("varcoef7", n, n, n, kx, ky, kz), 0.1, 1.9, 4, 4)
print("ok")
b = torch.from_numpy(inputs.rhs_uniform(n, n, n)).cuda()
x = S.solve(b, rtol=0.0, max_outer=1)
torch.cuda.synchronize()
print("solve ok", float(x.norm()))
