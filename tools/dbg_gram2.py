import math, sys, numpy as np, torch
sys.path.insert(0, '.')
import inputs, paper_2512_09642_b200 as sscg
N, S_, NU = int(sys.argv[1]), 16, 30
lmin, lmax = inputs.analytic_bounds("7pt", N, N, N); theta, sigma = 2/(lmax-lmin), (lmax+lmin)/2
first = None
if len(sys.argv) > 2:
    b = torch.from_numpy(inputs.rhs_uniform(N, N, N)).cuda()
    first = sscg.Solver(sscg.Stencil("7pt", N, N, N), lmin, lmax, S_, NU)
    first.solve(b, rtol=0.0, max_outer=0)
    print("first solver alive")
rng = np.random.default_rng(3)
modes = [tuple(int(v) for v in rng.integers(1, N+1, 3)) for _ in range(20)]
coef = rng.standard_normal(20)
r = torch.zeros(N**3, dtype=torch.float64, device="cuda")
ar = torch.arange(1, N+1, dtype=torch.float64, device="cuda")
for cm, (kx, ky, kz) in zip(coef, modes):
    sx, sy, sz = (torch.sin(k*math.pi*ar/(N+1)) for k in (kx, ky, kz))
    r += float(cm) * (sz[:, None, None]*sy[None, :, None]*sx[None, None, :]).reshape(-1)
with sscg.Solver(sscg.Stencil("7pt", N, N, N), lmin, lmax, S_, NU) as S:
    S.solve(r, rtol=0.0, max_outer=0)
    G, c = S.gram(0)
    p0 = S.basis(0)[0]
print("p0 == r:", np.array_equal(p0, r.cpu().numpy()))
nv2 = ((N+1)/2)**3
Gcf = np.zeros((S_, S_)); ccf = np.zeros(S_)
for cm, ks in zip(coef, modes):
    lamA = inputs.sine_mode_eig("7pt", (N, N, N), ks); x = theta*(lamA/6.0 - sigma)
    T = np.array([math.cos(j*math.acos(x)) for j in range(S_)])
    Gcf += cm*cm*nv2*lamA*np.outer(T, T); ccf += cm*cm*nv2*T
m = np.max(np.abs(Gcf))
print(N, "gpu-vs-cf %.2e" % (np.max(np.abs(G-Gcf))/m), "c %.2e" % (np.max(np.abs(c-ccf))/np.max(np.abs(ccf))))
print(np.argwhere(np.abs(G-Gcf) > 1e-9*m)[:8].tolist())
