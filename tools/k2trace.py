import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '.')
import inputs, paper_2512_09642_b200 as sscg
L = sscg.load('tools/libsscg_trace.so')
for N in [int(v) for v in sys.argv[1:]]:
    lmin, lmax = inputs.analytic_bounds("7pt", N, N, N)
    b = torch.from_numpy(inputs.rhs_uniform(N, N, N)).cuda()
    with sscg.Solver(sscg.Stencil("7pt", N, N, N), lmin, lmax, 16, 30) as S:
        x = S.solve(b, rtol=0.0, max_outer=0)
        S.iterate(x, 2)
        torch.cuda.synchronize()
        h = (C.c_ulonglong * (148 * 8))()
        print('rc', L.sscg_debug_k2_trace(h))
        t = np.array(h[:], dtype=np.float64).reshape(148, 8)
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3
        names = ['start', 'prod_done', 'cons_done', 'pre_bar', 'post_bar', 'pre_last', 'end']
        print(N, ' '.join('%s[min %.1f med %.1f max %.1f]' % (nm, rel[:, i].min(), np.median(rel[:, i]), rel[:, i].max()) for i, nm in enumerate(names)))
