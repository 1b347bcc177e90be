"""Accuracy of forming Ghat = P^T A P in Gram space (Ghat = E T, E = P^T P_{:,0:s+1};
SSCG_GRAM_SPACE=1, R27) against per-point recovery of w_j (the default
K2R arithmetic, R23), on the 2D 5-point Laplacian with Jacobi M = 4 I: a rough
residual (mix = 1) and smooth ones (mix = 1e-3, 0: the late-solve case), each
against the same Gram in extended precision.  Plain numpy (no oracle, no GPU).
Columns: max|dG| / max|G|, and max |dG_ij| / sqrt(G_ii G_jj).
    python tools/gram_space_accuracy.py > profiles/r02l_gram_space_accuracy.txt
"""
import numpy as np, sys
def lap2(u):
    v = 4*u.copy()
    v[1:,:]-=u[:-1,:]; v[:-1,:]-=u[1:,:]; v[:,1:]-=u[:,:-1]; v[:,:-1]-=u[:,1:]
    return v
def run(n, s, mix):
    rng=np.random.default_rng(1)
    x=np.arange(1,n+1)/(n+1)
    smooth=np.outer(np.sin(np.pi*x),np.sin(np.pi*x))
    r = smooth + mix*rng.uniform(-1,1,(n,n))
    lmin=(2-2*np.cos(np.pi/(n+1)))*2/4; lmax=(2+2*np.cos(np.pi/(n+1)))*2/4
    th=2/(lmax-lmin); sg=(lmax+lmin)/2; m=4.0
    P=[r]
    P.append(th*(lap2(r)/m - sg*r))
    for j in range(1,s):
        P.append(2*th*(lap2(P[j])/m - sg*P[j]) - P[j-1])
    P=np.array([p.ravel() for p in P])   # s+1
    W=np.array([lap2(p.reshape(n,n)).ravel() for p in P[:s]])
    G1=P[:s]@W[:s].T
    Wr=np.array([m*((P[j+1]/th if j==0 else (P[j+1]+P[j-1])/(2*th)) + sg*P[j]) for j in range(s)])   # R23, per point
    G3=P[:s]@Wr.T
    E=P[:s]@P.T
    T=np.zeros((s+1,s))
    for j in range(s):
        T[j,j]=m*sg; T[j+1,j]=m/th if j==0 else m/(2*th)
        if j>0: T[j-1,j]=m/(2*th)
    G2=E@T
    Pl=P.astype(np.longdouble); Wl=np.array([lap2(p.reshape(n,n)).ravel() for p in Pl[:s]])
    Gr=(Pl[:s]@Wl.T).astype(np.float64)
    sc=np.max(np.abs(Gr))
    # per-entry error relative to sqrt(Gii Gjj) (what Ruhe scaling sees)
    d=np.sqrt(np.diag(Gr))
    rel=lambda G: (np.max(np.abs(G-Gr))/sc, np.max(np.abs(G-Gr)/np.outer(d,d)))
    print(n, s, mix, "kappa~%.1e"%((lmax/lmin)), "SpMV W", "%.1e %.1e"%rel(G1), " per-point recovery", "%.1e %.1e"%rel(G3), " Gram space", "%.1e %.1e"%rel(G2))
for n in (64, 256, 1024):
    for mix in (1.0, 1e-3, 0.0):
        run(n, 16, mix)
