import sys, math, time
sys.path.insert(0, '/root/repo')
import numpy as np, scipy.sparse as sp
from paper_1210_6412_b200.generator import *
n, nnz = 10**6, 10**7
seed = trial_seed(0, n, None, nnz, 0)
m = generate_dd_matrix(GenSpec(n=n, nnz=nnz, seed=seed)); b = generate_rhs(n, seed)
A = sp.csr_matrix((m.nonzero, m.col, m.rstart), shape=(n, n))
def seqdot(u, v): return float(np.cumsum(u*v)[-1])
def fsum(u, v): return math.fsum((u*v).tolist())
def tiles(u, v):
    p = (u*v)
    # emulate per-2048-chunk partials + sequential over chunks
    parts = np.add.reduceat(p, np.arange(0, len(p), 2048))
    return float(np.cumsum(parts)[-1])
def run(dot, tol=1e-10):
    x = np.zeros(n); r = b - A@x; q = r.copy(); y=a=w=1.0; v=np.zeros(n); p=np.zeros(n)
    hist=[]
    for it in range(1, 10000):
        yp=y; y=dot(q,r); beta=(y*a)/(yp*w); p = r + beta*(p - w*v); v = A@p; qv=dot(q,v); a=y/qv
        s = r - a*v; t = A@s; ms = float(np.max(np.abs(s))); hist.append(ms)
        tt=dot(t,t); w = dot(t,s)/tt; x = x + a*p + w*s; r = s - w*t
        if ms <= tol: return it, hist
for name, d in (("seq", seqdot), ("npdot", np.dot), ("fsum", fsum), ("tiles", tiles)):
    t=time.time(); it, h = run(d); print(name, it, ["%.2e"%v for v in h[-8:]], time.time()-t, flush=True)
