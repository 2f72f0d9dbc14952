"""How much does BiCGStab's iteration count move when ONLY the inner-product summation order
changes? Runs the reference algorithm (solvers.py:450-491) in numpy with four dot products:
the reference's strict left-to-right cumsum, math.fsum (exactly rounded), numpy's BLAS dot and
per-2048 chunk partials summed in order (like the GPU tree). Usage:
    python tools/bicgstab_sensitivity.py [case ...]      (golden case names; default: all <= 20k)
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import scipy.sparse as sp

from golden_cases import case_names, manifest, system


def seqdot(u, v):
    return float(np.cumsum(u * v)[-1]) if len(u) else 0.0


def fsum(u, v):
    return math.fsum((u * v).tolist())


def chunks(u, v):
    p = u * v
    return float(np.cumsum(np.add.reduceat(p, np.arange(0, len(p), 2048)))[-1])


def bicgstab(A, b, dot, tol=1e-10, max_it=10000):
    n = len(b)
    x = np.zeros(n); r = b - A @ x
    if np.max(np.abs(r)) <= tol:
        return 0
    q = r.copy(); y = a = w = 1.0; v = np.zeros(n); p = np.zeros(n)
    for it in range(1, max_it + 1):
        yp = y; y = dot(q, r); den = yp * w
        if den == 0.0 or abs(den) < 1e-300:
            return f"bd@{it}"
        beta = (y * a) / den; p = r + beta * (p - w * v); v = A @ p; qv = dot(q, v)
        if qv == 0.0 or abs(qv) < 1e-300:
            return f"bd@{it}"
        a = y / qv; s = r - a * v; t = A @ s; small = np.max(np.abs(s)) <= tol
        tt = dot(t, t)
        if tt == 0.0 or abs(tt) < 1e-300:
            if not small:
                return f"bd@{it}"
            w = 0.0
        else:
            w = dot(t, s) / tt
        x = x + a * p + w * s; r = s - w * t
        if small:
            return it
    return f"nc@{max_it}"


if __name__ == "__main__":
    names = sys.argv[1:] or [c for c in case_names(max_n=20000)
                             if manifest()["cases"][c]["config"]["guess_seed"] is None]
    for name in names:
        m, b = system(name)
        A = sp.csr_matrix((m.nonzero, m.col, m.rstart), shape=(m.n, m.n))
        res = {k: bicgstab(A, b, f) for k, f in
               (("sequential", seqdot), ("fsum", fsum), ("blas", np.dot), ("chunks", chunks))}
        ref = manifest()["cases"][name]["results"]["bicgstab"].get("iterations")
        ints = [v for v in res.values() if isinstance(v, int)]
        spread = (max(ints) - min(ints)) if ints else 0
        print(f"{name:28s} ref={ref} {res} spread={spread}", flush=True)
