"""Profiling driver (run under ncu on the GPU box): C2 solves through the device API."""
import sys, os, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1210_6412_b200 import solvers
from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix, generate_rhs, trial_seed
ap = argparse.ArgumentParser()
ap.add_argument("--jacobi-it", type=int, default=10000)
ap.add_argument("--bicg-it", type=int, default=10000)
ap.add_argument("--dense", action="store_true")
a = ap.parse_args()
if a.dense:
    n, seed = 16384, 3
    m = generate_dd_matrix(GenSpec(n=n, density=1.0, seed=seed)); b = generate_rhs(n, seed)
else:
    n, nnz = 10**6, 10**7
    seed = trial_seed(0, n, None, nnz, 0)
    m = generate_dd_matrix(GenSpec(n=n, nnz=nnz, seed=seed)); b = generate_rhs(n, seed)
dm = solvers.device_matrix(m)
print(dm.info(), flush=True)
for method, it in (("jacobi", a.jacobi_it), ("bicgstab", a.bicg_it)):
    rc, x, rep = dm.solve(method, b, None, 1e-10, it)
    print(method, rc, rep.iterations, rep.device_seconds, rep.kernel_launches, flush=True)
