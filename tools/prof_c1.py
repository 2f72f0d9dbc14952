"""Profiling driver: C1 (n=2000, 10%) Jacobi / BiCGStab small-system kernels (run under ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1210_6412_b200 import solvers
from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix, generate_rhs, trial_seed
n = 2000; seed = trial_seed(0, n, 0.1, None, 0)
m = generate_dd_matrix(GenSpec(n=n, density=0.1, seed=seed)); b = generate_rhs(n, seed)
dm = solvers.device_matrix(m)
print(dm.info())
for method, it in (("jacobi", 300), ("bicgstab", 20)):
    rc, x, rep = dm.solve(method, b, None, 1e-10, it)
    print(method, rc, rep.iterations, rep.device_seconds)
