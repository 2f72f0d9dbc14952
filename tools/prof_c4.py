"""Profiling driver: one C4 (Table-1) shape, Jacobi and BiCGStab on the small-system kernels
(run under ncu). python tools/prof_c4.py [n] [m]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1210_6412_b200 import solvers
from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix, generate_rhs, trial_seed
n = int(sys.argv[1]) if len(sys.argv) > 1 else 92
m_ = int(sys.argv[2]) if len(sys.argv) > 2 else 211
seed = trial_seed(0, n, None, m_, 0)
m = generate_dd_matrix(GenSpec(n=n, nnz=m_, seed=seed)); b = generate_rhs(n, seed)
dm = solvers.device_matrix(m)
print(dm.info())
for method in ("jacobi", "bicgstab"):
    rc, x, rep = dm.solve(method, b, None, 1e-10, 10000)
    print(method, rc, rep.iterations, rep.device_seconds)
