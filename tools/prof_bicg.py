"""Profiling driver: a few C2 BiCGStab iterations (run under ncu -k regex:'k_phase|k_spmv')."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1210_6412_b200 import solvers
from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix, generate_rhs, trial_seed
n, nnz = 10**6, 10**7
seed = trial_seed(0, n, None, nnz, 0)
m = generate_dd_matrix(GenSpec(n=n, nnz=nnz, seed=seed)); b = generate_rhs(n, seed)
dm = solvers.device_matrix(m)
rc, x, rep = dm.solve("bicgstab", b, None, 1e-10, int(sys.argv[1]) if len(sys.argv) > 1 else 3)
print(rc, rep.iterations, rep.device_seconds)
