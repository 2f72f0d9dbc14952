"""Quick C2 timing through the host API (development probe, not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1210_6412_b200 import solvers
from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix, generate_rhs, trial_seed

n, nnz = 10**6, 10**7
seed = trial_seed(0, n, None, nnz, 0)
t = time.time(); m = generate_dd_matrix(GenSpec(n=n, nnz=nnz, seed=seed)); b = generate_rhs(n, seed)
print("gen", time.time() - t, flush=True)
t = time.time(); dm = solvers.device_matrix(m); print("upload", time.time() - t, dm.info(), flush=True)
for method in ("jacobi", "bicgstab", "jacobi", "bicgstab"):
    t = time.time()
    rc, x, rep = dm.solve(method, b, None, 1e-10, 10000)
    print(method, rc, rep.iterations, "dev_s", rep.device_seconds, "wall", time.time() - t,
          "launches", rep.kernel_launches, "resid", rep.residual_inf, flush=True)
y = np.random.default_rng(1).random(n)
for _ in range(3):
    t = time.time(); dm.matvec(y); print("matvec host", time.time() - t)
