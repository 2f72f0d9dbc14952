"""One BiCGStab solve in sequential-dot mode (for ncu launch lists / stats)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1210_6412_b200 import _lib, dots
from paper_1210_6412_b200.solvers import DeviceMatrix
from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix, generate_rhs, trial_seed
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
if name == "c2":
    spec = GenSpec(n=10**6, nnz=10**7, seed=trial_seed(0, 10**6, None, 10**7, 0))
else:
    n, nnz = {"c4_5647": (5647, 11293), "c1": (2000, None)}[name]
    spec = GenSpec(n=n, nnz=nnz, seed=trial_seed(0, n, None, nnz, 0)) if nnz else GenSpec(n=n, density=0.1, seed=trial_seed(0, n, 0.1, None, 0))
m = generate_dd_matrix(spec); b = generate_rhs(m.n, spec.seed)
dm = DeviceMatrix(m, 0)
for _ in range(reps):
    rc, x, rep = dm.solve("bicgstab", b, None, 1e-10, 10000, dots="sequential")
    print(name, rc, rep.iterations, rep.device_seconds * 1e3, "ms", flush=True)
if os.environ.get("MCR_XDOT_STATS"):
    st = np.zeros(len(dots.XDOT_STATS), dtype=np.uint64)
    _lib.load().mcr_xdot_stats(dm.handle, st.ctypes.data, len(st))
    print({k: int(v) for k, v in zip(dots.XDOT_STATS, st) if v})
