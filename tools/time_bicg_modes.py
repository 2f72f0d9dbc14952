"""BiCGStab on C2 (and C1 / a C4 shape) in each dot mode: iterations, device time, x equality."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1210_6412_b200 import _lib
from paper_1210_6412_b200.solvers import DeviceMatrix
from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix, generate_rhs, trial_seed

cases = {
    "c2": lambda: GenSpec(n=10**6, nnz=10**7, seed=trial_seed(0, 10**6, None, 10**7, 0)),
    "c1": lambda: GenSpec(n=2000, density=0.1, seed=trial_seed(0, 2000, 0.1, None, 0)),
    "c4_5647": lambda: GenSpec(n=5647, nnz=11293, seed=trial_seed(0, 5647, None, 11293, 0)),
}
L = _lib.load()
for name in (sys.argv[1:] or ["c2", "c1", "c4_5647"]):
    spec = cases[name]()
    m = generate_dd_matrix(spec)
    b = generate_rhs(m.n, spec.seed)
    dm = DeviceMatrix(m, 0)
    xs = {}
    for mode in ("tree", "sequential", "serial"):
        if mode == "serial" and name == "c2" and "--serial" not in os.environ.get("XARGS", ""):
            pass
        times = []
        for rep_i in range(4):
            rc, x, rep = dm.solve("bicgstab", b, None, 1e-10, 10000, dots=mode)
            times.append(rep.device_seconds)
        xs[mode] = x
        t = min(times[1:])
        print(f"{name:8s} {mode:10s} rc={rc} it={rep.iterations:3d} {t*1e3:8.3f} ms  "
              f"{t/max(rep.iterations,1)*1e6:7.1f} us/it  launches={rep.kernel_launches} resid={rep.residual_inf:.3e}", flush=True)
    print(f"{name:8s} sequential == serial bitwise: {np.array_equal(xs['sequential'], xs['serial'])}", flush=True)
