"""Iteration counts / errors of one golden case across storages and dot modes (GPU)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
from golden_cases import expected, system
from paper_1210_6412_b200.solvers import DeviceMatrix
for name in sys.argv[1:]:
    m, b = system(name)
    for meth in ("bicgstab", "jacobi"):
        exp = expected(name, meth)
        for storage in (2, 3, 4, 5):
            dm = DeviceMatrix(m, 0, storage)
            for dots in ("tree", "sequential"):
                rc, x, rep = dm.solve(meth, b, None, exp["config"]["tolerance"], exp["config"]["max_iterations"], dots)
                err = float(np.max(np.abs(x - exp["x"]))) if exp["x"] is not None else -1
                print(name, meth, storage, dots, "rc", rc, "it", rep.iterations, "ref", exp["iterations"], "err %.2e" % err, flush=True)
            dm.close()
