"""C4 (Table-1 shapes): time-to-solution of Jacobi and BiCGStab on the 18 JPF
shapes (GenSpec(n, nnz=m, seed=trial_seed(0, n, None, m, 0))), device time per solve."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1210_6412_b200 import solvers
from paper_1210_6412_b200.generator import (TABLE1_SHAPES, GenSpec, generate_dd_matrix,
                                            generate_rhs, trial_seed)
rows = []
for n, mm in TABLE1_SHAPES:
    spec = GenSpec(n=n, nnz=mm, seed=trial_seed(0, n, None, mm, 0))
    m = generate_dd_matrix(spec); b = generate_rhs(spec.n, spec.seed)
    dm = solvers.DeviceMatrix(m, 0)
    best = {}
    for method, dots in (("jacobi", "sequential"), ("bicgstab", "sequential"), ("bicgstab", "tree")):
        ts = []
        for _ in range(5):
            rc, x, rep = dm.solve(method, b, None, 1e-10, 10000, dots=dots)
            ts.append(rep.device_seconds)
        key = method if dots == "sequential" else f"{method}_{dots}"
        best[key] = (int(rep.iterations), 1e3 * sorted(ts)[2], int(rep.kernel_launches))
    rows.append({"n": spec.n, "m": int(m.m), "storage": dm.info()["storage"], **best})
    dm.close()
print(json.dumps({"c4": rows, "note": "(iterations, device ms median of 5, kernel launches); "
                  "bicgstab = reference-order dots (default), bicgstab_tree = opt-in tree dots"}))
