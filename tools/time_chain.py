"""Chain-shaped workload C2': n = 1e6 random DTMC -> reduced system -> solve.
Times the device path (ChainSystem build, Jacobi and BiCGStab solves) and, once, the
reference's own build_system + reachability_probabilities on the host cores."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1210_6412_b200 import markov
from paper_1210_6412_b200.chains import random_dtmc
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
d = random_dtmc(n, 4)
out = {"n": n}
for rep in range(3):
    t0 = time.perf_counter(); cs = markov.ChainSystem(d, d.goals); t1 = time.perf_counter()
    xj, rj = cs.solve("jacobi-gpu"); t2 = time.perf_counter()
    xb, rb = cs.solve("bicgstab-gpu"); t3 = time.perf_counter()
    out[f"run{rep}"] = {"build_s": t1 - t0, "jacobi_s": t2 - t1, "jacobi_it": rj.iterations,
                        "bicgstab_s": t3 - t2, "bicgstab_it": rb.iterations, "k": cs.k,
                        "m_nnz": cs.m_nnz}
    cs.close()
print(json.dumps(out), flush=True)
if "--reference" in sys.argv:
    sys.path.append(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref"))
    from mcreach.markov import GoalSet, MarkovChain, build_system, reachability_probabilities
    from mcreach.sparse import CsrMatrix
    ch = MarkovChain(n, CsrMatrix(n, d.transitions.rstart, d.transitions.col, d.transitions.nonzero), d.initial)
    t0 = time.perf_counter(); s = build_system(ch, GoalSet(d.goals.tolist())); t1 = time.perf_counter()
    x, r = reachability_probabilities(ch, GoalSet(d.goals.tolist()), "bicgstab-par"); t2 = time.perf_counter()
    print(json.dumps({"reference_build_system_s": t1 - t0, "reference_bicgstab_par_total_s": t2 - t1,
                      "bicgstab_it": r.iterations, "cores": os.cpu_count(),
                      "max_abs_diff_vs_gpu_bicgstab": float(np.max(np.abs(x - xb)))}), flush=True)
