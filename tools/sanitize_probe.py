"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family once on small systems -- tiles, cooperative small solvers, SELL, dense,
sequential dots, row shards (local group, 2 ranks), the C5 generator and the chain build."""
import os, sys
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests")]
import numpy as np
from golden_cases import system
from chain_cases import chain
from paper_1210_6412_b200 import dist, markov, solvers
for name in ("grid_20_9", "c4_667_1333", "kat_breakdown_qv", "dense_1024"):
    m, b = system(name)
    for storage in (0, 2, 3, 5):
        if storage == 2 and m.n < 64:
            continue
        dm = solvers.DeviceMatrix(m, 0, storage)
        for method in ("jacobi", "bicgstab"):
            dm.solve(method, b, None, 1e-10, 200)
        dm.solve("bicgstab", b, None, 1e-10, 50, dots="sequential")
        dm.matvec(np.ones(m.n))
        dm.close()
m, b = system("c1_seed77")  # grid-variant small solvers, long tiles (unrolled speculative gathers)
dm = solvers.DeviceMatrix(m, 0)
dm.solve("jacobi", b, None, 1e-10, 30)
dm.solve("bicgstab", b, None, 1e-10, 5)
dm.close()
m, b = system("c4_2000_3999")
dist.solve_local_group("jacobi", m, b, 2)
dist.solve_local_group("bicgstab", m, b, 2)
g = solvers.DeviceMatrix.generated(5000, 7.0, 1, 10, 3)
g.export()
g.close()
ch, goals = chain("oracle_chain_5")
markov.reachability_probabilities(ch, goals)
ch, goals = chain("dtmc_1000")
markov.reachability_probabilities(ch, goals, "bicgstab-gpu")
print("sanitize probe done")
