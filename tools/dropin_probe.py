"""Breakdown of bench.py's e2e step (the drop-in path): the reference CsrMatrix built over
pageable numpy arrays, jacobi-gpu (upload + solve + x to the host), bicgstab-gpu, cache drop.
Run with MCR_TRACE=1 for the library's own create / solve stage marks."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1210_6412_b200 import plugin
from paper_1210_6412_b200 import solvers as gsolvers

m, b, desc, spec = bench.make_workload("c2")
ms = bench.reference_module()
reg = dict(ms.SOLVERS)
plugin.install(reg)
from mcreach import CsrMatrix as RefCsr
n = int(m.n)
cfg = gsolvers.SolverConfig(dot_products="sequential", device=0)
rs_p, col_p, val_p, b_p = (np.array(m.rstart), np.array(m.col), np.array(m.nonzero), np.array(b))
torch.cuda.init()
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mat = RefCsr(n, rs_p, col_p, val_p)
    t1 = time.perf_counter()
    rj = bench._drop_in(reg["jacobi-gpu"], mat, b_p, cfg)
    t2 = time.perf_counter()
    rb = bench._drop_in(reg["bicgstab-gpu"], mat, b_p, cfg)
    t3 = time.perf_counter()
    del mat
    gsolvers._cache.clear()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"csr {1e3*(t1-t0):.2f} jacobi {1e3*(t2-t1):.2f} ({rj.iterations}) bicgstab {1e3*(t3-t2):.2f} "
          f"({rb.iterations}) drop {1e3*(t4-t3):.2f} total {1e3*(t4-t0):.2f} ms", flush=True)
