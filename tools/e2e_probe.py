"""Breakdown of the end-to-end (host-buffer) path: upload, solves, destroy."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1210_6412_b200 import _lib
from paper_1210_6412_b200.solvers import DeviceMatrix
from paper_1210_6412_b200.sparse import CsrMatrix
from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix, generate_rhs, trial_seed
n, nnz = 10**6, 10**7; seed = trial_seed(0, n, None, nnz, 0)
m = generate_dd_matrix(GenSpec(n=n, nnz=nnz, seed=seed)); b = generate_rhs(n, seed)
def pinned(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory(); return t, t.numpy()
ts = [pinned(a) for a in (m.rstart, m.col, m.nonzero, b, np.zeros(n))]
hm = CsrMatrix(n, ts[0][1], ts[1][1], ts[2][1]); bh = ts[3][1]; xh = ts[4][1]
L = _lib.load()
for it in range(4):
    t0 = time.perf_counter(); h = DeviceMatrix(hm, 0); t1 = time.perf_counter()
    out = []
    for fn in (L.mcr_jacobi, L.mcr_bicgstab):
        rep = _lib.Report(); a = time.perf_counter()
        rc = fn(h.handle, ctypes.c_void_p(bh.ctypes.data), None, 1e-10, 10000, ctypes.c_void_p(xh.ctypes.data), ctypes.byref(rep))
        out.append((rc, rep.iterations, round((time.perf_counter() - a) * 1e3, 2), round(rep.device_seconds * 1e3, 2)))
    t2 = time.perf_counter(); h.close(); t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f}ms solves {out} destroy {1e3*(t3-t2):.1f}ms total {1e3*(t3-t0):.1f}ms", flush=True)
