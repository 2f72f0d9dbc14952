"""Profiling driver: C2 SpMV launches + short solves through the device C ABI."""
import sys, os, ctypes, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1210_6412_b200 import _lib
from paper_1210_6412_b200.solvers import DeviceMatrix
from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix, generate_rhs, trial_seed
ap = argparse.ArgumentParser(); ap.add_argument("--mv", type=int, default=5); ap.add_argument("--jit", type=int, default=5); ap.add_argument("--bit", type=int, default=3)
a = ap.parse_args()
n, nnz = 10**6, 10**7
seed = trial_seed(0, n, None, nnz, 0)
m = generate_dd_matrix(GenSpec(n=n, nnz=nnz, seed=seed)); b = generate_rhs(n, seed)
L = _lib.load(); dm = DeviceMatrix(m, 0); print(dm.info(), flush=True)
x = torch.rand(n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
for i in range(a.mv):
    rc = L.mcr_matvec_device(dm.handle, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()))
    assert rc == 0, _lib.last_error()
torch.cuda.synchronize()
from oracle import oracle
ref = oracle.spmv(m, x.cpu().numpy())
print("spmv bitwise:", np.array_equal(ref, y.cpu().numpy()), flush=True)
bd = torch.from_numpy(b).cuda(); xo = torch.empty_like(bd)
for fn, it in ((L.mcr_jacobi_device, a.jit), (L.mcr_bicgstab_device, a.bit)):
    rep = _lib.Report()
    rc = fn(dm.handle, ctypes.c_void_p(bd.data_ptr()), None, 1e-10, it, ctypes.c_void_p(xo.data_ptr()), ctypes.byref(rep))
    print(rc, rep.iterations, rep.device_seconds, rep.kernel_launches, flush=True)
