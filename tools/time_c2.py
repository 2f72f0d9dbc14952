"""Quick C2 timing of one libmcr build (MCR_LIB selects the .so): SpMV alone + both solves."""
import ctypes, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1210_6412_b200 import _lib
from paper_1210_6412_b200.solvers import DeviceMatrix
from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix, generate_rhs, trial_seed
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
if cfg == "c2":
    n, nnz = 10**6, 10**7; seed = trial_seed(0, n, None, nnz, 0); spec = GenSpec(n=n, nnz=nnz, seed=seed)
elif cfg == "c1":
    n = 2000; seed = trial_seed(0, n, 0.1, None, 0); spec = GenSpec(n=n, density=0.1, seed=seed)
elif cfg == "c3":
    n = 16384; seed = 3; spec = GenSpec(n=n, density=1.0, seed=seed)
m = generate_dd_matrix(spec); b = generate_rhs(n, seed); nnz = m.m
L = _lib.load(); dm = DeviceMatrix(m, 0, int(os.environ.get('MCR_STORAGE', '0')))
s = torch.cuda.Stream(); L.mcr_set_stream(dm.handle, ctypes.c_void_p(s.cuda_stream))
x = torch.rand(n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
ts = []
with torch.cuda.stream(s):
    for i in range(25):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        rc = L.mcr_matvec_device(dm.handle, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()))
        e1.record(s); s.synchronize(); assert rc == 0, _lib.last_error()
        if i >= 5: ts.append(e0.elapsed_time(e1))
    spmv = statistics.median(ts) * 1e-3
    B = 12 * nnz + 8 * (n + 1) + 16 * n
    bd = torch.from_numpy(b).cuda(); xo = torch.empty_like(bd)
    res = {}
    for name, fn in (("jacobi", L.mcr_jacobi_device), ("bicgstab", L.mcr_bicgstab_device)):
        best = None
        for _ in range(3):
            flush.zero_(); s.synchronize()
            rep = _lib.Report()
            rc = fn(dm.handle, ctypes.c_void_p(bd.data_ptr()), None, 1e-10, 10000, ctypes.c_void_p(xo.data_ptr()), ctypes.byref(rep))
            best = rep if best is None or rep.device_seconds < best.device_seconds else best
        res[name] = (rc, best.iterations, round(best.device_seconds * 1e3, 3), best.kernel_launches)
print(os.environ.get("MCR_LIB", "default"), os.environ.get("MCR_STORAGE", "0"), cfg, f"spmv {spmv*1e6:.1f}us {B/spmv/1e9:.0f}GB/s", res, flush=True)
