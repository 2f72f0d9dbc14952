"""Profiling driver: dense slab GEMV (k_dense) on an n x n fully dense DD system (run under ncu)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1210_6412_b200 import _lib
from paper_1210_6412_b200.solvers import DeviceMatrix
from paper_1210_6412_b200.sparse import CsrMatrix
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
rng = np.random.default_rng(0)
val = rng.integers(1, 11, size=(n, n)).astype(np.float64)
val[np.arange(n), np.arange(n)] = val.sum(1) + 1
m = CsrMatrix(n, np.arange(0, n * n + 1, n, dtype=np.int64), np.tile(np.arange(n, dtype=np.int64), n), val.ravel())
L = _lib.load(); dm = DeviceMatrix(m, 0); print(dm.info(), flush=True)
x = torch.rand(n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
L.mcr_set_stream(dm.handle, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
for i in range(3):
    assert L.mcr_matvec_device(dm.handle, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr())) == 0
torch.cuda.synchronize()
ts = []
for i in range(10):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); L.mcr_matvec_device(dm.handle, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr())); e1.record()
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
t = sorted(ts)[len(ts) // 2] * 1e-3
print(f"dense GEMV n={n}: {t*1e6:.1f} us, {(8*n*n + 16*n)/t/1e9:.0f} GB/s algorithmic", flush=True)
