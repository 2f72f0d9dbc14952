"""Profiling driver: SpMV of a generated C5-family system (run under ncu)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_6412_b200 import _lib
from paper_1210_6412_b200.solvers import DeviceMatrix
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000000
L = _lib.load(); dm = DeviceMatrix.generated(n, 7.0, 1, 10, 2024, storage=_lib.STORAGE_TILES)
print(dm.info(), flush=True)
x = torch.rand(n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
for i in range(2):
    assert L.mcr_matvec_device(dm.handle, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr())) == 0
torch.cuda.synchronize()
