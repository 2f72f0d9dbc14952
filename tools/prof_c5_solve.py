"""C5 solve timing: python tools/prof_c5_solve.py [n] [storage] [max_it] [dots] -- Jacobi and
BiCGStab device time per sweep / iteration on the generated C5 system (run under ncu for a launch
list). dots: 0 tree (default), 1 the reference's order (k_xdot)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_6412_b200 import _lib
from paper_1210_6412_b200.solvers import DeviceMatrix
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000000
storage = int(sys.argv[2]) if len(sys.argv) > 2 else 0
max_it = int(sys.argv[3]) if len(sys.argv) > 3 else 10000
dots = int(sys.argv[4]) if len(sys.argv) > 4 else 0
L = _lib.load()
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
dm = DeviceMatrix.generated(n, 7.0, 1, 10, 2024, storage=storage)
L.mcr_set_stream(dm.handle, ctypes.c_void_p(stream.cuda_stream))
assert L.mcr_set_dot_mode(dm.handle, dots) == 0
b = torch.empty(n, dtype=torch.float64, device="cuda"); dm.generated_rhs(2024, b.data_ptr())
x = torch.empty_like(b)
for name, fn in (("jacobi", L.mcr_jacobi_device), ("bicgstab", L.mcr_bicgstab_device)):
    rep = _lib.Report()
    rc = fn(dm.handle, ctypes.c_void_p(b.data_ptr()), None, 1e-10, max_it, ctypes.c_void_p(x.data_ptr()), ctypes.byref(rep))
    it = max(1, rep.iterations)
    print(f"{name}: storage={dm.info()['storage']} rc={rc} it={rep.iterations} {rep.device_seconds*1e3:.1f} ms "
          f"({rep.device_seconds*1e3/it:.2f} ms/it) launches={rep.kernel_launches}", flush=True)
