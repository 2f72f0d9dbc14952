"""C5 staged SpMV vs solve timing in one process (PDL placement study):
python tools/prof_c5_pdl.py [n] -- matvec x5, Jacobi 40 sweeps, BiCGStab 20 iterations, matvec x5."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_6412_b200 import _lib
from paper_1210_6412_b200.solvers import DeviceMatrix
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000000
L = _lib.load()
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
dm = DeviceMatrix.generated(n, 7.0, 1, 10, 2024)
L.mcr_set_stream(dm.handle, ctypes.c_void_p(stream.cuda_stream))
b = torch.empty(n, dtype=torch.float64, device="cuda"); dm.generated_rhs(2024, b.data_ptr())
x = torch.rand(n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
tag = f"PDL={os.environ.get('MCR_STAGED_PDL', '0')} NO_PDL={os.environ.get('MCR_NO_PDL', '0')}"

def mv(reps=5):
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        L.mcr_matvec_device(dm.handle, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()))
        e1.record(stream); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return sorted(ts)[reps // 2]

print(tag, f"matvec {mv():.2f} ms", flush=True)
for name, fn, it in (("jacobi", L.mcr_jacobi_device, 40), ("bicgstab", L.mcr_bicgstab_device, 20)):
    rep = _lib.Report()
    fn(dm.handle, ctypes.c_void_p(b.data_ptr()), None, 1e-10, it, ctypes.c_void_p(y.data_ptr()), ctypes.byref(rep))
    print(tag, f"{name} {rep.device_seconds * 1e3 / rep.iterations:.2f} ms/it", flush=True)
print(tag, f"matvec {mv():.2f} ms", flush=True)
