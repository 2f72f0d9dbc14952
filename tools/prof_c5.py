"""C5-family SpMV timing / profiling driver: python tools/prof_c5.py [n] [storage ...]."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1210_6412_b200 import _lib
from paper_1210_6412_b200.solvers import DeviceMatrix
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000000
storages = [int(s) for s in sys.argv[2:]] or [0]
L = _lib.load()
x = torch.rand(n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
y0 = None
for st in storages:
    dm = DeviceMatrix.generated(n, 7.0, 1, 10, 2024, storage=st)
    L.mcr_set_stream(dm.handle, ctypes.c_void_p(stream.cuda_stream))
    inf = dm.info()
    ts = []
    for i in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream); assert L.mcr_matvec_device(dm.handle, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr())) == 0; e1.record(stream)
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    t = sorted(ts)[2] * 1e-3
    alg = 12 * inf["nnz"] + 8 * (n + 1) + 16 * n
    same = ""
    if y0 is None:
        y0 = y.clone()
    else:
        same = f" bit-identical to the first: {bool(torch.equal(y, y0))}"
    print(f"n={n} storage={inf['storage']} band={os.environ.get('MCR_STAGED_BAND', 'auto')} nnz={inf['nnz']} bytes={inf['device_bytes']/1e9:.1f}GB spmv {t*1e3:.3f} ms {alg/t/1e9:.0f} GB/s alg{same}", flush=True)
    dm.close()
