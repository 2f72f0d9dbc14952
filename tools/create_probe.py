"""Time mcr_matrix_create from pageable numpy arrays (the drop-in's upload) at C2 size, with
the pinned chunk ring (MCR_H2D_RING=1, default) and with plain pageable cudaMemcpyAsync
(MCR_H2D_RING=0): `python tools/create_probe.py` runs both in subprocesses."""
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child():
    import numpy as np
    from paper_1210_6412_b200 import _lib
    from paper_1210_6412_b200.solvers import DeviceMatrix
    from paper_1210_6412_b200.sparse import CsrMatrix
    n, k = 1_000_000, 10
    rng = np.random.default_rng(1)
    col = np.sort(rng.integers(0, n, size=(n, k)), axis=1).astype(np.int64)
    col += np.arange(k)[None, :]          # strictly increasing within a row
    col = np.minimum(col, n - 1)
    col = np.maximum.accumulate(col, axis=1)
    ok = np.all(np.diff(col, axis=1) > 0, axis=1)
    col[~ok] = np.arange(k)[None, :]
    col = col.ravel()
    rs = np.arange(0, n * k + 1, k, dtype=np.int64)
    val = rng.random(n * k)
    m = CsrMatrix(n, rs, col, val)
    _lib.load()
    ts = []
    for i in range(8):
        t0 = time.perf_counter()
        h = DeviceMatrix(m, 0)
        dt = time.perf_counter() - t0
        h.close()
        if i >= 2:
            ts.append(dt)
    mb = (rs.nbytes + col.nbytes + val.nbytes) / 1e6
    print(f"ring={os.environ.get('MCR_H2D_RING', '1')} threads={os.environ.get('MCR_H2D_THREADS', '8')}: create {1e3 * min(ts):.2f} ms min, "
          f"{1e3 * sum(ts) / len(ts):.2f} ms mean for {mb:.0f} MB ({mb / 1e3 / min(ts):.1f} GB/s)")


if __name__ == "__main__":
    if len(sys.argv) > 1:
        child()
    else:
        for ring, th in (("0", "8"), ("1", "4"), ("1", "8"), ("1", "12"), ("1", "16")):
            subprocess.run([sys.executable, __file__, "child"],
                           env={**os.environ, "MCR_H2D_RING": ring, "MCR_H2D_THREADS": th})
