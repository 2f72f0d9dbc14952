import sys, ctypes, numpy as np
sys.path.insert(0, '.')
from paper_1210_6412_b200 import _lib
from paper_1210_6412_b200.generator import pcg_words
L = _lib.load()
for size in (2**32, 2**32 - 1, 2**32 + 1):
    out = np.zeros(6, dtype=np.uint64)
    rc = L.mcr_refgen_u64(0, 6, ctypes.c_uint64(size), pcg_words(0).ctypes.data, out.ctypes.data)
    print(size, rc, _lib.last_error() if rc else "", out.tolist(), np.random.default_rng(0).integers(0, size, size=6, dtype=np.uint64).tolist())
