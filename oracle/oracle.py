"""ctypes front end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may import this
module; the product package never does. It wraps ``oracle/liboracle.so`` (built from
``oracle.c`` by ``oracle/Makefile``), a sequential C restatement of the reference solvers
(``mcreach/solvers.py``), and returns plain dicts so a test can compare them field by field
with the GPU solver's ``SolveResult``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

OK, NOT_CONVERGED, BREAKDOWN, ZERO_DIAGONAL = 0, 1, 2, 3
BREAKDOWN_NAMES = {1: "y_prev*w", 2: "q*v", 3: "t*t"}

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "oracle.c"))
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_set_threads.argtypes = [ctypes.c_int]
        L.orc_spmv.argtypes = [ctypes.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p]
        L.orc_dot.argtypes = [ctypes.c_int64, _f64p, _f64p]
        L.orc_dot.restype = ctypes.c_double
        L.orc_residual_inf.argtypes = [ctypes.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p]
        L.orc_residual_inf.restype = ctypes.c_double
        L.orc_jacobi.argtypes = [ctypes.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p,
                                 ctypes.c_double, ctypes.c_int64, _i64p, _f64p, _i64p]
        L.orc_bicgstab.argtypes = [ctypes.c_int64, _i64p, _i64p, _f64p, _f64p, _f64p,
                                   ctypes.c_double, ctypes.c_int64, _i64p, _f64p,
                                   ctypes.POINTER(ctypes.c_int)]
        L.orc_generate.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_double, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_int64, ctypes.c_int64, _i64p, _i64p,
                                   _f64p]
        L.orc_generate_rhs.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, _f64p]
        _lib = L
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(t)


def _csr(m):
    rp = np.ascontiguousarray(m.rstart, dtype=np.int64)
    col = np.ascontiguousarray(m.col, dtype=np.int64)
    val = np.ascontiguousarray(m.nonzero, dtype=np.float64)
    return int(m.n), rp, col, val


def set_threads(t: int) -> None:
    lib().orc_set_threads(int(t))


def initial_guess(n: int, guess_seed):
    """solvers.py:153-156"""
    if guess_seed is None:
        return np.zeros(n)
    return np.random.default_rng(guess_seed).random(n)


def spmv(m, x) -> np.ndarray:
    n, rp, col, val = _csr(m)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(n)
    lib().orc_spmv(n, _ptr(rp, _i64p), _ptr(col, _i64p), _ptr(val, _f64p),
                   _ptr(x, _f64p), _ptr(y, _f64p))
    return y


def dot(u, v) -> float:
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    return float(lib().orc_dot(len(u), _ptr(u, _f64p), _ptr(v, _f64p)))


def residual_inf(m, x, b) -> float:
    n, rp, col, val = _csr(m)
    x = np.ascontiguousarray(x, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return float(lib().orc_residual_inf(n, _ptr(rp, _i64p), _ptr(col, _i64p),
                                        _ptr(val, _f64p), _ptr(x, _f64p), _ptr(b, _f64p)))


def jacobi(m, b, tolerance=1e-10, max_iterations=10_000, guess_seed=None) -> dict:
    n, rp, col, val = _csr(m)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.ascontiguousarray(initial_guess(n, guess_seed), dtype=np.float64)
    it = ctypes.c_int64(0)
    res = ctypes.c_double(0.0)
    zi = ctypes.c_int64(-1)
    st = lib().orc_jacobi(n, _ptr(rp, _i64p), _ptr(col, _i64p), _ptr(val, _f64p),
                          _ptr(b, _f64p), _ptr(x, _f64p), float(tolerance),
                          int(max_iterations), ctypes.byref(it), ctypes.byref(res),
                          ctypes.byref(zi))
    return {"status": st, "x": x, "iterations": it.value, "converged": st == OK,
            "residual_inf": res.value, "zero_index": zi.value}


def bicgstab(m, b, tolerance=1e-10, max_iterations=10_000, guess_seed=None) -> dict:
    n, rp, col, val = _csr(m)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.ascontiguousarray(initial_guess(n, guess_seed), dtype=np.float64)
    it = ctypes.c_int64(0)
    res = ctypes.c_double(0.0)
    which = ctypes.c_int(0)
    st = lib().orc_bicgstab(n, _ptr(rp, _i64p), _ptr(col, _i64p), _ptr(val, _f64p),
                            _ptr(b, _f64p), _ptr(x, _f64p), float(tolerance),
                            int(max_iterations), ctypes.byref(it), ctypes.byref(res),
                            ctypes.byref(which))
    return {"status": st, "x": x, "iterations": it.value, "converged": st == OK,
            "residual_inf": res.value, "which": BREAKDOWN_NAMES.get(which.value)}


class _Rows:
    """Row block of a generated system: n rows, local rstart, global col (int64), nonzero."""

    def __init__(self, n, rstart, col, nonzero):
        self.n, self.rstart, self.col, self.nonzero = n, rstart, col, nonzero

    @property
    def m(self):
        return int(self.rstart[-1])


def generate(seed: int, n: int, mean: float = 7.0, lo: int = 1, hi: int = 10, row0: int = 0,
             rows=None):
    """Rows [row0, row0 + rows) of the row-keyed synthetic system (csrc/generator.cuh)."""
    rows = n - row0 if rows is None else rows
    rs = np.zeros(rows + 1, dtype=np.int64)
    L = lib()
    L.orc_generate(seed, n, mean, lo, hi, row0, rows, _ptr(rs, _i64p), None, None)
    col = np.empty(int(rs[-1]), dtype=np.int64)
    val = np.empty(int(rs[-1]), dtype=np.float64)
    L.orc_generate(seed, n, mean, lo, hi, row0, rows, _ptr(rs, _i64p), _ptr(col, _i64p),
                   _ptr(val, _f64p))
    return _Rows(rows, rs, col, val)


def generate_rhs(seed: int, n: int, row0: int = 0, rows=None) -> np.ndarray:
    rows = n - row0 if rows is None else rows
    b = np.empty(rows)
    lib().orc_generate_rhs(seed, row0, rows, _ptr(b, _f64p))
    return b
