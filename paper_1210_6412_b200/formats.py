"""Fast readers for the reference's text formats (``mcreach/formats.py``).

``read_matrix`` / ``read_vector`` / ``read_dtmc`` take the same files as the reference
(``formats.py:89-232``) and return the same results -- ``CsrMatrix`` in ``csr_from_triplets``
order, a float64 vector, ``(MarkovChain, GoalSet)`` validated like ``validate()`` -- parsed by
the multithreaded C++ readers in ``libmcr.so`` (``csrc/formats.cpp``). A file outside their
well-formed plain-decimal subset (any error, duplicate, failed check, ``inf``/``nan``,
underscores, non-ASCII) goes to this package's line-by-line readers (``textio.py``), which
restate the reference's rules, so results and errors (``ParseError`` with its line number,
``RowSumError``, ``DuplicateEntry``, ...) are the reference's -- its own classes when
``mcreach`` is importable. The reference's code is never run.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

from . import _lib, textio
from .sparse import CsrMatrix

__all__ = ["ParseError", "read_matrix", "read_vector", "read_dtmc"]


ParseError = textio.ParseError  # formats.py:51-56 (the reference's class is raised when importable)


def _read(fn_name: str, path):
    L = _lib.load()
    h = ctypes.c_void_p()
    rc = getattr(L, fn_name)(os.fsencode(os.fspath(path)), 0, ctypes.byref(h))
    if rc == _lib.MCR_OK:
        return L, h, None
    if rc == _lib.MCR_UNSUPPORTED_INPUT:
        return L, None, L.mcr_text_reason().decode(errors="replace")
    raise _lib.NativeLibraryError(f"{fn_name} failed with status {rc}")


def _info(L, h):
    n, m, initial, ng = (ctypes.c_int64() for _ in range(4))
    L.mcr_text_info(h, ctypes.byref(n), ctypes.byref(m), ctypes.byref(initial), ctypes.byref(ng))
    return n.value, m.value, initial.value, ng.value


def _csr(L, h, n, m):
    rs = np.empty(n + 1, dtype=np.int64)
    col = np.empty(m, dtype=np.int64)
    val = np.empty(m, dtype=np.float64)
    L.mcr_text_export(h, rs.ctypes.data, col.ctypes.data, val.ctypes.data, None)
    return rs, col, val


def _matrix_type():
    try:
        from mcreach.sparse import CsrMatrix as RefCsr
        return RefCsr
    except Exception:
        return CsrMatrix


def read_matrix(path):
    """formats.py:89-113."""
    L, h, why = _read("mcr_read_matrix", path)
    if h is None:
        return textio.read_matrix(path, _matrix_type())
    try:
        n, m, _, _ = _info(L, h)
        rs, col, val = _csr(L, h, n, m)
    finally:
        L.mcr_text_destroy(h)
    return _matrix_type()(n, rs, col, val)


def read_vector(path) -> np.ndarray:
    """formats.py:128-145."""
    L, h, why = _read("mcr_read_vector", path)
    if h is None:
        return textio.read_vector(path)
    try:
        n, _, _, _ = _info(L, h)
        v = np.empty(n, dtype=np.float64)
        L.mcr_text_export(h, None, None, v.ctypes.data, None)
    finally:
        L.mcr_text_destroy(h)
    return v


def read_dtmc(path):
    """formats.py:160-230: (MarkovChain, GoalSet), reference types when importable."""
    L, h, why = _read("mcr_read_dtmc", path)
    if h is None:
        n, initial, goals, p = textio.read_dtmc_parts(path)
        return _chain(n, p.rstart, p.col, p.nonzero, initial, np.array(goals, dtype=np.int64))
    try:
        n, m, initial, ng = _info(L, h)
        rs, col, val = _csr(L, h, n, m)
        goals = np.empty(ng, dtype=np.int64)
        L.mcr_text_export(h, None, None, None, goals.ctypes.data)
    finally:
        L.mcr_text_destroy(h)
    return _chain(n, rs, col, val, initial, goals)


def _chain(n, rs, col, val, initial, goals):
    try:
        from mcreach.markov import GoalSet, MarkovChain
        return MarkovChain(n=n, transitions=_matrix_type()(n, rs, col, val), initial=initial), \
            GoalSet(goals.tolist())
    except ImportError:
        from .chains import Chain
        return Chain(n, CsrMatrix(n, rs, col, val), initial, goals), goals
