"""Host-side CSR container accepted by the GPU solvers.

Mirrors ``mcreach.sparse.CsrMatrix`` (``/root/reference/pkg/src/mcreach/sparse.py:71-98``):
an immutable square matrix with ``rstart`` (int64, n+1), ``col`` (int64) and ``nonzero``
(float64), rows sorted by column, no duplicates, no explicit zeros. The solvers accept this
class, the reference's own ``CsrMatrix``, or any object with the same four attributes.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable

import numpy as np

__all__ = ["CsrMatrix", "csr_from_triplets", "SparseError", "DimensionMismatch",
           "DuplicateEntry", "IndexOutOfRange"]


class SparseError(ValueError):
    """sparse.py:38-39"""


class DuplicateEntry(SparseError):
    def __init__(self, row: int, col: int):
        super().__init__(f"duplicate entry at ({row}, {col})")
        self.row = row
        self.col = col


class IndexOutOfRange(SparseError):
    pass


class DimensionMismatch(SparseError):
    """sparse.py:55-56"""


@dataclass(frozen=True, eq=False)
class CsrMatrix:
    n: int
    rstart: np.ndarray
    col: np.ndarray
    nonzero: np.ndarray

    @property
    def m(self) -> int:
        return int(self.rstart[-1])


def csr_from_triplets(n: int, entries: Iterable[tuple]) -> CsrMatrix:
    """sparse.py:145-172: zeros dropped, rows sorted by column, duplicates rejected."""
    if n < 0:
        raise IndexOutOfRange(f"dimension must be nonnegative, got {n}")
    ent = [(int(e[0]), int(e[1]), float(e[2])) for e in entries]
    rows = np.array([e[0] for e in ent], dtype=np.int64)
    cols = np.array([e[1] for e in ent], dtype=np.int64)
    vals = np.array([e[2] for e in ent], dtype=np.float64)
    if len(ent):
        bad = (rows < 0) | (rows >= n) | (cols < 0) | (cols >= n)
        if np.any(bad):
            k = int(np.flatnonzero(bad)[0])
            raise IndexOutOfRange(f"entry ({rows[k]}, {cols[k]}) outside dimension {n}")
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if len(ent) > 1:
        dup = (rows[1:] == rows[:-1]) & (cols[1:] == cols[:-1])
        if np.any(dup):
            k = int(np.flatnonzero(dup)[0]) + 1
            raise DuplicateEntry(int(rows[k]), int(cols[k]))
    keep = vals != 0.0
    rows, cols, vals = rows[keep], cols[keep], vals[keep]
    rstart = np.zeros(n + 1, dtype=np.int64)
    if n:
        np.cumsum(np.bincount(rows, minlength=n), out=rstart[1:])
    return CsrMatrix(n, rstart, cols, vals)
