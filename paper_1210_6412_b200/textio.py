"""Line-by-line readers for the text files the multithreaded C++ readers do not take.

The fast readers in ``csrc/formats.cpp`` parse the well-formed plain-decimal files the
reference writes (``mcreach/formats.py``); anything else -- a malformed line, a duplicate, a
failed chain check, tokens only Python's ``int()`` / ``float()`` accept (``inf``, ``1_0``) --
comes here. This module restates the reference's reading rules (``S/formats.py:62-85`` tokens
and comments, ``:89-113`` matrix, ``:128-145`` vector, ``:160-232`` chain) and its checks
(``S/sparse.py:145-172`` assembly, ``S/markov.py:117-142`` ``validate``) so results and
errors are the reference's own: the same exception classes (the reference's when ``mcreach``
is importable, this package's mirrors otherwise), the same messages and line numbers. The
reference itself is never called.
"""

from __future__ import annotations

from typing import Optional

import numpy as np

from . import sparse as _sp

ROW_SUM_TOL = 1e-9  # S/markov.py:38-40


# ----------------------------------------------------------------------------- error classes

class ParseError(ValueError):
    """S/formats.py:51-56."""

    def __init__(self, message: str, line: Optional[int] = None):
        self.line = line
        super().__init__(f"line {line}: {message}" if line else message)


class MarkovChainError(ValueError):
    """S/markov.py:43-44."""


class RowSumError(MarkovChainError):
    """S/markov.py:47-53."""

    def __init__(self, state: int, total: float):
        super().__init__(f"row {state} sums to {total!r}, expected 1")
        self.state = state
        self.total = total


class ProbabilityOutOfRange(MarkovChainError):
    """S/markov.py:56-63."""

    def __init__(self, src: int, dst: int, value: float):
        super().__init__(f"transition {src} -> {dst} has probability {value!r}")
        self.src = src
        self.dst = dst
        self.value = value


def _ref(module: str):
    try:
        import importlib
        return importlib.import_module(module)
    except Exception:
        return None


def _cls(module: str, name: str, fallback):
    mod = _ref(module)
    return getattr(mod, name, fallback) if mod is not None else fallback


def parse_error(message: str, line: Optional[int] = None):
    return _cls("mcreach.formats", "ParseError", ParseError)(message, line)


def _sparse_error(err: Exception) -> Exception:
    """This package's assembly error as the reference's class (same message / fields)."""
    mod = _ref("mcreach.sparse")
    if mod is None:
        return err
    if isinstance(err, _sp.DuplicateEntry):
        return mod.DuplicateEntry(err.row, err.col)
    return getattr(mod, type(err).__name__, mod.SparseError)(str(err))


def _assemble(n: int, entries):
    try:
        return _sp.csr_from_triplets(n, entries)
    except _sp.SparseError as err:
        raise _sparse_error(err) from None


# ----------------------------------------------------------------------------- tokens

def _lines(path):
    """(1-based line number, tokens) of every significant line: '#' starts a comment that
    runs to the end of the line, blank lines are skipped, ASCII only (S/formats.py:62-68)."""
    with open(path, "r", encoding="ascii") as handle:
        for number, raw in enumerate(handle, start=1):
            text = raw.split("#", 1)[0].strip()
            if text:
                yield number, text.split()


def _int(token: str, line: int, what: str) -> int:
    try:
        return int(token)
    except ValueError:
        raise parse_error(f"expected an integer {what}, got {token!r}", line) from None


def _float(token: str, line: int, what: str) -> float:
    try:
        return float(token)
    except ValueError:
        raise parse_error(f"expected a number {what}, got {token!r}", line) from None


def _first(lines, what: str):
    try:
        return next(lines)
    except StopIteration:
        raise parse_error(f"empty {what} file") from None


# ----------------------------------------------------------------------------- readers

def read_matrix(path, matrix_type=_sp.CsrMatrix):
    """S/formats.py:89-113."""
    lines = _lines(path)
    number, tokens = _first(lines, "matrix")
    if len(tokens) != 3 or tokens[0] != "matrix":
        raise parse_error("expected header 'matrix <n> <m>'", number)
    n = _int(tokens[1], number, "dimension")
    m = _int(tokens[2], number, "entry count")
    entries = []
    for number, tokens in lines:
        if len(tokens) != 3:
            raise parse_error("expected '<row> <col> <value>'", number)
        entries.append((_int(tokens[0], number, "row index"), _int(tokens[1], number, "column index"),
                        _float(tokens[2], number, "value")))
    if len(entries) != m:
        raise parse_error(f"header promised {m} entries, file has {len(entries)}")
    a = _assemble(n, entries)
    return matrix_type(a.n, a.rstart, a.col, a.nonzero)


def read_vector(path) -> np.ndarray:
    """S/formats.py:128-145."""
    lines = _lines(path)
    number, tokens = _first(lines, "vector")
    if len(tokens) != 2 or tokens[0] != "vector":
        raise parse_error("expected header 'vector <n>'", number)
    n = _int(tokens[1], number, "length")
    values = []
    for number, tokens in lines:
        if len(tokens) != 1:
            raise parse_error("expected one value per line", number)
        values.append(_float(tokens[0], number, "value"))
    if len(values) != n:
        raise parse_error(f"header promised {n} values, file has {len(values)}")
    return np.array(values, dtype=np.float64)


def read_dtmc_parts(path):
    """S/formats.py:160-230 up to (not including) building the chain: returns
    (n, initial, goals, transitions CSR) after the reference's checks, ``validate`` included."""
    n = initial = goals = None
    transitions = []
    seen = {}
    lines = _lines(path)
    number, tokens = _first(lines, "chain")
    if tokens != ["dtmc"]:
        raise parse_error("expected 'dtmc' as the first line", number)
    for number, tokens in lines:
        key = tokens[0]
        if key == "states":
            if n is not None:
                raise parse_error("duplicate 'states' line", number)
            if len(tokens) != 2:
                raise parse_error("expected 'states <n>'", number)
            n = _int(tokens[1], number, "state count")
        elif key == "initial":
            if initial is not None:
                raise parse_error("duplicate 'initial' line", number)
            if len(tokens) != 2:
                raise parse_error("expected 'initial <s0>'", number)
            initial = _int(tokens[1], number, "initial state")
        elif key == "goal":
            if goals is not None:
                raise parse_error("duplicate 'goal' line", number)
            if len(tokens) < 2:
                raise parse_error("expected 'goal <g1> ...' with at least one state", number)
            goals = [_int(t, number, "goal state") for t in tokens[1:]]
        else:
            if len(tokens) != 3:
                raise parse_error("expected '<src> <dst> <prob>'", number)
            src = _int(tokens[0], number, "source state")
            dst = _int(tokens[1], number, "target state")
            prob = _float(tokens[2], number, "probability")
            if (src, dst) in seen:
                raise parse_error(f"duplicate transition {src} -> {dst} "
                                  f"(first on line {seen[(src, dst)]})", number)
            seen[(src, dst)] = number
            transitions.append((src, dst, prob))
    if n is None:
        raise parse_error("missing 'states' line")
    if initial is None:
        raise parse_error("missing 'initial' line")
    if goals is None:
        raise parse_error("missing 'goal' line")
    for s in goals:
        if not 0 <= s < n:
            raise parse_error(f"goal state {s} outside 0..{n - 1}")
    for src, dst, _ in transitions:
        if not 0 <= src < n or not 0 <= dst < n:
            raise parse_error(f"transition {src} -> {dst} outside 0..{n - 1} "
                              f"(line {seen[(src, dst)]})")
    p = _assemble(n, transitions)
    validate(n, p, initial)
    if not goals:
        raise _cls("mcreach.markov", "MarkovChainError", MarkovChainError)("goal set must not be empty")
    return n, initial, goals, p


# ----------------------------------------------------------------------------- chain checks

def row_sums(p) -> np.ndarray:
    """Every row of the CSR summed in ascending column order from 0.0 (matvec with a vector of
    ones, S/sparse.py:184-191 -> scipy csr_matvec): one vectorised add per column position."""
    n = int(p.n)
    rs = np.asarray(p.rstart, dtype=np.int64)
    vals = np.asarray(p.nonzero, dtype=np.float64)
    lens = np.diff(rs)
    acc = np.zeros(n)
    for j in range(int(lens.max()) if n else 0):
        live = np.flatnonzero(lens > j)
        acc[live] = acc[live] + vals[rs[live] + j]
    return acc


def validate(n: int, p, initial: int) -> None:
    """S/markov.py:117-142 on the transition CSR of an n-state chain."""
    err = _cls("mcreach.markov", "MarkovChainError", MarkovChainError)
    if p.n != n:
        raise err(f"matrix dimension {p.n} does not match state count {n}")
    if n < 1:
        raise err("a chain needs at least one state")
    if not 0 <= initial < n:
        raise err(f"initial state {initial} out of range")
    vals = np.asarray(p.nonzero, dtype=np.float64)
    bad = np.flatnonzero((vals <= 0.0) | (vals > 1.0))
    if bad.size:
        k = int(bad[0])
        src = int(np.searchsorted(p.rstart, k, side="right") - 1)
        raise _cls("mcreach.markov", "ProbabilityOutOfRange", ProbabilityOutOfRange)(
            src, int(p.col[k]), float(vals[k]))
    sums = row_sums(p)
    off = np.flatnonzero(np.abs(sums - 1.0) > ROW_SUM_TOL)
    if off.size:
        s = int(off[0])
        raise _cls("mcreach.markov", "RowSumError", RowSumError)(s, float(sums[s]))
