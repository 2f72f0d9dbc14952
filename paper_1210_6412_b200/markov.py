"""Reachability probabilities of a Markov chain on the GPU -- the caller side of the solve.

Mirrors ``mcreach/markov.py`` (``/root/reference/pkg/src/mcreach/markov.py``):

* ``build_system(chain, goals)`` (:237-256): partition by two backward closures
  (``partition_states`` :184-214), uncertain states in ascending order, ``M = I - A`` over them
  (``identity_minus``, sparse.py:208-224) and the one-step goal probabilities -- all built on
  the device (``mcr_chain_create``, csrc/chain.cuh) and bit-identical to the reference;
* ``reachability_probabilities(chain, goals, method, config)`` (:259-293): the same, then the
  solve on the device-resident ``M`` and the full vector (certain states exact, solved states
  clipped to [0, 1]) -- no host round trip between building and solving.

``chain`` is any object with ``n`` and a CSR ``transitions`` (``rstart``, ``col``,
``nonzero``), e.g. ``mcreach.MarkovChain``; ``goals`` a ``GoalSet`` (``members``) or an
iterable of states. Results and errors are the reference's types when ``mcreach`` is
importable (``LinearSystem``, ``StatePartition``, ``MarkovChainError``), else mirrors.
"""

from __future__ import annotations

import ctypes
import time
import weakref
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .solvers import SolverConfig, SolveResult, _raise_native, outcome
from .sparse import CsrMatrix

__all__ = ["ChainSystem", "build_system", "partition_states", "reachability_probabilities",
           "METHODS", "MarkovChainError"]

# method name -> (mcr_chain_solve method, reference-order dots: None = the config's
# dot_products, "sequential" by default, as the solvers of solvers.py)
METHODS = {"jacobi-gpu": (0, 0), "bicgstab-gpu": (1, None), "bicgstab-gpu-exact": (1, 1)}


def _reference():
    try:
        import mcreach.markov as mm
        return mm
    except Exception:
        return None


class MarkovChainError(ValueError):
    """markov.py:32-33 (the reference's class is raised when mcreach is importable)."""


def _chain_error(msg: str):
    mm = _reference()
    return mm.MarkovChainError(msg) if mm is not None else MarkovChainError(msg)


def _goal_list(chain, goals) -> np.ndarray:
    members = getattr(goals, "members", goals)
    g = np.array(sorted(int(s) for s in members), dtype=np.int64)
    if g.size == 0:
        raise _chain_error("goal set must not be empty")
    if g[0] < 0 or g[-1] >= chain.n:  # _check_goals, markov.py:145-149
        raise _chain_error(f"goal states {g.tolist()} must lie below {chain.n}")
    return g


@dataclass(frozen=True, eq=False)
class _Partition:
    prob_one: frozenset
    prob_zero: frozenset
    uncertain: np.ndarray
    index_of: dict


@dataclass(frozen=True, eq=False)
class _LinearSystem:
    matrix: CsrMatrix
    rhs: np.ndarray
    partition: _Partition


class ChainSystem:
    """A chain + goal set with its reduced system resident on the device."""

    def __init__(self, chain, goals, device: int = 0):
        L = _lib.load()
        self._L = L
        self.n = int(chain.n)
        self.goals = _goal_list(chain, goals)
        p = chain.transitions
        rs = np.ascontiguousarray(p.rstart, dtype=np.int64)
        col = np.ascontiguousarray(p.col, dtype=np.int64)
        val = np.ascontiguousarray(p.nonzero, dtype=np.float64)
        if int(getattr(p, "n", self.n)) != self.n:
            raise _chain_error(f"matrix dimension {p.n} does not match state count {self.n}")
        h = ctypes.c_void_p()
        rc = L.mcr_chain_create(self.n, rs.ctypes.data, col.ctypes.data, val.ctypes.data,
                                self.goals.ctypes.data, len(self.goals), int(device),
                                ctypes.byref(h))
        if rc != _lib.MCR_OK:
            _raise_native(rc)
        self._h = h
        self._finalizer = weakref.finalize(self, L.mcr_chain_destroy, h)
        k, one, zero, m = (ctypes.c_int64() for _ in range(4))
        L.mcr_chain_info(h, ctypes.byref(k), ctypes.byref(one), ctypes.byref(zero), ctypes.byref(m))
        self.k, self.n_one, self.n_zero, self.m_nnz = k.value, one.value, zero.value, m.value

    def close(self):
        self._finalizer()

    def export(self):
        """(classes int8[n], uncertain int64[k], M as CsrMatrix, rhs[k]) as host arrays."""
        cls = np.empty(self.n, dtype=np.int8)
        unc = np.empty(self.k, dtype=np.int64)
        mrs = np.empty(self.k + 1, dtype=np.int64)
        mcol = np.empty(self.m_nnz, dtype=np.int64)
        mval = np.empty(self.m_nnz, dtype=np.float64)
        rhs = np.empty(self.k, dtype=np.float64)
        rc = self._L.mcr_chain_export(self._h, cls.ctypes.data, unc.ctypes.data, mrs.ctypes.data,
                                      mcol.ctypes.data, mval.ctypes.data, rhs.ctypes.data)
        if rc != _lib.MCR_OK:
            _raise_native(rc)
        return cls, unc, CsrMatrix(self.k, mrs, mcol, mval), rhs

    def solve(self, method: str = "jacobi-gpu", config: Optional[SolverConfig] = None):
        """reachability_probabilities on the device: returns (x[n], SolveResult of M x = rhs)."""
        try:
            code, dots = METHODS[method]
        except KeyError:
            raise ValueError(f"unknown method {method!r}, expected one of {sorted(METHODS)}") from None
        cfg = config or SolverConfig()
        if dots is None:
            dots = 0 if getattr(cfg, "dot_products", "sequential") == "tree" else 1
        x0 = None
        seed = getattr(cfg, "guess_seed", None)
        if seed is not None and self.k:  # solvers.py:153-156 on the reduced system
            x0 = np.ascontiguousarray(np.random.default_rng(seed).random(self.k))
        x = np.empty(self.n)
        xs = np.empty(self.k)
        rep = _lib.Report()
        start = time.perf_counter()
        rc = self._L.mcr_chain_solve(self._h, code, dots, float(cfg.tolerance),
                                     int(cfg.max_iterations),
                                     None if x0 is None else x0.ctypes.data, x.ctypes.data,
                                     xs.ctypes.data, ctypes.byref(rep))
        if self.k == 0:  # markov.py:287-288
            return x, SolveResult(np.zeros(0), 0, True, 0.0, 0.0)
        result, err = outcome(rc, xs, rep, start)
        if err is not None:
            raise err
        return x, result


def _partition(cls: np.ndarray, unc: np.ndarray):
    mm = _reference()
    kind = mm.StatePartition if mm is not None else _Partition
    return kind(prob_one=frozenset(np.flatnonzero(cls == 1).tolist()),
                prob_zero=frozenset(np.flatnonzero(cls == 0).tolist()),
                uncertain=unc, index_of={int(s): i for i, s in enumerate(unc)})


def partition_states(chain, goals, device: int = 0):
    """markov.py:184-214 on the device: the StatePartition (prob one / prob zero / uncertain
    ascending, index_of) -- the reference's type when mcreach is importable."""
    cs = ChainSystem(chain, goals, device)
    try:
        cls = np.empty(cs.n, dtype=np.int8)
        unc = np.empty(cs.k, dtype=np.int64)
        rc = cs._L.mcr_chain_export(cs._h, cls.ctypes.data, unc.ctypes.data, None, None, None, None)
        if rc != _lib.MCR_OK:
            _raise_native(rc)
    finally:
        cs.close()
    return _partition(cls, unc)


def build_system(chain, goals, device: int = 0):
    """markov.py:237-256, built on the device; returns the reference's LinearSystem type when
    mcreach is importable (matrix as its CsrMatrix), else a mirror."""
    cs = ChainSystem(chain, goals, device)
    try:
        cls, unc, M, rhs = cs.export()
    finally:
        cs.close()
    part = _partition(cls, unc)
    mm = _reference()
    if mm is not None:
        from mcreach.sparse import CsrMatrix as RefCsr
        return mm.LinearSystem(RefCsr(M.n, M.rstart, M.col, M.nonzero), rhs, part)
    return _LinearSystem(M, rhs, part)


def reachability_probabilities(chain, goals, method: str = "jacobi-gpu",
                               config: Optional[SolverConfig] = None, device: int = 0):
    """markov.py:259-293 on the device: (x[n], SolveResult of the reduced system)."""
    if method not in METHODS:
        raise ValueError(f"unknown method {method!r}, expected one of {sorted(METHODS)}")
    cs = ChainSystem(chain, goals, device)
    try:
        return cs.solve(method, config)
    finally:
        cs.close()
