"""Seeded random Markov chains (input construction for the chain-shaped workload C2').

SURVEY.md 8d row C2': a random DTMC with a fraction of absorbing goal states, a fraction of
absorbing traps and ~10 successors per transient state with U{1..10} weights normalised per
row; ``build_system`` (``mcreach/markov.py:237-256``) turns it into the reduced system
``(I - A) x = b`` over the uncertain states. Vectorised numpy, deterministic in the seed; the
reference's own random chains (``T/oracles.py:102-116``) are used for the small parity cases.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .sparse import CsrMatrix

__all__ = ["Chain", "random_dtmc"]


@dataclass(frozen=True, eq=False)
class Chain:
    """Mirror of ``mcreach.markov.MarkovChain`` (n, transitions CSR, initial) + goal states."""

    n: int
    transitions: CsrMatrix
    initial: int
    goals: np.ndarray


def random_dtmc(n: int, seed: int, successors=(5, 15), goal_frac: float = 0.01,
                trap_frac: float = 0.01) -> Chain:
    """Transient rows get U{successors} distinct targets (self-loops allowed) with
    probabilities w / sum(w), w ~ U{1..10}; goal and trap states are absorbing."""
    rng = np.random.default_rng(seed)
    kind = rng.random(n)
    goal = kind < goal_frac
    trap = (kind >= goal_frac) & (kind < goal_frac + trap_frac)
    if not goal.any():
        goal[int(rng.integers(0, n))] = True
    absorbing = goal | trap
    lo, hi = successors
    k = rng.integers(lo, hi + 1, size=n)
    k = np.minimum(k, n)
    k[absorbing] = 1
    rows = np.repeat(np.arange(n, dtype=np.int64), k)
    cols = rng.integers(0, n, size=len(rows))
    cols[np.repeat(absorbing, k)] = rows[np.repeat(absorbing, k)]   # self-loop, p = 1
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    keep = np.ones(len(rows), dtype=bool)
    keep[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])   # drop repeated targets
    rows, cols = rows[keep], cols[keep]
    w = rng.integers(1, 11, size=len(rows)).astype(np.float64)
    w[absorbing[rows]] = 1.0
    rstart = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rstart[1:])
    totals = np.add.reduceat(w, rstart[:-1]) if len(w) else np.zeros(0)
    p = w / np.repeat(totals, np.diff(rstart))
    return Chain(n, CsrMatrix(n, rstart, cols, p), int(rng.integers(0, n)),
                 np.flatnonzero(goal).astype(np.int64))
