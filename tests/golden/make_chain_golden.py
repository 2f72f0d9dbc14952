"""Golden fixtures for the chain -> system build (markov.py:152-256), made by running the
UNMODIFIED reference here:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_chain_golden.py

For every case it records the chain (CSR arrays for the small ones, the random_dtmc spec for
the large ones), the goal states, and the reference's outputs: the state classes (0 = prob
zero, 1 = prob one, 2 = uncertain), the reduced matrix M = I - A (rstart / col / nonzero)
and the right-hand side, as arrays (small) or SHA-256 hashes (large), plus the reachability
vector from jacobi-seq for the small cases. Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

sys.dont_write_bytecode = True
REF = os.environ.get("MCREACH_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, "/root/reference/pkg/tests")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from mcreach.markov import GoalSet, MarkovChain, build_system, reachability_probabilities  # noqa: E402
from mcreach.solvers import SolverError  # noqa: E402
from mcreach.sparse import CsrMatrix as RefCsr  # noqa: E402
from oracles import random_chain, random_goals  # noqa: E402

from paper_1210_6412_b200.chains import random_dtmc  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def classes(part, n):
    c = np.full(n, 2, dtype=np.int8)
    c[sorted(part.prob_zero)] = 0
    c[sorted(part.prob_one)] = 1
    return c


def main():
    cases, arrays = {}, {}

    def record(name, chain, goals, spec=None, keep_arrays=True, solve=True):
        t0 = time.perf_counter()
        sysm = build_system(chain, GoalSet(goals))
        dt = time.perf_counter() - t0
        p = chain.transitions
        c = classes(sysm.partition, chain.n)
        M = sysm.matrix
        case = {"n": int(chain.n), "goals": [int(g) for g in goals], "spec": spec,
                "k": int(M.n), "m_nnz": int(M.m), "ref_build_seconds": dt,
                "chain_rstart_sha256": sha(p.rstart), "chain_col_sha256": sha(p.col),
                "chain_nonzero_sha256": sha(p.nonzero),
                "classes_sha256": sha(c), "uncertain_sha256": sha(sysm.partition.uncertain),
                "m_rstart_sha256": sha(M.rstart), "m_col_sha256": sha(M.col),
                "m_nonzero_sha256": sha(M.nonzero), "rhs_sha256": sha(sysm.rhs)}
        if keep_arrays:
            for key, a in (("rstart", p.rstart), ("col", p.col), ("nonzero", p.nonzero),
                           ("classes", c), ("m_rstart", M.rstart), ("m_col", M.col),
                           ("m_nonzero", M.nonzero), ("rhs", sysm.rhs)):
                arrays[f"{name}/{key}"] = np.asarray(a)
        if solve:
            for method in ("jacobi-seq", "bicgstab-seq"):
                try:
                    x, rep = reachability_probabilities(chain, GoalSet(goals), method)
                except SolverError as err:  # recorded: the GPU path must raise the same
                    case[method] = {"outcome": type(err).__name__,
                                    "iterations": int(getattr(err, "iteration", 0) or
                                                      err.result.iterations)}
                    continue
                case[method] = {"outcome": "ok", "iterations": int(rep.iterations),
                                "x_sha256": sha(x)}
                if keep_arrays:
                    arrays[f"{name}/{method}/x"] = x
        cases[name] = case
        print(name, chain.n, M.n, M.m, f"{dt:.2f}s", flush=True)

    # the 4-state chain of the paper (T/conftest.py:6-17) with several goal sets
    demo = RefCsr(4, np.array([0, 2, 3, 5, 6]), np.array([2, 3, 1, 0, 1, 3]),
                  np.array([0.5, 0.5, 1.0, 0.4, 0.6, 1.0]))
    dchain = MarkovChain(4, demo, 0)
    for tag, goals in (("demo_g3", [3]), ("demo_g1", [1]), ("demo_g0", [0]),
                       ("demo_all", [0, 1, 2, 3])):
        record(tag, dchain, goals)
    # the reference's random valid chains (T/oracles.py:102-121)
    rng = np.random.default_rng(20240)
    for i in range(40):
        n = int(rng.integers(2, 31))
        ch = random_chain(rng, n)
        goals = sorted(random_goals(rng, n).members)
        record(f"oracle_chain_{i}", ch, goals)
    # seeded random DTMCs (paper_1210_6412_b200/chains.py), C2'-shaped
    for n, seed, keep in ((1000, 1, True), (20000, 2, False), (100000, 3, False),
                          (1000000, 4, False)):
        d = random_dtmc(n, seed)
        ch = MarkovChain(n, RefCsr(n, d.transitions.rstart, d.transitions.col,
                                   d.transitions.nonzero), d.initial)
        record(f"dtmc_{n}", ch, d.goals.tolist(), spec={"n": n, "seed": seed},
               keep_arrays=keep, solve=n <= 20000)
    with open(os.path.join(HERE, "chain_golden.json"), "w") as fh:
        json.dump({"cases": cases}, fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "chain_golden.npz"), **arrays)


if __name__ == "__main__":
    main()
