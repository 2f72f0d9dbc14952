"""Generate the golden fixtures by running the UNMODIFIED reference (`mcreach`) here.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--skip-c2]

The reference is imported from /root/reference/pkg/src (read-only; bytecode writing is
disabled). Every case records the reference's inputs (explicit CSR arrays for the small
known-answer systems, GenSpec + SHA-256 of the generated arrays for the seeded systems) and
its outputs for `jacobi-seq` and `bicgstab-seq`: outcome (ok / NotConverged / Breakdown /
ZeroDiagonal), iterations, residual_inf (float.hex, exact) and x (full vector, or SHA-256 +
a strided sample for n = 1e6). These files are what pins the CPU oracle (oracle/) and the
bit-exact input generator (paper_1210_6412_b200/generator.py) to the reference; the GPU
parity tests compare against the same files. Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

sys.dont_write_bytecode = True
REF = os.environ.get("MCREACH_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, "/root/reference/pkg/tests")

import numpy as np  # noqa: E402

import mcreach  # noqa: E402
from mcreach import (Breakdown, GenSpec, GoalSet, NotConverged, SolverConfig,  # noqa: E402
                     ZeroDiagonal, build_system, csr_from_triplets, generate_dd_matrix,
                     generate_rhs)
from mcreach.bench import trial_seed  # noqa: E402
from mcreach.generator import TABLE1_SHAPES  # noqa: E402
from mcreach.solvers import SOLVERS  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SAMPLE_STRIDE = 997


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run(method, m, b, cfg):
    begin = time.perf_counter()
    out = {}
    try:
        res = SOLVERS[method](m, b, cfg)
        out["outcome"] = "ok"
    except NotConverged as err:
        res = err.result
        out["outcome"] = "not_converged"
    except Breakdown as err:
        res = err.result
        out["outcome"] = "breakdown"
        out["which"] = err.which
        out["breakdown_iteration"] = err.iteration
    except ZeroDiagonal as err:
        out["outcome"] = "zero_diagonal"
        out["zero_index"] = err.index
        return out, None
    out["iterations"] = int(res.iterations)
    out["converged"] = bool(res.converged)
    out["residual_inf"] = float(res.residual_inf).hex()
    out["x_sha256"] = sha(res.x)
    out["ref_seconds"] = time.perf_counter() - begin
    return out, np.asarray(res.x, dtype=np.float64)


def cfg_dict(cfg: SolverConfig):
    return {"tolerance": cfg.tolerance, "max_iterations": cfg.max_iterations,
            "guess_seed": cfg.guess_seed}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c2", action="store_true")
    args = ap.parse_args()

    cases = {}
    arrays = {}

    def add(name, m, b, cfg=None, spec=None, methods=("jacobi-seq", "bicgstab-seq"),
            full_x=True, store_matrix=False, cfgs=None):
        cfg = cfg or SolverConfig()
        case = {"n": int(m.n), "m": int(m.m), "b_sha256": sha(np.asarray(b, np.float64)),
                "rstart_sha256": sha(m.rstart), "col_sha256": sha(m.col),
                "nonzero_sha256": sha(m.nonzero), "config": cfg_dict(cfg), "results": {}}
        if spec is not None:
            case["spec"] = spec
        if store_matrix:
            arrays[f"{name}/rstart"] = np.asarray(m.rstart, np.int64)
            arrays[f"{name}/col"] = np.asarray(m.col, np.int64)
            arrays[f"{name}/nonzero"] = np.asarray(m.nonzero, np.float64)
            arrays[f"{name}/b"] = np.asarray(b, np.float64)
        for method in methods:
            c = (cfgs or {}).get(method, cfg)
            out, x = run(method, m, b, c)
            out["config"] = cfg_dict(c)
            key = method.split("-")[0]
            if x is not None:
                if full_x:
                    arrays[f"{name}/{key}/x"] = x
                else:
                    arrays[f"{name}/{key}/x_sample"] = x[::SAMPLE_STRIDE].copy()
                    out["x_inf_norm"] = float(np.max(np.abs(x))).hex()
            case["results"][key] = out
        cases[name] = case
        print(f"{name}: " + ", ".join(
            f"{k}={v.get('outcome')}/{v.get('iterations')}" for k, v in case["results"].items()),
            flush=True)

    # ---- known-answer systems (tests/test_solvers.py) ----
    golden = csr_from_triplets(2, [(0, 0, 1.0), (0, 1, -0.5), (1, 0, -0.4), (1, 1, 1.0)])
    add("kat_golden2x2", golden, np.array([0.5, 0.0]), store_matrix=True)
    eye4 = csr_from_triplets(4, [(i, i, 1.0) for i in range(4)])
    add("kat_identity4", eye4, np.array([3.0, -1.5, 2.25, 0.5]), store_matrix=True)
    zd = csr_from_triplets(2, [(0, 1, -0.5), (1, 0, -0.4), (1, 1, 1.0)])
    add("kat_zero_diagonal", zd, np.array([0.5, 0.0]), store_matrix=True)
    div = csr_from_triplets(2, [(0, 0, 1.0), (0, 1, -2.0), (1, 0, -2.0), (1, 1, 1.0)])
    add("kat_divergent", div, np.array([1.0, 1.0]), SolverConfig(max_iterations=40),
        store_matrix=True)
    skew = csr_from_triplets(2, [(0, 1, 1.0), (1, 0, -1.0)])
    add("kat_breakdown_qv", skew, np.array([1.0, 1.0]), store_matrix=True,
        methods=("bicgstab-seq", "jacobi-seq"))
    sing = csr_from_triplets(2, [(0, 0, 1.0), (0, 1, -1.0), (1, 0, 2.0), (1, 1, -2.0)])
    add("kat_breakdown_tt", sing, np.array([1.0, -1.0]), store_matrix=True,
        cfg=SolverConfig(max_iterations=50))
    add("kat_singular_consistent", sing, np.array([1.0, 2.0]), store_matrix=True,
        cfg=SolverConfig(max_iterations=50))
    add("kat_tiny_budget", golden, np.array([0.5, 0.0]), SolverConfig(max_iterations=1),
        store_matrix=True)
    add("kat_zero_rhs", golden, np.zeros(2), store_matrix=True)

    # ---- chain systems: I - A with negative off-diagonals (markov.py:237-256) ----
    demo = mcreach.MarkovChain(n=4, transitions=csr_from_triplets(4, [
        (0, 2, 0.5), (0, 3, 0.5), (1, 1, 1.0), (2, 0, 0.4), (2, 1, 0.6), (3, 3, 1.0)]), initial=0)
    sysd = build_system(demo, GoalSet([3]))
    add("chain_demo", sysd.matrix, sysd.rhs, store_matrix=True)
    # random DTMCs in the C2' shape: absorbing goals and traps, a few
    # successors per transient state with U{1..10} weights normalised to probabilities
    rng = np.random.default_rng(4242)
    for k, n in enumerate((60, 400, 3000)):
        n_goal = max(1, n // 100)
        n_trap = max(1, n // 100)
        entries = []
        for s in range(n):
            if s < n_goal + n_trap:
                entries.append((s, s, 1.0))
                continue
            deg = int(rng.integers(1, 6))
            tgt = rng.choice(n, size=deg, replace=False)
            w = rng.integers(1, 10, size=deg, endpoint=True).astype(float)
            for t, wt in zip(tgt, w):
                entries.append((s, int(t), float(wt) / float(w.sum())))
        ch = mcreach.MarkovChain(n=n, transitions=csr_from_triplets(n, entries), initial=n - 1)
        s = build_system(ch, GoalSet(range(n_goal)))
        add(f"chain_random{k}", s.matrix, s.rhs, store_matrix=True)

    # ---- seeded generated systems ----
    def dom(name, n, nnz=None, density=None, seed=0, cfg=None, **kw):
        spec = {"n": n, "nnz": nnz, "density": density, "seed": int(seed)}
        m = generate_dd_matrix(GenSpec(n=n, nnz=nnz, density=density, seed=seed))
        b = generate_rhs(n, seed)
        add(name, m, b, cfg=cfg, spec=spec, **kw)

    sizes = (5, 10, 15, 20, 25, 30, 35, 40, 45, 50)
    dens = (0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0)
    for i, n in enumerate(sizes):           # T/test_solvers.py:52-58
        for j, d in enumerate(dens):
            dom(f"grid_{n}_{j}", n, nnz=max(n, round(d * n * n)), seed=1000 + 10 * i + j)
    dom("seeded_guess", 80, nnz=800, seed=21, cfg=SolverConfig(guess_seed=1234))
    dom("parallel_large", 1000, nnz=12000, seed=5)
    ns = np.linspace(50, 2000, 20).astype(int)  # T/test_acceptance.py:114-129
    for idx, n in enumerate(ns[::4]):
        dom(f"crit3_{int(n)}", int(n), nnz=int(min(n * n, 8 * n)), seed=31000 + 4 * idx)
    for s in range(2):                          # T/test_acceptance.py:132-140
        dom(f"crit4_{s}", 1000, nnz=round(0.10 * 1000 * 1000), seed=41000 + s)
    for n, m in TABLE1_SHAPES:                  # C4
        dom(f"c4_{n}_{m}", n, nnz=m, seed=trial_seed(0, n, None, m, 0))
    dom("c1_seed77", 2000, density=0.1, seed=77)  # C1 (T/test_solvers.py:251)
    dom("c1_trial0", 2000, density=0.1, seed=trial_seed(0, 2000, 0.1, None, 0))
    dom("dense_1024", 1024, density=1.0, seed=3,
        cfgs={"jacobi-seq": SolverConfig(max_iterations=300), "bicgstab-seq": SolverConfig()})
    if not args.skip_c2:
        n, nnz = 10 ** 6, 10 ** 7
        dom("c2_trial0", n, nnz=nnz, seed=trial_seed(0, n, None, nnz, 0), full_x=False)

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump({"reference": "mcreach " + mcreach.__version__,
                   "numpy": np.__version__, "sample_stride": SAMPLE_STRIDE,
                   "cases": cases}, fh, indent=1, sort_keys=True)
    print("wrote", len(cases), "cases")


if __name__ == "__main__":
    main()
