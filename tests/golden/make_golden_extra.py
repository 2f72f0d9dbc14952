"""Extra golden fixtures from the UNMODIFIED reference (`mcreach`), run here:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_extra.py [--skip-c3]

* parallel_dot_products (solvers.py:98, 384-396): bicgstab_solve_parallel with the per-block
  dot mode at workers 2 / 4 / 16 on golden systems of tests/golden/golden.json: iterations,
  outcome, residual (float.hex) and x.
* C3: GenSpec(n=16384, density=1.0, seed=3) + generate_rhs(16384, 3) (the bench's
  C3 system; complete structure via the shortcut in generator.py:85-86): BiCGStab in full and
  Jacobi capped at 50 sweeps (NotConverged, the capped iterate), x as SHA-256 + a strided
  sample, residual as float.hex. (~3 min, ~40 GB of host memory for the reference.)

Outputs: golden_extra.json / golden_extra.npz next to this file.
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
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from mcreach import (Breakdown, GenSpec, NotConverged, SolverConfig,  # noqa: E402
                     generate_dd_matrix, generate_rhs)
from mcreach.solvers import bicgstab_solve_parallel, bicgstab_solve, jacobi_solve  # noqa: E402

SAMPLE_STRIDE = 997


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run(fn, m, b, cfg):
    out = {}
    try:
        res = fn(m, b, cfg)
        out["outcome"] = "ok"
    except NotConverged as err:
        res = err.result
        out["outcome"] = "not_converged"
    except Breakdown as err:
        res = err.result
        out["outcome"] = "breakdown"
        out["which"] = err.which
        out["breakdown_iteration"] = err.iteration
    out["iterations"] = int(res.iterations)
    out["residual_inf"] = float(res.residual_inf).hex()
    out["x_sha256"] = sha(res.x)
    return out, np.asarray(res.x, np.float64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c3", action="store_true")
    args = ap.parse_args()
    from golden_cases import system  # the base fixtures' systems (SHA-checked)
    cases, arrays = {}, {}
    for name in ("grid_50_5", "crit3_460", "c1_seed77", "c4_2000_3999", "chain_random2",
                 "c4_5647_11293", "parallel_large"):
        from mcreach.sparse import CsrMatrix
        mm, b = system(name)
        m = CsrMatrix(mm.n, mm.rstart, mm.col, mm.nonzero)
        for w in (2, 4, 16):
            cfg = SolverConfig(workers=w, parallel_dot_products=True)
            t = time.perf_counter()
            out, x = run(bicgstab_solve_parallel, m, b, cfg)
            out["workers"] = w
            out["ref_seconds"] = time.perf_counter() - t
            key = f"pardots/{name}/w{w}"
            cases[key] = out
            arrays[key + "/x"] = x
            print(key, out["outcome"], out["iterations"], flush=True)
    if not args.skip_c3:
        n, seed = 16384, 3
        t = time.perf_counter()
        m = generate_dd_matrix(GenSpec(n=n, density=1.0, seed=seed))
        b = generate_rhs(n, seed)
        print(f"C3 generated in {time.perf_counter() - t:.1f}s", flush=True)
        c3 = {"n": n, "m": int(m.m), "seed": seed, "b_sha256": sha(b), "rstart_sha256": sha(m.rstart),
              "col_sha256": sha(m.col), "nonzero_sha256": sha(m.nonzero), "results": {}}
        for method, fn, cfg in (("bicgstab", bicgstab_solve, SolverConfig()),
                                ("jacobi", jacobi_solve, SolverConfig(max_iterations=50))):
            t = time.perf_counter()
            out, x = run(fn, m, b, cfg)
            out["max_iterations"] = cfg.max_iterations
            out["ref_seconds"] = time.perf_counter() - t
            out["x_inf_norm"] = float(np.max(np.abs(x))).hex()
            arrays[f"c3/{method}/x_sample"] = x[::SAMPLE_STRIDE].copy()
            c3["results"][method] = out
            print("C3", method, out["outcome"], out["iterations"], f"{out['ref_seconds']:.1f}s", flush=True)
        cases["c3"] = c3
    with open(os.path.join(HERE, "golden_extra.json"), "w") as fh:
        json.dump({"sample_stride": SAMPLE_STRIDE, "cases": cases}, fh, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden_extra.npz"), **arrays)


if __name__ == "__main__":
    main()
