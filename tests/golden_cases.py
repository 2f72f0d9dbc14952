"""Loader for the reference golden fixtures (tests/golden/, made by make_golden.py)."""

from __future__ import annotations

import functools
import hashlib
import json
import os

import numpy as np

from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix, generate_rhs
from paper_1210_6412_b200.sparse import CsrMatrix

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=1)
def manifest() -> dict:
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        return json.load(fh)


@functools.lru_cache(maxsize=1)
def arrays():
    return dict(np.load(os.path.join(GOLDEN, "golden.npz")))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def case_names(max_n=None, min_n=None):
    out = []
    for name, c in manifest()["cases"].items():
        if max_n is not None and c["n"] > max_n:
            continue
        if min_n is not None and c["n"] < min_n:
            continue
        out.append(name)
    return out


@functools.lru_cache(maxsize=8)
def _system_cached(name):
    return system(name, check=True)


def system(name, check=True):
    """(CsrMatrix, b) for a case: stored arrays, or regenerated from the GenSpec."""
    c = manifest()["cases"][name]
    a = arrays()
    if f"{name}/rstart" in a:
        m = CsrMatrix(c["n"], a[f"{name}/rstart"], a[f"{name}/col"], a[f"{name}/nonzero"])
        b = a[f"{name}/b"]
    else:
        s = c["spec"]
        m = generate_dd_matrix(GenSpec(n=s["n"], nnz=s["nnz"], density=s["density"],
                                       seed=s["seed"]))
        b = generate_rhs(s["n"], s["seed"])
    if check:
        assert sha(m.rstart) == c["rstart_sha256"], name
        assert sha(m.col) == c["col_sha256"], name
        assert sha(m.nonzero) == c["nonzero_sha256"], name
        assert sha(b) == c["b_sha256"], name
    return m, b


def expected(name, method):
    """Reference result dict for method 'jacobi' / 'bicgstab' plus its x (or x sample)."""
    r = dict(manifest()["cases"][name]["results"][method])
    a = arrays()
    r["x"] = a.get(f"{name}/{method}/x")
    r["x_sample"] = a.get(f"{name}/{method}/x_sample")
    return r
