"""Loader for the chain -> system golden fixtures (tests/golden/chain_golden.*, made by
tests/golden/make_chain_golden.py from the unmodified reference)."""

from __future__ import annotations

import functools
import json
import os

import numpy as np

from golden_cases import sha
from paper_1210_6412_b200.chains import random_dtmc
from paper_1210_6412_b200.sparse import CsrMatrix

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=1)
def manifest() -> dict:
    with open(os.path.join(GOLDEN, "chain_golden.json")) as fh:
        return json.load(fh)["cases"]


@functools.lru_cache(maxsize=1)
def arrays():
    return dict(np.load(os.path.join(GOLDEN, "chain_golden.npz")))


class _Chain:
    def __init__(self, n, transitions):
        self.n, self.transitions = n, transitions


def chain(name):
    """(chain, goals) of a case, checked against the recorded input hashes."""
    c = manifest()[name]
    a = arrays()
    if f"{name}/rstart" in a:
        p = CsrMatrix(c["n"], a[f"{name}/rstart"], a[f"{name}/col"], a[f"{name}/nonzero"])
    else:
        p = random_dtmc(c["spec"]["n"], c["spec"]["seed"]).transitions
    assert sha(p.rstart) == c["chain_rstart_sha256"], name
    assert sha(p.col) == c["chain_col_sha256"], name
    assert sha(p.nonzero) == c["chain_nonzero_sha256"], name
    return _Chain(c["n"], p), c["goals"]
