"""Pin the CPU oracle and the input generator to the reference's golden fixtures.

Every fixture was produced by the unmodified reference (tests/golden/make_golden.py). The
oracle restates the reference's arithmetic in C without FMA, so it must agree BIT FOR BIT:
same outcome, same iteration count, same residual, same x.
"""

import numpy as np
import pytest

from golden_cases import case_names, expected, manifest, sha, system
from oracle import oracle

SMALL = case_names(max_n=5000)


def _check(name, method, got):
    exp = expected(name, method)
    cfg = exp["config"]
    if exp["outcome"] == "zero_diagonal":
        assert got["status"] == oracle.ZERO_DIAGONAL
        assert got["zero_index"] == exp["zero_index"]
        return
    status = {"ok": oracle.OK, "not_converged": oracle.NOT_CONVERGED,
              "breakdown": oracle.BREAKDOWN}[exp["outcome"]]
    assert got["status"] == status, (name, method, got["status"], exp["outcome"])
    if exp["outcome"] == "breakdown":
        assert got["which"] == exp["which"]
        assert got["iterations"] == exp["breakdown_iteration"]
    assert got["iterations"] == exp["iterations"], (name, method)
    assert float(got["residual_inf"]).hex() == exp["residual_inf"], (name, method)
    if exp["x"] is not None:
        assert np.array_equal(got["x"], exp["x"]), (name, method)
        assert sha(got["x"]) == exp["x_sha256"]
    else:
        assert np.array_equal(got["x"][:: manifest()["sample_stride"]], exp["x_sample"])
        assert sha(got["x"]) == exp["x_sha256"]
    del cfg


@pytest.mark.parametrize("name", SMALL)
def test_generator_reproduces_reference_inputs(name):
    system(name, check=True)


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("method", ["jacobi", "bicgstab"])
def test_oracle_matches_reference_bitwise(name, method):
    m, b = system(name)
    if method not in manifest()["cases"][name]["results"]:
        pytest.skip("method not recorded")
    cfg = manifest()["cases"][name]["results"][method]["config"]
    fn = oracle.jacobi if method == "jacobi" else oracle.bicgstab
    got = fn(m, b, cfg["tolerance"], cfg["max_iterations"], cfg["guess_seed"])
    _check(name, method, got)


@pytest.mark.slow
@pytest.mark.parametrize("method", ["jacobi", "bicgstab"])
def test_oracle_matches_reference_c2(method):
    m, b = system("c2_trial0")
    oracle.set_threads(8)
    try:
        fn = oracle.jacobi if method == "jacobi" else oracle.bicgstab
        got = fn(m, b)
    finally:
        oracle.set_threads(1)
    _check("c2_trial0", method, got)


def test_oracle_threads_bitwise_equal():
    m, b = system("c1_seed77")
    one = oracle.bicgstab(m, b)
    oracle.set_threads(4)
    try:
        four = oracle.bicgstab(m, b)
    finally:
        oracle.set_threads(1)
    assert np.array_equal(one["x"], four["x"])
    assert one["iterations"] == four["iterations"]


def test_oracle_spmv_matches_rowwise_loop():
    # T/test_sparse.py:133-142: row sums run left to right, bitwise equal to a scalar loop
    rng = np.random.default_rng(2024)
    from paper_1210_6412_b200.sparse import csr_from_triplets
    for _ in range(60):
        n = int(rng.integers(1, 33))
        ent = [(i, j, float(rng.uniform(-3, 3))) for i in range(n) for j in range(n)
               if rng.random() < 0.5]
        a = csr_from_triplets(n, ent)
        x = rng.uniform(-5.0, 5.0, n)
        exp = []
        for i in range(n):
            acc = 0.0
            for k in range(a.rstart[i], a.rstart[i + 1]):
                acc += float(a.nonzero[k]) * float(x[a.col[k]])
            exp.append(acc)
        assert np.array_equal(oracle.spmv(a, x), np.array(exp))


def test_oracle_dot_matches_scalar_loop():
    # T/test_solvers.py:85-94
    rng = np.random.default_rng(11)
    for _ in range(50):
        n = int(rng.integers(0, 400))
        u = rng.uniform(-3, 3, n)
        v = rng.uniform(-3, 3, n)
        acc = 0.0
        for a, c in zip(u.tolist(), v.tolist()):
            acc += a * c
        assert oracle.dot(u, v) == acc


# ------------------------------------------------------------------ C5 row-keyed generator
def test_generator_c5_family_properties():
    """The oracle restatement of csrc/generator.cuh: strictly dominant, rows sorted, mean
    row length 1 + mean_offdiag, values in range, diagonal present once per row."""
    from oracle import oracle
    n = 20000
    g = oracle.generate(11, n, 7.0)
    lens = np.diff(g.rstart)
    assert abs(lens.mean() - 8.0) < 0.1 and lens.min() >= 1
    rid = np.repeat(np.arange(n), lens)
    assert np.all((np.diff(g.col) > 0) | (np.diff(rid) > 0))
    on = g.col == rid
    assert np.array_equal(np.bincount(rid[on], minlength=n), np.ones(n))
    off = ~on
    assert g.nonzero[off].min() >= 1 and g.nonzero[off].max() <= 10
    sums = np.bincount(rid[off], weights=g.nonzero[off], minlength=n)
    slack = g.nonzero[on] - sums
    assert slack.min() >= 1 and slack.max() <= 10
    b = oracle.generate_rhs(11, n)
    assert b.min() >= 1 and b.max() <= 10 and np.all(b == np.round(b))


def test_generator_c5_shard_invariant():
    from oracle import oracle
    from paper_1210_6412_b200 import dist
    n = 5003
    full = oracle.generate(3, n, 7.0)
    for world in (2, 3, 8):
        for r in range(world):
            row0, rows = dist.shard_rows(n, world, r)
            part = oracle.generate(3, n, 7.0, row0=row0, rows=rows)
            e0, e1 = full.rstart[row0], full.rstart[row0 + rows]
            assert np.array_equal(part.rstart, full.rstart[row0:row0 + rows + 1] - e0)
            assert np.array_equal(part.col, full.col[e0:e1])
            assert np.array_equal(part.nonzero, full.nonzero[e0:e1])
            assert np.array_equal(oracle.generate_rhs(3, n, row0, rows),
                                  oracle.generate_rhs(3, n)[row0:row0 + rows])


def test_generator_c5_tiny_dimension_caps_count():
    from oracle import oracle
    g = oracle.generate(1, 3, 30.0)  # k capped at n - 1 = 2: dense 3x3
    assert np.array_equal(np.diff(g.rstart), [3, 3, 3])
