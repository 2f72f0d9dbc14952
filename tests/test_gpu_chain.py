"""build_system / reachability_probabilities on the device against the
reference's outputs (tests/golden/chain_golden.*): the state partition, M = I - A and the
right-hand side bit for bit; the reachability vector from Jacobi bit for bit; the reference's
errors for bad goal sets and unknown methods."""

import numpy as np
import pytest

from chain_cases import arrays, chain, manifest
from golden_cases import sha

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gm():
    from paper_1210_6412_b200 import _lib, markov
    _lib.load()
    assert _lib.device_count() >= 1
    return markov


NAMES = sorted(manifest())


@pytest.mark.parametrize("name", NAMES)
def test_system_bit_identical(gm, name):
    c = manifest()[name]
    ch, goals = chain(name)
    cs = gm.ChainSystem(ch, goals)
    try:
        cls, unc, M, rhs = cs.export()
    finally:
        cs.close()
    assert cs.k == c["k"] and M.rstart[-1] == c["m_nnz"]
    assert sha(cls) == c["classes_sha256"]
    assert sha(unc) == c["uncertain_sha256"]
    assert sha(M.rstart) == c["m_rstart_sha256"]
    assert sha(M.col) == c["m_col_sha256"]
    assert sha(M.nonzero) == c["m_nonzero_sha256"], name
    assert sha(rhs) == c["rhs_sha256"], name


@pytest.mark.parametrize("name", [n for n in NAMES if "jacobi-seq" in manifest()[n]])
def test_reachability_jacobi_bit_identical(gm, name):
    from paper_1210_6412_b200.solvers import Breakdown, NotConverged
    c = manifest()[name]
    ch, goals = chain(name)
    exp = c["jacobi-seq"]
    if exp["outcome"] != "ok":
        with pytest.raises((NotConverged, Breakdown)):
            gm.reachability_probabilities(ch, goals, "jacobi-gpu")
        return
    x, rep = gm.reachability_probabilities(ch, goals, "jacobi-gpu")
    assert rep.iterations == exp["iterations"]
    assert sha(x) == exp["x_sha256"], name


@pytest.mark.parametrize("name", [n for n in NAMES if "bicgstab-seq" in manifest()[n]])
def test_reachability_bicgstab(gm, name):
    from paper_1210_6412_b200.solvers import Breakdown, NotConverged
    c = manifest()[name]
    ch, goals = chain(name)
    exp = c["bicgstab-seq"]
    if exp["outcome"] != "ok":  # the exact-dots mode reproduces the reference's failure
        with pytest.raises((NotConverged, Breakdown)) as info:
            gm.reachability_probabilities(ch, goals, "bicgstab-gpu-exact")
        assert type(info.value).__name__ == exp["outcome"]
        return
    for method in ("bicgstab-gpu-exact", "bicgstab-gpu"):  # reference-order dots by default
        x, rep = gm.reachability_probabilities(ch, goals, method)
        assert rep.iterations == exp["iterations"]
        assert sha(x) == exp["x_sha256"], (name, method)
    from paper_1210_6412_b200.solvers import SolverConfig
    try:
        xt, rept = gm.reachability_probabilities(ch, goals, "bicgstab-gpu",
                                                 SolverConfig(dot_products="tree"))
    except (NotConverged, Breakdown):
        return  # the opt-in tree order may stop elsewhere; nothing to compare
    ref = arrays().get(f"{name}/bicgstab-seq/x")
    if ref is not None:
        assert np.max(np.abs(xt - ref)) <= 1e-9


def test_demo_chain_values(gm):
    ch, goals = chain("demo_g3")
    x, rep = gm.reachability_probabilities(ch, goals)
    assert rep.converged
    assert np.allclose(x, [0.625, 0.0, 0.25, 1.0], atol=1e-8)   # T/test_markov.py:184-187
    x, rep = gm.reachability_probabilities(ch, [0, 1, 2, 3])
    assert rep.iterations == 0 and rep.converged and x.tolist() == [1.0] * 4


def test_bad_goals_and_method(gm):
    ch, _ = chain("demo_g3")
    with pytest.raises(ValueError):
        gm.reachability_probabilities(ch, [])
    with pytest.raises(ValueError):
        gm.reachability_probabilities(ch, [4])
    with pytest.raises(ValueError):
        gm.reachability_probabilities(ch, [3], method="gauss")


def test_build_system_returns_reference_types(gm):
    pytest.importorskip("mcreach")
    import mcreach.markov as mm
    ch, goals = chain("oracle_chain_3")
    s = gm.build_system(ch, goals)
    assert isinstance(s, mm.LinearSystem) and isinstance(s.partition, mm.StatePartition)
    c = manifest()["oracle_chain_3"]
    assert sha(s.rhs) == c["rhs_sha256"] and sha(s.matrix.nonzero) == c["m_nonzero_sha256"]


def test_seeded_guess_chain(gm):
    """guess_seed starts the reduced solve from default_rng(seed).random(k), as the
    reference's _initial_guess does (solvers.py:153-156)."""
    from paper_1210_6412_b200.solvers import SolverConfig
    ch, goals = chain("dtmc_1000")
    x0, r0 = gm.reachability_probabilities(ch, goals, "jacobi-gpu")
    x1, r1 = gm.reachability_probabilities(ch, goals, "jacobi-gpu", SolverConfig(guess_seed=7))
    assert r1.converged and np.max(np.abs(x1 - x0)) <= 1e-8
    assert r1.iterations != r0.iterations or not np.array_equal(x1, x0)


@pytest.mark.parametrize("name", ["demo_g3", "oracle_chain_7", "dtmc_1000"])
def test_partition_states(gm, name):
    c = manifest()[name]
    ch, goals = chain(name)
    part = gm.partition_states(ch, goals)
    cls = np.full(ch.n, 2, dtype=np.int8)
    cls[sorted(part.prob_zero)] = 0
    cls[sorted(part.prob_one)] = 1
    assert sha(cls) == c["classes_sha256"] and sha(part.uncertain) == c["uncertain_sha256"]
    assert all(part.index_of[int(s)] == i for i, s in enumerate(part.uncertain))


@pytest.mark.parametrize("name", [n for n in NAMES if "jacobi-seq" in manifest()[n]
                                  and "bicgstab-seq" in manifest()[n]])
def test_reachability_on_staged_layout(gm, name, monkeypatch):
    """The chain's M = I - A (negative off-diagonals) solved on the band-staged layout (AUTO
    picks it for large systems; the cut is lowered to 0 here): the same bits as the tiles."""
    from paper_1210_6412_b200.solvers import Breakdown, NotConverged
    monkeypatch.setenv("MCR_STAGED_MIN_X_BYTES", "0")
    c = manifest()[name]
    ch, goals = chain(name)
    for method, key in (("jacobi-gpu", "jacobi-seq"), ("bicgstab-gpu-exact", "bicgstab-seq")):
        exp = c[key]
        if exp["outcome"] != "ok":
            with pytest.raises((NotConverged, Breakdown)):
                gm.reachability_probabilities(ch, goals, method)
            continue
        x, rep = gm.reachability_probabilities(ch, goals, method)
        assert rep.iterations == exp["iterations"]
        assert sha(x) == exp["x_sha256"], (name, method)
