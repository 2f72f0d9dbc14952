"""Row-sharded solves against the reference's golden outputs, on one GPU.

`solve_local_group` runs `world` ranks as threads of this process: each rank uploads its
row block (global columns) with mcr_shard_create and runs the same multi-rank driver a
torchrun/NCCL job runs, with the collectives as event-ordered device copies. Bar, as for
the reference's own row-block parallel solvers (T/test_solvers.py:157-172, 242-256):
Jacobi and BiCGStab bit-identical to the reference at every world size (x, iterations,
residual): the sharded BiCGStab gathers the vectors of each inner product and every rank sums
the whole vectors in the reference's order (k_xdot), so all ranks take the reference's scalar
steps. The opt-in tree order (per-rank trees combined in rank order) is checked within the
north-star tolerance.
The NCCL transport itself is exercised at world size 1 (one GPU per box here).
"""

import numpy as np
import pytest

from golden_cases import case_names, expected, manifest, sha, system

pytestmark = pytest.mark.gpu

REL_TOL = 1e-9


@pytest.fixture(scope="module")
def mods():
    from paper_1210_6412_b200 import _lib, dist, solvers
    _lib.load()
    assert _lib.device_count() >= 1, "no CUDA device visible"
    return dist, solvers


def run(mods, method, name, world, p2p=False, dots="sequential"):
    dist, gs = mods
    m, b = system(name)
    if dist.shard_rows(m.n, world, world - 1)[1] < 1:
        pytest.skip(f"n = {m.n} leaves a rank of {world} without rows")
    exp = expected(name, method)
    c = exp["config"]
    conf = gs.SolverConfig(tolerance=c["tolerance"], max_iterations=c["max_iterations"],
                           guess_seed=c["guess_seed"], dot_products=dots)
    try:
        res, per = dist.solve_local_group(method, m, b, world, conf, p2p=p2p)
        return exp, "ok", res, None, per
    except gs.NotConverged as err:
        return exp, "not_converged", err.result, err, None
    except gs.Breakdown as err:
        return exp, "breakdown", err.result, err, None
    except gs.ZeroDiagonal as err:
        return exp, "zero_diagonal", None, err, None


def rel_err(x, ref):
    scale = max(1.0, float(np.max(np.abs(ref)))) if len(ref) else 1.0
    return float(np.max(np.abs(x - ref))) / scale if len(ref) else 0.0


def check(mods, method, name, world, iter_slack=1, p2p=False, dots="sequential"):
    exp, outcome, res, err, per = run(mods, method, name, world, p2p, dots)
    assert outcome == exp["outcome"], (name, world, outcome, exp["outcome"])
    if outcome == "zero_diagonal":
        assert err.index == exp["zero_index"]
        return
    if per is not None:  # every rank reports the same count and residual
        assert len({r.iterations for r in per}) == 1
        assert len({float(r.residual_inf).hex() for r in per}) == 1
    stride = manifest()["sample_stride"]
    ref_x = exp["x"] if exp["x"] is not None else exp["x_sample"]
    got_x = res.x if exp["x"] is not None else res.x[::stride]
    if outcome == "breakdown":
        assert err.which == exp["which"]
        assert err.iteration == exp["breakdown_iteration"]
    if method == "jacobi" or dots == "sequential":
        assert res.iterations == exp["iterations"], (name, world, res.iterations, exp["iterations"])
        assert np.array_equal(got_x, ref_x), (name, world, rel_err(got_x, ref_x))
        assert sha(res.x) == exp["x_sha256"]
        assert float(res.residual_inf).hex() == exp["residual_inf"]
    else:
        assert abs(res.iterations - exp["iterations"]) <= iter_slack, (name, world, res.iterations)
        if outcome == "ok":
            assert rel_err(got_x, ref_x) <= REL_TOL, (name, world, rel_err(got_x, ref_x))


CASES = ["c1_seed77", "c4_92_211", "c4_2000_3999", "c4_7647_15293", "chain_random1",
         "chain_random2", "crit3_1281", "crit4_0", "parallel_large", "seeded_guess", "grid_50_3",
         "grid_5_0", "dense_1024"]
KATS = ["kat_breakdown_qv", "kat_breakdown_tt", "kat_divergent", "kat_golden2x2",
        "kat_identity4", "kat_singular_consistent", "kat_tiny_budget", "kat_zero_diagonal",
        "kat_zero_rhs"]


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("name", CASES)
def test_sharded_jacobi_bit_identical(mods, name, world):
    check(mods, "jacobi", name, world)


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("name", CASES)
def test_sharded_bicgstab_matches_reference(mods, name, world):
    check(mods, "bicgstab", name, world)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name", ["c1_seed77", "c4_2000_3999", "crit3_1281", "parallel_large"])
def test_sharded_bicgstab_tree_order(mods, name, world):
    """The opt-in tree order on shards: x within the north-star tolerance; its stopping
    iteration may move with the order (c2 below)."""
    check(mods, "bicgstab", name, world, iter_slack=3, dots="tree")


@pytest.mark.parametrize("name", KATS)
@pytest.mark.parametrize("method", ["jacobi", "bicgstab"])
def test_sharded_known_answers(mods, name, method):
    check(mods, method, name, 2)


def test_sharded_world_one_equals_single_gpu(mods):
    """world = 1 runs the shard driver (exchange points included): same bits as the plain
    handle streaming the same tiles."""
    dist, gs = mods
    m, b = system("c1_trial0")
    r1, _ = dist.solve_local_group("bicgstab", m, b, 1)
    r0 = gs.DeviceMatrix(m, 0, 5).solve("bicgstab", b, None, 1e-10, 10_000)  # TILES_STREAM
    assert r0[0] == 0 and r1.iterations == r0[2].iterations
    assert np.array_equal(r1.x, r0[1])


@pytest.mark.slow
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_c2(mods, world):
    """Jacobi and BiCGStab bit-identical (BiCGStab stops at the reference's 79). In the opt-in
    tree order the stopping iteration moves (reference cumsum 79, exactly rounded fsum 83, BLAS
    dot 84: tools/bicgstab_sensitivity.py; rank-order partials land at 85), x within 1e-9."""
    check(mods, "jacobi", "c2_trial0", world)
    check(mods, "bicgstab", "c2_trial0", world)
    check(mods, "bicgstab", "c2_trial0", world, iter_slack=6, dots="tree")


def test_shard_bounds_rejected(mods):
    dist, gs = mods
    m, b = system("c4_92_211")
    comms = dist.Comm.local_group(2)
    try:
        row0, rows, rs, col, val = dist.shard_of(m, 2, 1)
        with pytest.raises(Exception):
            dist.ShardMatrix(comms[0], m.n, row0, rows, rs, col, val)  # rank 0 given rank 1's rows
    finally:
        for c in comms:
            c.close()


def test_nccl_transport_world_one(mods):
    """The NCCL transport end to end (bootstrap id over torch.distributed, grouped
    allgather + slot exchange inside every sweep) at the world size one box allows."""
    import os
    import torch.distributed as tdist
    dist, gs = mods
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    tdist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = dist.Comm.nccl(0)
        assert (comm.world, comm.rank) == (1, 0)
        m, b = system("c4_2000_3999")
        sh = dist.ShardMatrix.from_matrix(comm, m)
        exp = expected("c4_2000_3999", "jacobi")
        r = dist.jacobi_solve_sharded(sh, b)
        assert r.iterations == exp["iterations"] and sha(r.x) == exp["x_sha256"]
        rb = dist.bicgstab_solve_sharded(sh, b)
        expb = expected("c4_2000_3999", "bicgstab")
        assert abs(rb.iterations - expb["iterations"]) <= 1
        assert rel_err(rb.x, expb["x"]) <= REL_TOL
        sh.close()
        # fused-exchange setup over NCCL (IPC export + byte allgather; no peer at world 1)
        sh = dist.ShardMatrix.from_matrix(comm, m)
        sh.enable_p2p()
        r2 = dist.jacobi_solve_sharded(sh, b)
        assert r2.iterations == exp["iterations"] and sha(r2.x) == exp["x_sha256"]
        sh.close()
        comm.close()
    finally:
        tdist.destroy_process_group()


P2P_CASES = ["c1_seed77", "c4_2000_3999", "chain_random2", "crit3_1281", "seeded_guess",
             "grid_50_3", "kat_breakdown_qv", "kat_divergent"]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", P2P_CASES)
@pytest.mark.parametrize("method", ["jacobi", "bicgstab"])
def test_fused_p2p_exchange(mods, name, world, method):
    """mcr_shard_enable_p2p: the producers store their rows straight into every peer's copy
    of x / p / s; the per-sweep collective is only the slot exchange. Same bar."""
    check(mods, method, name, world, p2p=True)


def test_fused_p2p_bit_identical_to_allgather(mods):
    """Fused and allgather exchange give the same bits (BiCGStab included: the exchange only
    moves data, the arithmetic and its order are unchanged)."""
    dist, gs = mods
    m, b = system("c4_7647_15293")
    for method in ("jacobi", "bicgstab"):
        r1, _ = dist.solve_local_group(method, m, b, 3)
        r2, _ = dist.solve_local_group(method, m, b, 3, p2p=True)
        assert r1.iterations == r2.iterations
        assert np.array_equal(r1.x, r2.x)
        assert float(r1.residual_inf).hex() == float(r2.residual_inf).hex()


@pytest.mark.slow
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", P2P_CASES)
@pytest.mark.parametrize("method", ["jacobi", "bicgstab"])
def test_sharded_staged(mods, name, world, method, monkeypatch):
    """Row shards in the band-staged layout (AUTO picks it once x is large; the cut is lowered
    to 0 here): the same results as the tiled shards and the reference."""
    monkeypatch.setenv("MCR_STAGED_MIN_X_BYTES", "0")
    check(mods, method, name, world)
    check(mods, method, name, world, p2p=True)


def test_sharded_staged_layout_in_use(mods, monkeypatch):
    dist, _ = mods
    m, _ = system("c1_seed77")
    monkeypatch.setenv("MCR_STAGED_MIN_X_BYTES", "0")
    comms = dist.Comm.local_group(2)
    try:
        sh = dist.ShardMatrix.from_matrix(comms[1], m)
        try:
            assert sh.info()["storage"] == 6
        finally:
            sh.close()
    finally:
        for c in comms:
            c.close()


def test_fused_p2p_c2(mods):
    check(mods, "jacobi", "c2_trial0", 4, p2p=True)
    check(mods, "bicgstab", "c2_trial0", 4, p2p=True)


# ---- the registry's row-sharded drop-ins (SOLVERS["jacobi-gpu-par" / "bicgstab-gpu-par"]),
# the GPU analogue of jacobi_solve_parallel / bicgstab_solve_parallel (S/solvers.py:233-274,
# 429-447). MCR_GPU_DEVICES places several shards on the one GPU of this box.
def run_registry(mods, method, name, devices, monkeypatch):
    dist, gs = mods
    monkeypatch.setenv("MCR_GPU_DEVICES", devices)
    m, b = system(name)
    exp = expected(name, method)
    c = exp["config"]
    conf = gs.SolverConfig(tolerance=c["tolerance"], max_iterations=c["max_iterations"],
                           guess_seed=c["guess_seed"])
    fn = gs.SOLVERS[f"{method}-gpu-par"]
    try:
        return exp, "ok", fn(m, b, conf), None
    except gs.NotConverged as err:
        return exp, "not_converged", err.result, err
    except gs.Breakdown as err:
        return exp, "breakdown", err.result, err
    except gs.ZeroDiagonal as err:
        return exp, "zero_diagonal", None, err


@pytest.mark.parametrize("devices", ["0", "0,0", "0,0,0"])
@pytest.mark.parametrize("name", ["c1_seed77", "c4_2000_3999", "chain_random1", "seeded_guess",
                                  "dense_1024"] + KATS)
@pytest.mark.parametrize("method", ["jacobi", "bicgstab"])
def test_registry_parallel_methods(mods, method, name, devices, monkeypatch):
    exp, outcome, res, err = run_registry(mods, method, name, devices, monkeypatch)
    m, _ = system(name)
    assert outcome == exp["outcome"], (name, devices, outcome, exp["outcome"])
    if outcome == "zero_diagonal":
        assert err.index == exp["zero_index"]
        return
    stride = manifest()["sample_stride"]
    ref_x = exp["x"] if exp["x"] is not None else exp["x_sample"]
    got_x = res.x if exp["x"] is not None else res.x[::stride]
    assert res.x.shape == (m.n,) and res.wall_time > 0.0
    if outcome == "breakdown":
        assert err.which == exp["which"] and err.iteration == exp["breakdown_iteration"]
    # bit-identical to the reference at every shard count: Jacobi's iterates do not depend on
    # the row split, and bicgstab-gpu-par's default (reference-order) inner products are summed
    # over the gathered vectors on every shard, as the reference's bicgstab_solve_parallel is
    # bit-identical to its sequential one
    assert res.iterations == exp["iterations"]
    assert np.array_equal(got_x, ref_x)
    assert float(res.residual_inf).hex() == exp["residual_inf"]


def test_registry_parallel_workers_clamped(mods, monkeypatch):
    """Without MCR_GPU_DEVICES the shard count is min(workers, visible GPUs, n); one GPU
    runs the plain single-device solve (same bits)."""
    dist, gs = mods
    monkeypatch.delenv("MCR_GPU_DEVICES", raising=False)
    from paper_1210_6412_b200 import _lib
    count = _lib.device_count()
    assert gs.parallel_devices(10, gs.SolverConfig(workers=64)) == list(range(min(count, 10)))
    assert gs.parallel_devices(1, gs.SolverConfig()) == [0]
    m, b = system("c4_2000_3999")
    one = gs.SOLVERS["jacobi-gpu"](m, b)
    par = gs.SOLVERS["jacobi-gpu-par"](m, b, gs.SolverConfig(workers=8))
    assert par.iterations == one.iterations and np.array_equal(par.x, one.x)
    from paper_1210_6412_b200.sparse import CsrMatrix
    empty = gs.SOLVERS["bicgstab-gpu-par"](CsrMatrix(0, np.zeros(1, np.int64),
                                                     np.zeros(0, np.int64), np.zeros(0)),
                                           np.zeros(0))
    assert empty.converged and empty.iterations == 0


def test_registry_parallel_sequential_dots_is_exact(mods, monkeypatch):
    """bicgstab-gpu-par with the reference's sequential inner products on two shards (one
    chain over all gathered rows on each): bit-identical to the reference's bicgstab."""
    dist, gs = mods
    monkeypatch.setenv("MCR_GPU_DEVICES", "0,0")
    name = "c4_2000_3999"
    m, b = system(name)
    exp = expected(name, "bicgstab")
    c = exp["config"]
    conf = gs.SolverConfig(tolerance=c["tolerance"], max_iterations=c["max_iterations"],
                           guess_seed=c["guess_seed"], dot_products="sequential")
    got = gs.SOLVERS["bicgstab-gpu-par"](m, b, conf)
    assert got.iterations == exp["iterations"]
    assert sha(got.x) == exp["x_sha256"]


@pytest.mark.parametrize("devices", ["0,0", "0,0,0"])
@pytest.mark.parametrize("key", ["pardots/c1_seed77/w4", "pardots/c4_2000_3999/w2",
                                 "pardots/c4_5647_11293/w16", "pardots/parallel_large/w4"])
def test_registry_parallel_dot_products_on_shards(mods, key, devices, monkeypatch):
    """parallel_dot_products=True with config.workers = k on row shards (the shard count is
    independent of k): the k _row_blocks chains of the gathered vectors, combined in order --
    the reference's bicgstab_solve_parallel bit for bit (golden_extra, made by the reference)."""
    import json
    import os
    dist, gs = mods
    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    with open(os.path.join(here, "golden_extra.json")) as fh:
        exp = json.load(fh)["cases"][key]
    monkeypatch.setenv("MCR_GPU_DEVICES", devices)
    m, b = system(key.split("/")[1])
    res = gs.SOLVERS["bicgstab-gpu-par"](m, b, gs.SolverConfig(workers=exp["workers"],
                                                               parallel_dot_products=True))
    assert res.iterations == exp["iterations"], (key, devices, res.iterations)
    assert sha(res.x) == exp["x_sha256"]
    assert float(res.residual_inf).hex() == exp["residual_inf"]

