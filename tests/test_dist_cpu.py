"""Host logic of the row-sharded path, on CPU (gloo, world size 2).

* the row split (`shard_rows`, restated in Python) equals the library's `mcr_shard_rows`;
* `shard_of` blocks reassemble the matrix with global column indices kept;
* the NCCL bootstrap id reaches every rank through torch.distributed;
* the exchange semantics the CUDA driver relies on -- every rank sweeps its own rows against
  the full iterate, the iterate is rebuilt by an allgather of chunk-padded blocks (so global
  column == buffer index), partial max / dots are reduced in rank order -- reproduce the
  reference Jacobi bit for bit and the reference BiCGStab within tolerance, with the CPU
  oracle standing in for the device kernels (test infrastructure only).
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from golden_cases import expected, system


def test_shard_rows_matches_library():
    import ctypes
    from paper_1210_6412_b200 import _lib, dist
    L = _lib.load()
    for n in (0, 1, 2, 5, 10, 97, 1000, 2 * 10 ** 8):
        for world in (1, 2, 3, 4, 7, 8):
            covered = 0
            for r in range(world):
                a, b = ctypes.c_int64(), ctypes.c_int64()
                assert L.mcr_shard_rows(n, world, r, ctypes.byref(a), ctypes.byref(b)) == 0
                assert (a.value, b.value) == dist.shard_rows(n, world, r)
                assert a.value == min(n, covered)
                covered = a.value + b.value
            assert covered == n


def test_shard_of_reassembles():
    from paper_1210_6412_b200 import dist
    m, _ = system("c4_667_1333")
    for world in (1, 2, 3, 5):
        rs, cols, vals, r0s = [np.zeros(1, np.int64)], [], [], []
        for r in range(world):
            row0, rows, lrs, col, val = dist.shard_of(m, world, r)
            r0s.append(row0)
            assert lrs[0] == 0 and len(lrs) == rows + 1
            rs.append(lrs[1:] + rs[-1][-1])
            cols.append(col)
            vals.append(val)
        assert np.array_equal(np.concatenate(rs), m.rstart)
        assert np.array_equal(np.concatenate(cols), m.col)
        assert np.array_equal(np.concatenate(vals), m.nonzero)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)


def _worker_id(rank, world, port, out):
    _init(rank, world, port)
    from paper_1210_6412_b200 import dist
    uid = dist.Comm.broadcast_id()
    with open(os.path.join(out, f"id{rank}"), "wb") as fh:
        fh.write(uid)
    tdist.destroy_process_group()


def test_nccl_id_bootstrap_gloo():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker_id, args=(2, _free_port(), d), nprocs=2, join=True)
        ids = [open(os.path.join(d, f"id{r}"), "rb").read() for r in range(2)]
    assert len(ids[0]) == 128 and ids[0] == ids[1]


class _Block:
    """A row block in the shape oracle.spmv expects (n rows, local rstart, global col)."""

    def __init__(self, rows, rs, col, val):
        self.n, self.rstart, self.col, self.nonzero = rows, rs, col, val


def _allgather_padded(mine, chunk, world):
    """In-place allgather of chunk-padded blocks: global index == buffer index."""
    buf = torch.zeros(chunk, dtype=torch.float64)
    buf[:len(mine)] = torch.from_numpy(mine)
    parts = [torch.empty(chunk, dtype=torch.float64) for _ in range(world)]
    tdist.all_gather(parts, buf)
    return torch.cat(parts).numpy()


def _rank_order(vals, world):
    """Every rank's partials, then a sum in ascending rank order (k_finalize)."""
    t = torch.tensor(vals, dtype=torch.float64)
    parts = [torch.empty_like(t) for _ in range(world)]
    tdist.all_gather(parts, t)
    return [p.numpy() for p in parts]


def _worker_solve(rank, world, port, out, name):
    _init(rank, world, port)
    from oracle import oracle
    from paper_1210_6412_b200 import dist
    m, b = system(name)
    n = m.n
    row0, rows, rs, col, val = dist.shard_of(m, world, rank)
    chunk = -(-n // world)
    blk = _Block(rows, rs, col, val)
    # diagonal / off-diagonal split of this block, like k_diag / k_split_offdiag
    rid = np.repeat(np.arange(rows), np.diff(rs)) + row0
    on = col == rid
    d = np.zeros(rows)
    d[rid[on] - row0] = val[on]
    keep = ~on
    offrs = np.concatenate([[0], np.cumsum(np.bincount(rid[keep] - row0, minlength=rows))])
    off = _Block(rows, offrs.astype(np.int64), col[keep], val[keep])
    bl = b[row0:row0 + rows]
    # ---- Jacobi: sweep own rows against the full iterate, allgather, max in rank order
    x = np.zeros(chunk * world)
    it = 0
    while True:
        it += 1
        xn = (bl - oracle.spmv(off, x)) / d
        md = np.max(np.abs(xn - x[row0:row0 + rows]))
        x = _allgather_padded(xn, chunk, world)
        mds = _rank_order([md], world)
        if max(p[0] for p in mds) <= 1e-10 or it >= 10_000:
            break
    np.save(os.path.join(out, f"jac{rank}.npy"), np.concatenate([[it], x[:n]]))
    # ---- BiCGStab with per-rank dots reduced in rank order (solvers.py:450-491)
    def mv(full):
        return oracle.spmv(blk, full)

    def gdot(u, v):
        return sum(float(p[0]) for p in _rank_order([oracle.dot(u, v)], world))

    def gmax(u):
        return max(float(p[0]) for p in _rank_order([np.max(np.abs(u))], world))

    xl = np.zeros(rows)
    r = bl - 1.0 * mv(np.zeros(chunk * world))
    q = r.copy()
    y = a = w = 1.0
    v = np.zeros(rows)
    p = np.zeros(rows)
    its = 0
    if gmax(r) > 1e-10:
        while its < 10_000:
            yp, y = y, gdot(q, r)
            beta = (y * a) / (yp * w)
            p = r + beta * (p - w * v)
            v = mv(_allgather_padded(p, chunk, world))
            a = y / gdot(q, v)
            s = r - a * v
            t = mv(_allgather_padded(s, chunk, world))
            small = gmax(s) <= 1e-10
            w = gdot(t, s) / gdot(t, t)
            xl = (xl + a * p) + w * s
            r = s - w * t
            its += 1
            if small:
                break
    xb = _allgather_padded(xl, chunk, world)[:n]
    np.save(os.path.join(out, f"bic{rank}.npy"), np.concatenate([[its], xb]))
    tdist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("c4_2000_3999", 2), ("chain_random1", 2),
                                        ("crit3_460", 3)])
def test_row_block_exchange_semantics_gloo(name, world):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker_solve, args=(world, _free_port(), d, name), nprocs=world, join=True)
        jac = [np.load(os.path.join(d, f"jac{r}.npy")) for r in range(world)]
        bic = [np.load(os.path.join(d, f"bic{r}.npy")) for r in range(world)]
    ej, eb = expected(name, "jacobi"), expected(name, "bicgstab")
    for r in range(world):
        assert int(jac[r][0]) == ej["iterations"]
        assert np.array_equal(jac[r][1:], ej["x"])
        assert abs(int(bic[r][0]) - eb["iterations"]) <= 1
        err = np.max(np.abs(bic[r][1:] - eb["x"])) / max(1.0, np.max(np.abs(eb["x"])))
        assert err <= 1e-9


def test_registry_parallel_device_choice(monkeypatch):
    """SOLVERS' row-sharded drop-ins: MCR_GPU_DEVICES picks the shard devices (repeats allowed,
    at most one shard per row); the names mirror the reference's jacobi-par / bicgstab-par."""
    from paper_1210_6412_b200 import solvers as gs
    assert {"jacobi-gpu-par", "bicgstab-gpu-par"} <= set(gs.SOLVERS)
    monkeypatch.setenv("MCR_GPU_DEVICES", "0,0,1")
    assert gs.parallel_devices(100, gs.SolverConfig()) == [0, 0, 1]
    assert gs.parallel_devices(2, gs.SolverConfig()) == [0, 0]
    monkeypatch.setenv("MCR_GPU_DEVICES", ",")
    import pytest
    with pytest.raises(ValueError):
        gs.parallel_devices(10, gs.SolverConfig())


def test_malformed_csr_rejected_before_ranks_start():
    """solve_local_group validates the CSR once on the host (no rank can fail alone and leave
    the others waiting at an exchange)."""
    import numpy as np
    import pytest
    from paper_1210_6412_b200 import dist
    from paper_1210_6412_b200.sparse import CsrMatrix, DimensionMismatch
    rs = np.array([0, 2, 3], dtype=np.int64)
    good = CsrMatrix(2, rs, np.array([0, 1, 1]), np.array([1.0, 2.0, 3.0]))
    dist.check_csr(good)
    for col in ([1, 0, 1], [0, 0, 1], [0, 2, 1]):
        with pytest.raises(DimensionMismatch):
            dist.check_csr(CsrMatrix(2, rs, np.array(col), np.array([1.0, 2.0, 3.0])))
    with pytest.raises(DimensionMismatch):
        dist.solve_local_group("jacobi", CsrMatrix(2, rs, np.array([1, 0, 1]),
                                                   np.array([1.0, 2.0, 3.0])), np.ones(2), 2)
