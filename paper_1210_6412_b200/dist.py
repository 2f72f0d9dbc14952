"""Row-sharded solves over several GPUs.

The reference parallelises one solve over CPU worker threads by contiguous row blocks
(``_row_blocks``, ``mcreach/solvers.py:159-168``; ``jacobi_solve_parallel`` :233-274;
``_ParOps`` :314-396): every worker computes its rows of ``x'`` (or of ``M p``) against the
whole current vector, then a barrier. Here the workers are GPUs: rank ``r`` of ``world`` owns
rows ``[r*c, min(n, (r+1)*c))`` with ``c = ceil(n / world)`` as a CSR whose columns stay
global, and the barrier is an in-place allgather of the vector the next SpMV gathers from,
plus an exchange of every rank's reduction partials (dots, max) that each rank then reduces
in rank order -- so all ranks hold bit-identical scalars and take the same stop decision.
Jacobi iterates are bit-identical to one GPU and to the reference at every world size
(max is order-free), exactly as ``jacobi_solve_parallel`` is bit-identical to
``jacobi_solve`` (``T/test_solvers.py:157-172``).

Two transports behind the same C ABI (``include/mcr.h``):

* ``Comm.nccl(device)`` -- one process per GPU (torchrun), NCCL over NVLink; the NCCL
  unique id is broadcast with ``torch.distributed`` (any backend).
* ``Comm.local_group(world)`` -- ``world`` ranks as threads of this process (on one or
  several devices), collectives as event-ordered peer copies; ``solve_local_group`` uses it
  to run the multi-rank path end to end on a single GPU.
"""

from __future__ import annotations

import ctypes
import threading
import time
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from .solvers import SolverConfig, SolveResult, _raise_native, outcome
from .sparse import DimensionMismatch

__all__ = ["shard_rows", "shard_of", "Comm", "ShardMatrix", "jacobi_solve_sharded",
           "bicgstab_solve_sharded", "solve_local_group"]


def shard_rows(n: int, world: int, rank: int):
    """(first row, row count) of ``rank`` -- the same split as ``mcr_shard_rows``."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError(f"bad shard request n={n} world={world} rank={rank}")
    c = -(-n // world)
    lo = min(n, c * rank)
    hi = min(n, lo + c)
    return lo, hi - lo


def shard_of(m, world: int, rank: int):
    """This rank's rows of a CSR matrix: (row0, rows, local rstart, global col, nonzero)."""
    row0, rows = shard_rows(int(m.n), world, rank)
    rs = np.asarray(m.rstart, dtype=np.int64)[row0:row0 + rows + 1]
    e0, e1 = int(rs[0]), int(rs[-1])
    return (row0, rows, np.ascontiguousarray(rs - e0),
            np.ascontiguousarray(np.asarray(m.col, dtype=np.int64)[e0:e1]),
            np.ascontiguousarray(np.asarray(m.nonzero, dtype=np.float64)[e0:e1]))


class Comm:
    """A communicator handle (``mcr_comm``)."""

    def __init__(self, handle: ctypes.c_void_p):
        self._L = _lib.load()
        self._h = handle
        w, r, d = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        self._L.mcr_comm_info(handle, ctypes.byref(w), ctypes.byref(r), ctypes.byref(d))
        self.world, self.rank, self.device = w.value, r.value, d.value

    @property
    def handle(self):
        return self._h

    @staticmethod
    def unique_id() -> bytes:
        L = _lib.load()
        buf = ctypes.create_string_buffer(_lib.COMM_ID_BYTES)
        rc = L.mcr_comm_unique_id(buf)
        if rc != _lib.MCR_OK:
            _raise_native(rc)
        return buf.raw

    @staticmethod
    def broadcast_id(group=None) -> bytes:
        """Rank 0 creates the NCCL id; every rank of the torch.distributed group receives it."""
        import torch.distributed as dist
        obj = [Comm.unique_id() if dist.get_rank(group) == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return obj[0]

    @classmethod
    def nccl(cls, device: int, group=None, uid: Optional[bytes] = None) -> "Comm":
        """Collective over the ranks of the (initialised) torch.distributed group."""
        import torch.distributed as dist
        if uid is None:
            uid = cls.broadcast_id(group)
        L = _lib.load()
        h = ctypes.c_void_p()
        rc = L.mcr_comm_create_nccl(uid, dist.get_world_size(group), dist.get_rank(group),
                                    int(device), ctypes.byref(h))
        if rc != _lib.MCR_OK:
            _raise_native(rc)
        return cls(h)

    @classmethod
    def local_group(cls, world: int, devices: Optional[Sequence[int]] = None) -> List["Comm"]:
        L = _lib.load()
        out = (ctypes.c_void_p * world)()
        devs = None
        if devices is not None:
            devs = (ctypes.c_int * world)(*[int(d) for d in devices])
        rc = L.mcr_comm_create_local(int(world), devs, out)
        if rc != _lib.MCR_OK:
            _raise_native(rc)
        return [cls(ctypes.c_void_p(out[r])) for r in range(world)]

    def close(self):
        if self._h:
            self._L.mcr_comm_destroy(self._h)
            self._h = None


class ShardMatrix:
    """This rank's rows of an ``n_global`` system, resident on the communicator's device."""

    def __init__(self, comm: Comm, n_global: int, row0: int, rows: int, rstart, col, nonzero,
                 _handle=None):
        L = _lib.load()
        self._L = L
        self.comm = comm
        self.n_global, self.row0, self.n = int(n_global), int(row0), int(rows)
        if _handle is None:
            rs = np.ascontiguousarray(rstart, dtype=np.int64)
            c = np.ascontiguousarray(col, dtype=np.int64)
            v = np.ascontiguousarray(nonzero, dtype=np.float64)
            h = ctypes.c_void_p()
            rc = L.mcr_shard_create(comm.handle, self.n_global, self.row0, self.n,
                                    rs.ctypes.data, c.ctypes.data, v.ctypes.data, ctypes.byref(h))
            if rc != _lib.MCR_OK:
                _raise_native(rc)
            _handle = h
        self._h = _handle

    @classmethod
    def generated(cls, comm: Comm, n: int, mean_offdiag: float = 7.0, lo: int = 1, hi: int = 10,
                  seed: int = 0, storage: int = _lib.STORAGE_AUTO) -> "ShardMatrix":
        """This rank's rows of the row-keyed synthetic system, generated in HBM (config C5)."""
        L = _lib.load()
        h = ctypes.c_void_p()
        rc = L.mcr_generate(comm.handle, comm.device, int(n), float(mean_offdiag), int(lo),
                            int(hi), int(seed), int(storage), ctypes.byref(h))
        if rc != _lib.MCR_OK:
            _raise_native(rc)
        row0, rows = shard_rows(int(n), comm.world, comm.rank)
        return cls(comm, n, row0, rows, None, None, None, _handle=h)

    def generated_rhs(self, seed: int, out_device_ptr: int) -> None:
        rc = self._L.mcr_generate_rhs(self._h, int(seed), ctypes.c_void_p(out_device_ptr))
        if rc != _lib.MCR_OK:
            _raise_native(rc)

    def solve_device(self, method: str, d_b: int, d_x0, tol: float, max_it: int, d_x: int):
        """Device-pointer solve of this rank's rows (inputs resident in HBM)."""
        fn = {"jacobi": self._L.mcr_jacobi_device, "bicgstab": self._L.mcr_bicgstab_device}[method]
        rep = _lib.Report()
        rc = fn(self._h, ctypes.c_void_p(d_b), None if d_x0 is None else ctypes.c_void_p(d_x0),
                float(tol), int(max_it), ctypes.c_void_p(d_x), ctypes.byref(rep))
        return rc, rep

    def enable_p2p(self) -> None:
        """Fused exchange (mcr_shard_enable_p2p): collective, before the first solve."""
        rc = self._L.mcr_shard_enable_p2p(self._h)
        if rc != _lib.MCR_OK:
            _raise_native(rc)

    def set_stream(self, stream_ptr: int) -> None:
        self._L.mcr_set_stream(self._h, ctypes.c_void_p(stream_ptr))

    @classmethod
    def from_matrix(cls, comm: Comm, m) -> "ShardMatrix":
        row0, rows, rs, col, val = shard_of(m, comm.world, comm.rank)
        return cls(comm, int(m.n), row0, rows, rs, col, val)

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        inf = _lib.MatrixInfo()
        self._L.mcr_matrix_info_get(self._h, ctypes.byref(inf))
        return {f: getattr(inf, f) for f, _ in _lib.MatrixInfo._fields_}

    def close(self):
        if self._h:
            self._L.mcr_matrix_destroy(self._h)
            self._h = None

    def set_dots(self, dots: str = "sequential", dot_blocks: int = 1) -> None:
        """BiCGStab's inner products on this shard (mcr_set_dot_mode / mcr_set_dot_blocks):
        "sequential" -- the reference's left-to-right sums of the whole gathered vectors, the same
        bits on every rank and as one GPU; "tree" -- per-rank trees combined in rank order."""
        rc = self._L.mcr_set_dot_mode(self._h, _lib.DOT_MODES[dots])
        if rc == _lib.MCR_OK:
            rc = self._L.mcr_set_dot_blocks(self._h, int(dot_blocks))
        if rc != _lib.MCR_OK:
            _raise_native(rc)

    def solve(self, method: str, b_local, x0_local, tol: float, max_it: int):
        fn = {"jacobi": self._L.mcr_jacobi, "bicgstab": self._L.mcr_bicgstab}[method]
        b = np.ascontiguousarray(b_local, dtype=np.float64)
        if b.shape != (self.n,):
            raise DimensionMismatch(f"right-hand side slice of shape {b.shape} for {self.n} rows")
        x = np.empty(self.n)
        x0p = None
        if x0_local is not None:
            x0 = np.ascontiguousarray(x0_local, dtype=np.float64)
            x0p = x0.ctypes.data
        rep = _lib.Report()
        rc = fn(self._h, b.ctypes.data, x0p, float(tol), int(max_it), x.ctypes.data,
                ctypes.byref(rep))
        return rc, x, rep


def _guess_slice(shard: ShardMatrix, cfg) -> Optional[np.ndarray]:
    """solvers.py:153-156 on the whole vector, then this rank's rows."""
    seed = getattr(cfg, "guess_seed", None)
    if seed is None:
        return None
    return np.random.default_rng(seed).random(shard.n_global)[shard.row0:shard.row0 + shard.n]


def _solve_sharded(method, shard: ShardMatrix, b_local, config, raise_errors=True):
    cfg = config or SolverConfig()
    start = time.perf_counter()
    if method == "bicgstab":  # the reference's dot order by default (solvers.py:136-141, 384-396)
        dots = getattr(cfg, "dot_products", "sequential")
        blocks = cfg.resolved_workers() if getattr(cfg, "parallel_dot_products", False) else 1
        shard.set_dots("tree" if dots == "tree" else "sequential", max(1, int(blocks)))
    rc, x, rep = shard.solve(method, b_local, _guess_slice(shard, cfg), cfg.tolerance,
                             cfg.max_iterations)
    result, err = outcome(rc, x, rep, start)
    if err is not None and raise_errors:
        raise err
    return result, err


def jacobi_solve_sharded(shard: ShardMatrix, b_local, config: Optional[SolverConfig] = None):
    """``jacobi_solve`` on this rank's rows; x of the result is this rank's slice."""
    return _solve_sharded("jacobi", shard, b_local, config)[0]


def bicgstab_solve_sharded(shard: ShardMatrix, b_local, config: Optional[SolverConfig] = None):
    """``bicgstab_solve`` on this rank's rows; x of the result is this rank's slice."""
    return _solve_sharded("bicgstab", shard, b_local, config)[0]


def check_csr(m) -> None:
    """The CsrMatrix invariants the upload enforces (sparse.py:101-118: row starts from 0 to
    nnz, non-decreasing; columns in range and strictly ascending within each row), checked on
    the host before any rank starts, so a malformed matrix fails at once on every rank instead
    of leaving the other ranks waiting at the first exchange."""
    n = int(m.n)
    rs = np.asarray(m.rstart, dtype=np.int64)
    col = np.asarray(m.col, dtype=np.int64)
    if rs.shape != (n + 1,) or rs[0] != 0 or rs[-1] != col.shape[0] or np.any(np.diff(rs) < 0):
        raise DimensionMismatch("malformed CSR row starts")
    if col.size and (col.min() < 0 or col.max() >= n):
        raise DimensionMismatch("CSR column index out of range")
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rs))
    same = rows[1:] == rows[:-1]
    if np.any(np.diff(col)[same] <= 0):
        raise DimensionMismatch("CSR columns not strictly ascending within a row")


def solve_local_group(method: str, m, b, world: int, config: Optional[SolverConfig] = None,
                      devices: Optional[Sequence[int]] = None, p2p: bool = False):
    """Solve ``m x = b`` as ``world`` row shards driven by ``world`` threads of this process.

    Returns ``(result, per_rank)``: the assembled SolveResult (full x, rank 0's iteration
    count and residual) and every rank's own SolveResult. Raises the reference's exception
    (with the assembled x) when the ranks report one.
    """
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (m.n,):
        raise DimensionMismatch(f"right-hand side of shape {b.shape} against dimension {m.n}")
    if m.n < 1 or shard_rows(int(m.n), world, world - 1)[1] < 1:
        raise ValueError(f"{world} ranks need every rank to hold rows (n = {m.n})")
    check_csr(m)
    comms = Comm.local_group(world, devices)
    shards = [None] * world
    out = [None] * world
    errs = [None] * world
    start = time.perf_counter()

    def run(r):
        try:
            sh = ShardMatrix.from_matrix(comms[r], m)
            shards[r] = sh
            if p2p:
                sh.enable_p2p()
            out[r] = _solve_sharded(method, sh, b[sh.row0:sh.row0 + sh.n], config,
                                    raise_errors=False)
        except BaseException as e:  # surfaced below
            errs[r] = e

    try:
        threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    finally:
        for sh in shards:
            if sh is not None:
                sh.close()
        for c in comms:
            c.close()
    for e in errs:
        if e is not None:
            raise e
    results = [o[0] for o in out]
    kinds = [type(o[1]) for o in out]
    if len(set(kinds)) != 1:
        raise RuntimeError(f"ranks disagree on the outcome: {kinds}")
    err0 = out[0][1]
    if results[0] is None:  # ZeroDiagonal: no result
        raise err0
    x = np.concatenate([r.x for r in results])
    full = SolveResult(x, results[0].iterations, results[0].converged, results[0].residual_inf,
                       time.perf_counter() - start)
    if err0 is not None:
        from .solvers import Breakdown, NotConverged
        if isinstance(err0, Breakdown):
            raise Breakdown(err0.which, err0.iteration, full)
        raise NotConverged(full)
    return full, results
