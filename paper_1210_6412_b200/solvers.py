"""Drop-in GPU solvers with the reference's interface (mcreach/solvers.py).

Every public name here mirrors ``/root/reference/pkg/src/mcreach/solvers.py``:

* ``SolverConfig`` (:81-109), ``SolveResult`` (:112-120), ``SolverError`` / ``ZeroDiagonal`` /
  ``NotConverged`` / ``Breakdown`` (:43-78) -- same fields, validation and messages;
* ``jacobi_solve`` (:194-230) and ``bicgstab_solve`` (:399-426) -- same signature
  ``fn(m, b, config=None) -> SolveResult``, same stopping rules, same exceptions, same
  ``wall_time`` region (after the right-hand-side check, through the final residual);
* ``residual_inf_norm`` (:123-133) and ``matvec`` (sparse.py:184-191);
* ``jacobi_solve_parallel`` (:233-274) / ``bicgstab_solve_parallel`` (:429-447): row shards
  over ``config.workers`` GPUs;
* ``SOLVERS`` (:494-499) with the GPU methods ``jacobi-gpu``, ``bicgstab-gpu``,
  ``bicgstab-gpu-exact``, ``jacobi-gpu-par`` and ``bicgstab-gpu-par``.

The arithmetic runs in libmcr.so (CUDA, sm_100a) behind the C ABI in include/mcr.h; the
matrix is uploaded once per ``CsrMatrix`` object and cached while that object lives, like
the reference caches its scipy handle (sparse.py:91-98). ``plugin.install()`` registers these
methods into the reference's own ``mcreach.solvers.SOLVERS``.
"""

from __future__ import annotations

import ctypes
import os
import threading
import time
import weakref
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _lib
from .sparse import DimensionMismatch

__all__ = [
    "SolverConfig", "SolveResult", "SolverError", "ZeroDiagonal", "NotConverged", "Breakdown",
    "DeviceMatrix", "device_matrix", "jacobi_solve", "bicgstab_solve", "bicgstab_solve_exact",
    "jacobi_solve_parallel", "bicgstab_solve_parallel", "parallel_devices",
    "residual_inf_norm", "matvec", "SOLVERS",
]


class SolverError(RuntimeError):
    """Base class for solver failures (solvers.py:43-44)."""


class ZeroDiagonal(SolverError):
    def __init__(self, index: int):
        super().__init__(f"zero diagonal entry in row {index}")
        self.index = index


class NotConverged(SolverError):
    def __init__(self, result: "SolveResult"):
        super().__init__(
            f"no convergence after {result.iterations} iterations "
            f"(residual sup-norm {result.residual_inf:.3e})")
        self.result = result
        self.iterations = result.iterations
        self.residual_inf = result.residual_inf


class Breakdown(SolverError):
    def __init__(self, which: str, iteration: int, result: "SolveResult"):
        super().__init__(f"breakdown: {which} vanished at iteration {iteration}")
        self.which = which
        self.iteration = iteration
        self.result = result


@dataclass(frozen=True)
class SolverConfig:
    """solvers.py:81-109, plus two GPU fields.

    ``device``: CUDA ordinal of the solve. ``dot_products``: how BiCGStab's inner products
    are summed. ``"sequential"`` (default) is the reference's own left-to-right order
    (``_dot_ascending``, solvers.py:136-141), bit for bit, computed in parallel by k_xdot
    (csrc/xdot.cuh), so x, the iteration count, the residual and breakdowns equal the
    reference's; with ``parallel_dot_products`` the row-sharded solvers sum per
    ``_row_blocks`` block and add the block results in order, as ``_ParOps.dot``
    (solvers.py:384-396). ``"tree"`` is the fastest mode: deterministic fixed-shape trees
    fused into the producing kernels -- not the reference's order, so the stopping iteration
    can differ (C2: 82 vs the reference's 79). ``"serial"`` gives the sequential bits from a
    single dependent add chain (a slow cross-check of k_xdot).
    """

    tolerance: float = 1e-10
    max_iterations: int = 10_000
    guess_seed: Optional[int] = None
    workers: Optional[int] = None
    parallel_dot_products: bool = False
    device: int = 0
    dot_products: str = "sequential"

    def __post_init__(self):
        if not self.tolerance > 0.0:
            raise ValueError("tolerance must be positive")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be at least 1")
        if self.workers is not None and self.workers < 1:
            raise ValueError("workers must be at least 1")
        if self.dot_products not in ("sequential", "tree", "serial"):
            raise ValueError("dot_products must be 'sequential', 'tree' or 'serial'")

    def resolved_workers(self) -> int:
        return self.workers if self.workers is not None else (os.cpu_count() or 1)


@dataclass(frozen=True, eq=False)
class SolveResult:
    x: np.ndarray
    iterations: int
    converged: bool
    residual_inf: float
    wall_time: float


# ----------------------------------------------------------------------------- device handle

def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class DeviceMatrix:
    """Device-resident copy of a CSR matrix (one libmcr handle)."""

    def __init__(self, m, device: int = 0, storage: int = _lib.STORAGE_AUTO, _handle=None):
        L = _lib.load()
        if _handle is None:
            n = int(m.n)
            rs = np.ascontiguousarray(m.rstart, dtype=np.int64)
            col = np.ascontiguousarray(m.col, dtype=np.int64)
            val = np.ascontiguousarray(m.nonzero, dtype=np.float64)
            h = ctypes.c_void_p()
            rc = L.mcr_matrix_create(n, _ptr(rs), _ptr(col), _ptr(val), int(device),
                                     int(storage), ctypes.byref(h))
            if rc != _lib.MCR_OK:
                _raise_native(rc)
        else:
            h = _handle
        self._h = h
        self._L = L
        self.lock = threading.Lock()
        self._finalizer = weakref.finalize(self, L.mcr_matrix_destroy, h)
        inf = self.info()
        self.n = int(inf["n"])
        self.device = int(inf["device"])

    @classmethod
    def generated(cls, n: int, mean_offdiag: float = 7.0, lo: int = 1, hi: int = 10,
                  seed: int = 0, device: int = 0, storage: int = _lib.STORAGE_AUTO,
                  comm=None) -> "DeviceMatrix":
        """Row-keyed synthetic system built in HBM (mcr_generate; config C5). With ``comm``
        (a dist.Comm) the handle holds that rank's rows only."""
        L = _lib.load()
        h = ctypes.c_void_p()
        rc = L.mcr_generate(comm.handle if comm is not None else None, int(device), int(n),
                            float(mean_offdiag), int(lo), int(hi), int(seed), int(storage),
                            ctypes.byref(h))
        if rc != _lib.MCR_OK:
            _raise_native(rc)
        return cls(None, _handle=h)

    @classmethod
    def reference_generated(cls, spec, device: int = 0, storage: int = _lib.STORAGE_AUTO):
        """``generate_dd_matrix(spec)`` (S/generator.py:100-124) drawn on the device from the
        reference's own random stream (mcr_refgen_matrix): the same arrays, straight into HBM."""
        from .generator import pcg_words
        n = int(spec.n)
        count = int(spec.target_nnz()) - n
        lo, hi = spec.value_range
        words = pcg_words(spec.seed)
        L = _lib.load()
        h = ctypes.c_void_p()
        rc = L.mcr_refgen_matrix(int(device), n, count, int(lo), int(hi), words.ctypes.data, int(storage),
                                 ctypes.byref(h))
        if rc != _lib.MCR_OK:
            _raise_native(rc)
        return cls(None, _handle=h)

    def generated_rhs(self, seed: int, out_device_ptr: int) -> None:
        rc = self._L.mcr_generate_rhs(self._h, int(seed), ctypes.c_void_p(out_device_ptr))
        if rc != _lib.MCR_OK:
            _raise_native(rc)

    def export(self):
        """Host copy of the handle's CSR: (local rstart, global col, nonzero)."""
        inf = self.info()
        rs = np.empty(int(inf["n"]) + 1, dtype=np.int64)
        col = np.empty(int(inf["nnz"]), dtype=np.int64)
        val = np.empty(int(inf["nnz"]), dtype=np.float64)
        rc = self._L.mcr_matrix_export(self._h, _ptr(rs), _ptr(col), _ptr(val))
        if rc != _lib.MCR_OK:
            _raise_native(rc)
        return rs, col, val

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    def info(self) -> dict:
        inf = _lib.MatrixInfo()
        self._L.mcr_matrix_info_get(self._h, ctypes.byref(inf))
        return {f: getattr(inf, f) for f, _ in _lib.MatrixInfo._fields_}

    def close(self) -> None:
        self._finalizer()

    def matvec(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.n)
        rc = self._L.mcr_matvec(self._h, _ptr(x), _ptr(y))
        if rc != _lib.MCR_OK:
            _raise_native(rc)
        return y

    def residual_inf(self, x, b) -> float:
        x = np.ascontiguousarray(x, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = ctypes.c_double(0.0)
        rc = self._L.mcr_residual_inf(self._h, _ptr(x), _ptr(b), ctypes.byref(out))
        if rc != _lib.MCR_OK:
            _raise_native(rc)
        return out.value

    def solve(self, method: str, b: np.ndarray, x0: Optional[np.ndarray], tol: float,
              max_it: int, dots: str = "sequential", dot_blocks: int = 1):
        fn = {"jacobi": self._L.mcr_jacobi, "bicgstab": self._L.mcr_bicgstab}[method]
        rc = self._L.mcr_set_dot_mode(self._h, _lib.DOT_MODES[dots])
        if rc == _lib.MCR_OK:
            rc = self._L.mcr_set_dot_blocks(self._h, int(dot_blocks))
        if rc != _lib.MCR_OK:
            _raise_native(rc)
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(self.n)
        x0p = None
        if x0 is not None:
            x0 = np.ascontiguousarray(x0, dtype=np.float64)
            x0p = _ptr(x0)
        rep = _lib.Report()
        rc = fn(self._h, _ptr(b), x0p, float(tol), int(max_it), _ptr(x), ctypes.byref(rep))
        return rc, x, rep


_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_cache_lock = threading.Lock()


def device_matrix(m, device: int = 0) -> DeviceMatrix:
    """Cached device copy of ``m`` (uploaded once per matrix object and device)."""
    with _cache_lock:
        per = _cache.get(m)
        if per is None:
            per = {}
            try:
                _cache[m] = per
            except TypeError:  # not weak-referenceable: no caching
                return DeviceMatrix(m, device)
        dm = per.get(device)
        if dm is None:
            dm = DeviceMatrix(m, device)
            per[device] = dm
        return dm


def _raise_native(rc: int):
    msg = _lib.last_error()
    if rc == _lib.MCR_DIMENSION:
        raise DimensionMismatch(msg)
    if rc == _lib.MCR_INVALID_ARGUMENT:
        raise ValueError(msg)
    raise _lib.NativeLibraryError(f"libmcr error {rc}: {msg}")


# ----------------------------------------------------------------------------- solvers

def _check_system(m, b) -> np.ndarray:
    """solvers.py:144-150"""
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (m.n,):
        raise DimensionMismatch(f"right-hand side of shape {b.shape} against dimension {m.n}")
    return b


def _initial_guess(n: int, cfg) -> Optional[np.ndarray]:
    """solvers.py:153-156; None means the zero vector (filled on the device)."""
    seed = getattr(cfg, "guess_seed", None)
    if seed is None:
        return None
    return np.random.default_rng(seed).random(n)


def _empty_result(start: float) -> SolveResult:
    return SolveResult(np.zeros(0), 0, True, 0.0, time.perf_counter() - start)


def _solve(method: str, m, b, config, dots: Optional[str] = None,
           device: Optional[int] = None, dot_blocks: int = 1) -> SolveResult:
    cfg = config or SolverConfig()
    b = _check_system(m, b)
    start = time.perf_counter()
    if m.n == 0:
        return _empty_result(start)
    dm = device_matrix(m, int(getattr(cfg, "device", 0) or 0) if device is None else device)
    x0 = _initial_guess(m.n, cfg)
    with dm.lock:
        rc, x, rep = dm.solve(method, b, x0, cfg.tolerance, cfg.max_iterations,
                              dots or getattr(cfg, "dot_products", "sequential"), dot_blocks)
    return finish(rc, x, rep, start)


def outcome(rc: int, x: np.ndarray, rep, start: float):
    """(SolveResult, exception or None) of a native solve; raises on library errors."""
    if rc == _lib.MCR_ZERO_DIAGONAL:
        return None, ZeroDiagonal(int(rep.zero_diagonal_index))
    if rc not in (_lib.MCR_OK, _lib.MCR_NOT_CONVERGED, _lib.MCR_BREAKDOWN):
        _raise_native(rc)
    result = SolveResult(x, int(rep.iterations), rc == _lib.MCR_OK, float(rep.residual_inf),
                         time.perf_counter() - start)
    if rc == _lib.MCR_BREAKDOWN:
        return result, Breakdown(_lib.BREAKDOWN_NAMES[int(rep.breakdown_which)],
                                 int(rep.breakdown_iteration), result)
    if rc == _lib.MCR_NOT_CONVERGED:
        return result, NotConverged(result)
    return result, None


def finish(rc: int, x: np.ndarray, rep, start: float) -> SolveResult:
    """Map a native status onto the reference's result / exceptions (solvers.py:43-78)."""
    result, err = outcome(rc, x, rep, start)
    if err is not None:
        raise err
    return result


def jacobi_solve(m, b, config: Optional[SolverConfig] = None) -> SolveResult:
    """Jacobi iteration on the GPU (solvers.py:194-230 semantics, bit-identical iterates).

    Raises ZeroDiagonal before any sweep, NotConverged after ``max_iterations`` sweeps with
    the last iterate attached.
    """
    return _solve("jacobi", m, b, config)


def bicgstab_solve(m, b, config: Optional[SolverConfig] = None) -> SolveResult:
    """Un-preconditioned BiCGStab on the GPU (solvers.py:399-491 semantics).

    Raises Breakdown (snapshot before the failing iteration) or NotConverged.
    """
    return _solve("bicgstab", m, b, config)


def bicgstab_solve_exact(m, b, config: Optional[SolverConfig] = None) -> SolveResult:
    """BiCGStab with the reference's sequential inner products: bit-identical to
    ``mcreach.bicgstab_solve`` (x, iteration count, residual, breakdowns)."""
    return _solve("bicgstab", m, b, config, dots="sequential")


def residual_inf_norm(m, x, b) -> float:
    """solvers.py:123-133 on the device."""
    x = np.asarray(x, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if x.shape != (m.n,) or b.shape != (m.n,):
        raise DimensionMismatch(f"system of dimension {m.n} with x{x.shape}, b{b.shape}")
    if m.n == 0:
        return 0.0
    dm = device_matrix(m)
    with dm.lock:
        return dm.residual_inf(x, b)


def matvec(m, x) -> np.ndarray:
    """sparse.py:184-191 on the device (bit-identical row sums)."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (m.n,):
        raise DimensionMismatch(f"vector of shape {x.shape} against dimension {m.n}")
    if m.n == 0:
        return np.zeros(0)
    dm = device_matrix(m)
    with dm.lock:
        return dm.matvec(x)


def parallel_devices(n: int, cfg) -> list:
    """Devices of a row-sharded solve: ``cfg.workers`` GPUs (default: every visible GPU),
    at most one per row, starting at ``cfg.device`` -- the GPU analogue of the reference's
    ``resolved_workers`` + ``_row_blocks`` (solvers.py:98-99,159-168). ``MCR_GPU_DEVICES``
    (comma-separated ordinals, repeats allowed) overrides the choice, e.g. ``0,0`` runs two
    shards on one GPU."""
    env = os.environ.get("MCR_GPU_DEVICES")
    if env:
        devs = [int(d) for d in env.split(",") if d.strip()]
        if not devs:
            raise ValueError("MCR_GPU_DEVICES lists no device")
        return devs[:max(1, min(len(devs), n))]
    count = _lib.device_count()
    if count < 1:
        raise _lib.NativeLibraryError("no CUDA device visible")
    workers = cfg.workers if cfg.workers is not None else count
    k = max(1, min(workers, count, n))
    dev0 = int(getattr(cfg, "device", 0) or 0)
    return [(dev0 + i) % count for i in range(k)]


def _solve_parallel(method: str, m, b, config) -> SolveResult:
    cfg = config or SolverConfig()
    b = _check_system(m, b)
    start = time.perf_counter()
    if m.n == 0:
        return _empty_result(start)
    dots = getattr(cfg, "dot_products", "sequential")
    blocks = cfg.resolved_workers() if getattr(cfg, "parallel_dot_products", False) else 1
    if method == "bicgstab" and dots == "serial":  # the one-CTA check mode: one GPU
        return _solve(method, m, b, cfg, dots=dots, dot_blocks=max(1, int(blocks)))
    # BiCGStab's inner products (solvers.py:384-396) on row shards: every rank sums the whole
    # gathered vectors left to right (one chain, or with parallel_dot_products one chain per
    # _row_blocks block of resolved_workers() blocks, combined in order) -- the same bits as
    # the reference and as one GPU (dist._solve_sharded)
    devices = parallel_devices(int(m.n), cfg)
    from .dist import shard_rows, solve_local_group
    while len(devices) > 1 and shard_rows(int(m.n), len(devices), len(devices) - 1)[1] < 1:
        devices = devices[:-1]  # ceil(n/k) blocks: every shard must hold rows
    if len(devices) == 1:
        return _solve(method, m, b, cfg, device=devices[0], dot_blocks=max(1, int(blocks)))
    result, _ = solve_local_group(method, m, b, len(devices), cfg, devices=devices)
    return SolveResult(result.x, result.iterations, result.converged, result.residual_inf,
                       time.perf_counter() - start)


def jacobi_solve_parallel(m, b, config: Optional[SolverConfig] = None) -> SolveResult:
    """Row-sharded Jacobi over ``config.workers`` GPUs (solvers.py:233-274 semantics): one
    contiguous row block per GPU, the iterate exchanged every sweep, the stop test decided
    identically on every shard. Iterates are bit-identical to ``jacobi_solve``, as the
    reference's row-block variant is to its sequential one."""
    return _solve_parallel("jacobi", m, b, config)


def bicgstab_solve_parallel(m, b, config: Optional[SolverConfig] = None) -> SolveResult:
    """solvers.py:429-447. With the reference's dots (default) the result is the reference's
    ``bicgstab_solve_parallel`` bit for bit -- sequential inner products, or per-block ones
    when ``parallel_dot_products`` is set (blocks = ``resolved_workers()``, as the reference)
    -- computed on one GPU. With ``dot_products="tree"`` the rows shard over
    ``config.workers`` GPUs: p and s exchanged before each product, every inner product
    reduced per shard and summed in ascending shard order, identically on all shards."""
    return _solve_parallel("bicgstab", m, b, config)


SOLVERS: dict[str, Callable[..., SolveResult]] = {
    "jacobi-gpu": jacobi_solve,
    "bicgstab-gpu": bicgstab_solve,
    "bicgstab-gpu-exact": bicgstab_solve_exact,
    "jacobi-gpu-par": jacobi_solve_parallel,
    "bicgstab-gpu-par": bicgstab_solve_parallel,
}
