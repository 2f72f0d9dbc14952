"""Benchmark: time-to-solution of the reachability linear solve (Jacobi + BiCGStab) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

Workload (BASELINE.json configs[1], "C2"): the reference generator's strictly diagonally
dominant system n = 1e6, nnz = 1e7 (GenSpec(n=10**6, nnz=10**7, seed=trial_seed(0, 1e6,
None, 1e7, 0)), bit-identical to mcreach.generate_dd_matrix) with rhs generate_rhs(n, seed).
One step = one Jacobi solve + one BiCGStab solve from x0 = 0 to tol 1e-10, each including
its final true residual. Metric value = solves per second over the whole job (N replicas at
N > 1 the system's rows shard over the N GPUs: strong scaling of one solve, run_sharded).

Our arm: inputs resident in HBM (device-pointer C ABI), L2 flushed (512 MiB write) before
every step, CUDA events on the stream the library launches on, barrier + synchronize around
the timed loop, max over ranks. `e2e` repeats the step through the public API with HOST
buffers (pinned): matrix upload + both solves + x back to the host, every step.
`roofline` is the dominant kernel (the CSR SpMV tile kernel, k_spmv) timed alone with CUDA
events (L2 flushed between launches) against its algorithmic bytes 12*nnz + 8*(n+1) + 16*n.
`cpu_baseline` times the reference's own CPU path (mcreach jacobi-par + bicgstab-par,
workers = all host cores) on one full solve pair, falling back to the C oracle port.
`--impl reference` times the reference's CPU path alone, same metric and unit.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-solution & SpMV HBM GB/s (Jacobi/BiCGStab) at 1/2/4/8 B200 vs CPU"
UNIT = "solves/s"
STORAGES = {"auto": 0, "tiles": 5, "staged": 6}  # C5 layouts (include/mcr.h MCR_STORAGE_*)
FALLBACK_HBM_GBS = 6650.0


# ----------------------------------------------------------------------------- workload

def make_workload(config: str):
    from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix, generate_rhs, trial_seed
    if config == "c2":
        n, nnz = 10 ** 6, 10 ** 7
        seed = trial_seed(0, n, None, nnz, 0)
        spec = GenSpec(n=n, nnz=nnz, seed=seed)
        desc = ("C2: reference-generator DD system n=1e6, nnz=1e7 "
                "(GenSpec(n=10**6, nnz=10**7, seed=trial_seed(0,1e6,None,1e7,0)))")
    elif config == "c1":
        n = 2000
        seed = trial_seed(0, n, 0.1, None, 0)
        spec = GenSpec(n=n, density=0.1, seed=seed)
        desc = "C1: reference-generator DD system n=2000, density 0.1"
    elif config == "c3":
        n, seed = 16384, 3
        spec = GenSpec(n=n, density=1.0, seed=seed)
        desc = "C3: dense DD system n=16384 (dense slab storage)"
    else:
        raise SystemExit(f"unknown config {config}")
    m = generate_dd_matrix(spec)
    b = generate_rhs(spec.n, spec.seed)
    return m, b, desc, spec


def alg_bytes(n: int, nnz: int, nnz_off: int) -> dict:
    """f64 values, int32 columns, int64 row pointers, x gathered once."""
    spmv = 12 * nnz + 8 * (n + 1) + 16 * n
    return {"spmv": spmv,
            "jacobi_sweep": 12 * nnz_off + 8 * (n + 1) + 32 * n,
            "bicgstab_iteration": 2 * (12 * nnz + 8 * (n + 1)) + 152 * n}


def load_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def load_traffic(kernel_key: str, prefix: str = "c2"):
    """DRAM bytes per launch of `kernel_key` from the newest committed ncu summary
    (profiles/rNN_<prefix>_ncu.json, one `ncu --set full` capture)."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_{prefix}_ncu.json")),
                       reverse=True):
        try:
            with open(path) as fh:
                return json.load(fh)["kernels"][kernel_key]["dram_bytes_per_launch"]
        except Exception:
            continue
    return None


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """Samples SM clock + throttle reasons with NVML while the timed region runs."""

    def __init__(self, index: int):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            pass

    _NAMES = {0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
              0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
              0x80: "hw_power_brake_slowdown"}

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self._NAMES.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self._ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._ok:
            self._t.join(timeout=1)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU legs

def reference_module():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "mcreach")) and ref not in sys.path:
        sys.path.append(ref)
    try:
        import mcreach  # noqa: F401
        from mcreach import solvers as ms
        return ms
    except Exception:
        return None


def cpu_solve_pair(m, b, threads: int, jacobi_cap: int = 0):
    """One Jacobi + BiCGStab solve pair of the reference's CPU path. Returns (seconds, kind,
    iterations, note). kind 'reference' = mcreach itself (baseline/_ref), 'port' = the C
    restatement in oracle/ (when the reference is not installed). Solver failures are timed
    like successes (bench.py:184-187 records them in-row). jacobi_cap > 0 bounds the sample:
    Jacobi runs `jacobi_cap` sweeps and its time is scaled to the 10 000-sweep budget (C3,
    where the reference's Jacobi never converges)."""
    ms = reference_module()
    budget = 10_000
    if ms is not None:
        from mcreach import CsrMatrix as RefCsr
        rm = RefCsr(m.n, m.rstart, m.col, m.nonzero)

        def run(name, max_it):
            cfg = ms.SolverConfig(workers=threads, max_iterations=max_it)
            t0 = time.perf_counter()
            try:
                r = ms.SOLVERS[name](rm, b, cfg)
                it = r.iterations
            except ms.SolverError as err:
                it = getattr(getattr(err, "result", None), "iterations", max_it)
            return time.perf_counter() - t0, it
        kind = "reference"
    else:
        from oracle import oracle
        oracle.set_threads(threads)

        def run(name, max_it):
            t0 = time.perf_counter()
            r = (oracle.jacobi if name.startswith("jacobi") else oracle.bicgstab)(
                m, b, max_iterations=max_it)
            return time.perf_counter() - t0, r["iterations"]
        kind = "port"
    if jacobi_cap:
        tj, ij = run("jacobi-par", jacobi_cap)
        tj *= budget / jacobi_cap
        ij = budget
        note = f"jacobi {jacobi_cap} sweeps timed, scaled to the {budget}-sweep budget"
    else:
        tj, ij = run("jacobi-par", budget)
        note = "full solves"
    tb, ib = run("bicgstab-par", budget)
    return tj + tb, kind, (ij, ib), note


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    m, b, desc, spec = make_workload(args.config)
    threads = os.cpu_count() or 1
    times = []
    kind = None
    iters = None
    for i in range(args.warmup + args.steps):
        dt, kind, iters, note = cpu_solve_pair(m, b, threads, 25 if args.config == "c3" else 0)
        if i >= args.warmup:
            times.append(dt)
    total = sum(times)
    value = 2 * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference generator, bit-identical inputs",
        "config": {"workload": desc, "n": spec.n, "nnz": int(m.m), "tolerance": 1e-10,
                   "solve_pair": "jacobi-par + bicgstab-par", "parallelism": "cpu threads"},
        "iterations": {"jacobi": iters[0], "bicgstab": iters[1]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{args.config.upper()} solve pair per step ({note}; {'mcreach' if kind == 'reference' else 'oracle C port'}, {threads} threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm

def _drop_in(fn, m, b, cfg):
    """One registry call; a capped solve (C3's Jacobi) raises NotConverged carrying its result,
    as the reference does (S/solvers.py:174-179)."""
    try:
        return fn(m, b, cfg)
    except Exception as err:  # the reference's or this package's NotConverged
        if type(err).__name__ == "NotConverged" and getattr(err, "result", None) is not None:
            return err.result
        raise


def run_ours(args):
    import ctypes

    import numpy as np
    import torch

    from paper_1210_6412_b200 import _lib
    from paper_1210_6412_b200.solvers import DeviceMatrix
    from paper_1210_6412_b200.sparse import CsrMatrix

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    L = _lib.load()

    m, b, desc, spec = make_workload(args.config)
    n, nnz = int(m.n), int(m.m)
    nnz_off = nnz - int(np.count_nonzero(np.repeat(np.arange(n), np.diff(m.rstart)) == m.col))
    ab = alg_bytes(n, nnz, nnz_off)
    stream = torch.cuda.Stream(dev)  # a real stream: the legacy default stream (0) cannot be handed over
    torch.cuda.set_stream(stream)

    dm = DeviceMatrix(m, local)
    L.mcr_set_stream(dm.handle, ctypes.c_void_p(stream.cuda_stream))
    L.mcr_set_dot_mode(dm.handle, _lib.DOT_MODES[args.dots])
    b_dev = torch.from_numpy(b).to(dev)
    x_dev = torch.empty(n, dtype=torch.float64, device=dev)
    y_dev = torch.empty(n, dtype=torch.float64, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)

    def solve(fn):
        rep = _lib.Report()
        rc = fn(dm.handle, ctypes.c_void_p(b_dev.data_ptr()), None, 1e-10, 10_000,
                ctypes.c_void_p(x_dev.data_ptr()), ctypes.byref(rep))
        if rc not in (_lib.MCR_OK, _lib.MCR_NOT_CONVERGED):
            raise RuntimeError(f"solve failed rc={rc}: {_lib.last_error()}")
        return rep

    def step():
        rj = solve(L.mcr_jacobi_device)
        rb = solve(L.mcr_bicgstab_device)
        return rj, rb

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms, jac_ms, bic_ms = [], [], []
    launches = 0
    reps = None
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rj, rb = step()
            e1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            jac_ms.append(rj.device_seconds * 1e3)
            bic_ms.append(rb.device_seconds * 1e3)
            launches += rj.kernel_launches + rb.kernel_launches
            reps = (rj, rb)
    torch.cuda.synchronize()
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    value = 2.0 * world * args.steps / (total_ms / 1e3)

    # ---- the opt-in tree-dot BiCGStab on the same handle (not the reference's order)
    other = None
    if args.dots != "tree":
        L.mcr_set_dot_mode(dm.handle, _lib.DOTS_TREE)
        tms, trep = [], None
        for i in range(args.warmup + 3):
            flush.zero_()
            trep = solve(L.mcr_bicgstab_device)
            if i >= args.warmup:
                tms.append(trep.device_seconds * 1e3)
        L.mcr_set_dot_mode(dm.handle, _lib.DOT_MODES[args.dots])
        other = {"dots": "tree (fused fixed-shape trees; not the reference's summation order)",
                 "bicgstab_ms": statistics.median(tms), "bicgstab_iterations": int(trep.iterations),
                 "step_ms_estimate": statistics.median(jac_ms) + statistics.median(tms)}

    # ---- dominant kernel alone: CSR SpMV (k_spmv) with CUDA events, L2 flushed
    spmv_ms = []
    xin = torch.rand(n, dtype=torch.float64, device=dev)
    for i in range(args.warmup + max(args.steps, 10)):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        L.mcr_matvec_device(dm.handle, ctypes.c_void_p(xin.data_ptr()),
                            ctypes.c_void_p(y_dev.data_ptr()))
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= args.warmup:
            spmv_ms.append(e0.elapsed_time(e1))
    spmv_s = statistics.mean(spmv_ms) / 1e3
    peak, peak_src = load_peak()
    dense = dm.info()["storage"] == _lib.STORAGE_DENSE
    if dense:  # dense GEMV 8n^2 + 16n, Jacobi 8n^2 + 32n, BiCGStab 16n^2 + 152n
        ab = {"spmv": 8 * n * n + 16 * n, "jacobi_sweep": 8 * n * n + 32 * n,
              "bicgstab_iteration": 16 * n * n + 152 * n}
    # Roofline of the step's top kernel -- the fused Jacobi sweep (k_spmv<EPI_JACOBI>, 42% of
    # the step in the ncu launch list, profiles/) -- measured INSIDE the timed region: the
    # Jacobi solve's CUDA-event time covers its sweeps plus one full-matrix residual SpMV,
    # so achieved = (sweeps * B_jacobi + B_spmv) / that time.
    kernel = "k_dense<EPI_JACOBI>" if dense else "k_spmv<EPI_JACOBI>"
    jac_it0 = int(reps[0].iterations)
    jac_s = statistics.median(jac_ms) / 1e3
    achieved = (ab["jacobi_sweep"] * jac_it0 + ab["spmv"]) / jac_s / 1e9
    sweep_us = 1e6 * jac_s / (jac_it0 + 1)
    traffic = load_traffic(kernel, {"c2": "c2", "c3": "c3dense"}.get(args.config, "none"))
    spmv_alone = {"kernel": ("k_dense<EPI_Y>" if dense else "k_spmv<EPI_Y>"),
                  "launch_us": spmv_s * 1e6, "algorithmic_bytes": ab["spmv"],
                  "achieved_gbs": ab["spmv"] / spmv_s / 1e9,
                  "frac": ab["spmv"] / spmv_s / 1e9 / peak,
                  "how": "one M x launch, L2 flushed (512 MiB write) before each, CUDA events"}

    # ---- end to end through the drop-in: the reference's registry with the GPU methods
    # installed (plugin.install()), a fresh reference CsrMatrix over pageable numpy arrays every
    # step (so every step uploads the matrix), b from the host, x back to the host: exactly
    # what `SOLVERS["jacobi-gpu"](m, b)` costs a reference caller
    from paper_1210_6412_b200 import plugin
    from paper_1210_6412_b200 import solvers as gsolvers
    ms = reference_module()
    if ms is not None:
        from mcreach import CsrMatrix as RefCsr
        reg = dict(ms.SOLVERS)
        plugin.install(reg)
        make_csr = RefCsr
        via = "mcreach.solvers.SOLVERS with plugin.install() (reference CsrMatrix, pageable numpy)"
    else:
        reg = gsolvers.SOLVERS
        make_csr = CsrMatrix
        via = "paper_1210_6412_b200.solvers.SOLVERS (no mcreach importable; pageable numpy)"
    gcfg = gsolvers.SolverConfig(dot_products=args.dots, device=local)
    rs_p, col_p, val_p, b_p = (np.array(m.rstart), np.array(m.col), np.array(m.nonzero), np.array(b))
    e2e_s = []
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mat = make_csr(n, rs_p, col_p, val_p)        # a new object: the drop-in uploads it
        rj_e = _drop_in(reg["jacobi-gpu"], mat, b_p, gcfg)
        rb_e = _drop_in(reg["bicgstab-gpu"], mat, b_p, gcfg)
        del mat
        gsolvers._cache.clear()                       # release the device copy every step
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_s.append(time.perf_counter() - t0)
    e2e_total = sum(e2e_s)
    if dist:
        t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = 2.0 * world * args.steps / e2e_total
    e2e_iters = {"jacobi": int(rj_e.iterations), "bicgstab": int(rb_e.iterations)}
    h2d = 8 * (n + 1) + 8 * nnz + 4 * nnz + 2 * 8 * n  # columns cross PCIe as int32 (narrowed on the host)
    d2h = 2 * 8 * n

    # the same through the device handle API with pinned host buffers (sub-record)
    def pinned(a):
        t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        return t, t.numpy()

    _rs_t, rs_h = pinned(m.rstart)
    _col_t, col_h = pinned(m.col)
    _val_t, val_h = pinned(m.nonzero)
    _b_t, b_h = pinned(b)
    _x_t, x_h = pinned(np.zeros(n))
    hm = CsrMatrix(n, rs_h, col_h, val_h)
    pin_s = []
    for i in range(1 + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = DeviceMatrix(hm, local)             # H2D: rowptr, col, val
        L.mcr_set_dot_mode(h.handle, _lib.DOT_MODES[args.dots])
        for method in ("jacobi", "bicgstab"):   # H2D: b; D2H: x
            fn = L.mcr_jacobi if method == "jacobi" else L.mcr_bicgstab
            rep = _lib.Report()
            rc = fn(h.handle, ctypes.c_void_p(b_h.ctypes.data), None, 1e-10, 10_000,
                    ctypes.c_void_p(x_h.ctypes.data), ctypes.byref(rep))
            assert rc in (_lib.MCR_OK, _lib.MCR_NOT_CONVERGED), _lib.last_error()
        h.close()
        torch.cuda.synchronize()
        if i >= 1:
            pin_s.append(time.perf_counter() - t0)
    e2e_pinned = 2.0 * world * len(pin_s) / sum(pin_s)

    # ---- CPU baseline (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        dt, kind, iters, note = cpu_solve_pair(m, b, threads, 25 if args.config == "c3" else 0)
        cpu = {"value": 2.0 / dt, "unit": UNIT, "cores": threads, "kind": kind,
               "sample": f"one {args.config.upper()} solve pair (jacobi {iters[0]} sweeps + "
                         f"bicgstab {iters[1]} iterations; {note}) by "
                         f"{'mcreach jacobi-par/bicgstab-par' if kind == 'reference' else 'the oracle C port'}, "
                         f"{threads} threads, {dt:.1f} s"}

    rj, rb = reps
    jac_it, bic_it = int(rj.iterations), int(rb.iterations)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference generator (bit-identical to mcreach.generate_dd_matrix)",
        "config": {"workload": desc, "n": n, "nnz": nnz, "tolerance": 1e-10,
                   "solve_pair": ("jacobi + bicgstab from x0=0, BiCGStab inner products in "
                                  + {"sequential": "the reference's left-to-right order (k_xdot)",
                                     "serial": "the reference's order (one add chain)",
                                     "tree": "fused trees (not the reference's order)"}[args.dots]),
                   "dots": args.dots,
                   "l2": "flushed before every step (512 MiB write); SpMV working set 144 MB",
                   "parallelism": f"replicas x{world}"},
        "time_to_solution_ms": {"jacobi": statistics.median(jac_ms),
                                "bicgstab": statistics.median(bic_ms)},
        "iterations": {"jacobi": jac_it, "bicgstab": bic_it},
        "per_iteration": {
            "jacobi_sweep_us": 1e3 * statistics.median(jac_ms) / max(jac_it, 1),
            "jacobi_sweep_gbs": ab["jacobi_sweep"] * jac_it / (statistics.median(jac_ms) / 1e3) / 1e9,
            "bicgstab_iteration_us": 1e3 * statistics.median(bic_ms) / max(bic_it, 1),
            "bicgstab_iteration_gbs": ab["bicgstab_iteration"] * bic_it / (statistics.median(bic_ms) / 1e3) / 1e9,
        },
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": kernel + " (fused Jacobi sweep; timed inside the step)",
                     "algorithmic_bytes": ab["jacobi_sweep"], "launch_us": sweep_us,
                     "peak_source": peak_src,
                     "bound_note": ("gather-bound: 1 random 8-byte x gather per entry; the "
                                    "measured B200 gather floor for C2's 1e7 gathers is "
                                    "~52 us (profiles/r01_gather_microbench.txt). The largest "
                                    "single kernel of the step (21% under ncu, profiles/r02_c2_launches.txt); "
                                    "the reference-order dots (k_xdot, 3 launches per BiCGStab "
                                    "iteration) take 35% together and are bound by dependent adds "
                                    "and integer work, not memory (16 B read per product): "
                                    "DESIGN.md 2.1"),
                     "spmv_alone": spmv_alone},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "iterations": e2e_iters,
                "note": f"drop-in per step: {via}: fresh matrix object (upload), jacobi-gpu + bicgstab-gpu, x to the host",
                "pinned_device_api": {"value": e2e_pinned, "unit": UNIT,
                                      "note": "DeviceMatrix from pinned arrays + mcr_jacobi + mcr_bicgstab + destroy"}},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if other:
        line["tree_dots"] = other
    if cpu:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- C5 (sharded)

def c5_cpu_proxy(threads: int, n_proxy: int, sweeps: int, n_full: int, iters: dict):
    """The reference path cannot build C5 (n = 2e8; its generator needs ~141 B/nnz of host
    RAM). Bounded sample: the oracle's Jacobi sweep (the reference's operation
    order, all host threads) on an n_proxy-row system of the same family, `sweeps` sweeps,
    scaled linearly to n_full rows and to the GPU run's iteration counts."""
    from oracle import oracle
    oracle.set_threads(threads)
    m = oracle.generate(2024, n_proxy, 7.0)
    b = oracle.generate_rhs(2024, n_proxy)
    t0 = time.perf_counter()
    oracle.jacobi(m, b, max_iterations=sweeps)
    per_sweep = (time.perf_counter() - t0) / sweeps * (n_full / n_proxy)
    # one BiCGStab iteration ~ 2 SpMV + vector work ~ 2.5 Jacobi sweeps (SURVEY 6 ratios)
    pair = per_sweep * iters["jacobi"] + 2.5 * per_sweep * iters["bicgstab"]
    return 2.0 / pair, (f"oracle Jacobi, {sweeps} sweeps on an n={n_proxy:.0e} system of the C5 "
                        f"family ({threads} threads), per-sweep time scaled x{n_full / n_proxy:.0f} "
                        f"to n={n_full:.0e} and to the GPU iteration counts "
                        f"({iters['jacobi']} sweeps + {iters['bicgstab']} BiCGStab iterations "
                        f"at 2.5 sweeps each): extrapolated, not run")


def c5_traffic(storage, n):
    """DRAM bytes of one C5 SpMV from the committed ncu capture (profiles/r01_c5_staged_ncu.json:
    both staged passes, n = 2e8), or None for another size or the tiled layout."""
    from paper_1210_6412_b200 import _lib
    if storage != _lib.STORAGE_STAGED or n != 2 * 10 ** 8:
        return None
    a = load_traffic("k_stage_products<0>", "c5_staged")
    b = load_traffic("k_spmv_staged<0>", "c5_staged")
    return a + b if a is not None and b is not None else None


def run_c5(args):
    import ctypes

    import torch

    from paper_1210_6412_b200 import _lib
    from paper_1210_6412_b200.dist import Comm, ShardMatrix
    from paper_1210_6412_b200.solvers import DeviceMatrix

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    L = _lib.load()
    n, mean, seed = args.n, 7.0, 2024
    t_gen = time.perf_counter()
    refgen = world == 1 and args.gen == "reference"
    if world > 1:
        comm = Comm.nccl(local)
        h = ShardMatrix.generated(comm, n, mean, 1, 10, seed, storage=STORAGES[args.storage])
        if args.p2p:
            h.enable_p2p()
    elif refgen:  # the reference's generator and random stream (GenSpec(n, nnz=8n), trial 0)
        from paper_1210_6412_b200.generator import GenSpec, generate_rhs_device, trial_seed
        comm = None
        seed = trial_seed(0, n, None, 8 * n, 0)
        h = DeviceMatrix.reference_generated(GenSpec(n=n, nnz=8 * n, seed=seed), device=local,
                                             storage=STORAGES[args.storage])
    else:
        comm = None
        h = DeviceMatrix.generated(n, mean, 1, 10, seed, device=local, storage=STORAGES[args.storage])
    info = h.info()
    rows, nnz_local = int(info["n"]), int(info["nnz"])
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    L.mcr_set_stream(h.handle, ctypes.c_void_p(stream.cuda_stream))
    if world == 1:
        L.mcr_set_dot_mode(h.handle, _lib.DOT_MODES[args.dots])
    b = torch.empty(rows, dtype=torch.float64, device=dev)
    if refgen:
        b.copy_(torch.from_numpy(generate_rhs_device(n, seed, local)))
    else:
        h.generated_rhs(seed, b.data_ptr())
    x = torch.empty(rows, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    nnz = torch.tensor([nnz_local], dtype=torch.int64, device=dev)
    if dist:
        dist.all_reduce(nnz)
    nnz = int(nnz.item())

    def solve(fn):
        rep = _lib.Report()
        rc = fn(h.handle, ctypes.c_void_p(b.data_ptr()), None, 1e-10, 10_000,
                ctypes.c_void_p(x.data_ptr()), ctypes.byref(rep))
        if rc not in (_lib.MCR_OK, _lib.MCR_NOT_CONVERGED):
            raise RuntimeError(f"solve failed rc={rc}: {_lib.last_error()}")
        return rep

    def step():
        return solve(L.mcr_jacobi_device), solve(L.mcr_bicgstab_device)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms, launches, reps = [], 0, None
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rj, rb = step()
            e1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            launches += rj.kernel_launches + rb.kernel_launches
            reps = (rj, rb)
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = 2.0 * args.steps / (total_ms / 1e3)   # solves of the ONE sharded system per second

    # SpMV of this rank's rows against the full x (k_spmv<EPI_Y>), L2 is far smaller than x
    xin = torch.rand(-(-n // world) * world, dtype=torch.float64, device=dev)
    y = torch.empty(rows, dtype=torch.float64, device=dev)
    sp = []
    for i in range(3 + 5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        L.mcr_matvec_device(h.handle, ctypes.c_void_p(xin.data_ptr()), ctypes.c_void_p(y.data_ptr()))
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= 3:
            sp.append(e0.elapsed_time(e1))
    spmv_s = statistics.mean(sp) / 1e3
    alg = 12 * nnz_local + 8 * (rows + 1) + 8 * rows + 8 * rows  # local rows; x read once per own row
    peak, peak_src = load_peak()
    achieved = alg / spmv_s / 1e9

    # e2e through the public host-pointer C ABI: b from pinned host memory, x back to host
    bh = torch.empty(rows, dtype=torch.float64).pin_memory()
    bh.copy_(b.cpu())
    xh = torch.empty(rows, dtype=torch.float64).pin_memory()
    e2e = []
    for i in range(1 + max(1, args.steps // 2)):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for fn in (L.mcr_jacobi, L.mcr_bicgstab):
            rep = _lib.Report()
            rc = fn(h.handle, ctypes.c_void_p(bh.data_ptr()), None, 1e-10, 10_000,
                    ctypes.c_void_p(xh.data_ptr()), ctypes.byref(rep))
            assert rc in (_lib.MCR_OK, _lib.MCR_NOT_CONVERGED), _lib.last_error()
        if i >= 1:
            e2e.append(time.perf_counter() - t0)
    e2e_total = sum(e2e)
    if dist:
        t = torch.tensor([e2e_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = 2.0 * len(e2e) / e2e_total

    rj, rb = reps
    iters = {"jacobi": int(rj.iterations), "bicgstab": int(rb.iterations)}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, sample = c5_cpu_proxy(threads, 2 * 10 ** 6, 5, n, iters)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic: the reference's generate_dd_matrix / generate_rhs drawn on the device from "
                 "numpy's default_rng stream (mcr_refgen_matrix; the same arrays the reference would build)"
                 if refgen else "synthetic: row-keyed device generator of the reference's DD family (C5)"),
        "config": {"workload": (f"C5: GenSpec(n={n}, nnz={8 * n}, seed=trial_seed(0, n, None, nnz, 0))"
                                if refgen else
                                f"C5: n={n}, ~8 nnz/row (1 + Poisson(7)), row-sharded over {world} GPU(s)"),
                   "n": n, "nnz": nnz, "tolerance": 1e-10,
                   "solve_pair": ("jacobi + bicgstab from x0=0, BiCGStab dots: "
                                  + (args.dots if world == 1 else "tree (rank-order)")),
                   "l2": "inputs (x 1.6 GB, matrix ~19 GB) far larger than L2",
                   "parallelism": (f"row shards x{world} ("
                                   + ("fused P2P stores + NCCL slot exchange" if args.p2p and world > 1
                                      else "NCCL allgather + rank-order reductions") + ")"),
                   "generation_s": t_gen},
        "iterations": iters,
        "time_to_solution_ms": {"jacobi": rj.device_seconds * 1e3, "bicgstab": rb.device_seconds * 1e3},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": c5_traffic(info["storage"], n),
                     "kernel": ("k_stage_products + k_spmv_staged (band-staged SpMV, both passes)"
                                if info["storage"] == _lib.STORAGE_STAGED else "k_spmv<EPI_Y>")
                               + " on this rank's rows",
                     "storage": {0: "auto", 4: "tiles", 5: "tiles", 6: "staged"}.get(info["storage"], str(info["storage"])),
                     "algorithmic_bytes": alg, "launch_us": spmv_s * 1e6, "peak_source": peak_src},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * 8 * rows,
                "d2h_bytes_per_step": 2 * 8 * rows,
                "note": "mcr_jacobi + mcr_bicgstab with pinned host b / x; matrix generated in HBM"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


# ----------------------------------------------------------------------------- N > 1: row shards

def run_sharded(args):
    """N GPUs on ONE system: the C1/C2/C3 system's rows split contiguously over N shards
    (the reference's _row_blocks up to +-1 row), Jacobi bit-identical to one GPU,
    BiCGStab with the reference's dot order (every shard sums the gathered vectors; --dots tree:
    per-rank trees combined in rank order).
    Under torchrun (WORLD_SIZE = N) one process per GPU with NCCL; otherwise one process
    drives N shards as threads (devices from MCR_GPU_DEVICES, e.g. 0,0 puts two shards on one
    GPU, else 0..N-1) with the in-process transport. Strong scaling: value = solves of the one
    system per second, timed per rank with CUDA events, max over ranks."""
    import ctypes

    import numpy as np
    import torch

    from paper_1210_6412_b200 import _lib
    from paper_1210_6412_b200.dist import Comm, ShardMatrix

    world = args.gpus
    env_world = int(os.environ.get("WORLD_SIZE", "1"))
    torchrun = env_world > 1
    m, b, desc, spec = make_workload(args.config)
    n, nnz = int(m.n), int(m.m)
    L = _lib.load()
    if torchrun:
        rank, local = int(os.environ["RANK"]), int(os.environ.get("LOCAL_RANK", "0"))
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comms = {rank: Comm.nccl(local)}
        devices = {rank: local}
        ranks = [rank]
        transport = "NCCL (one process per GPU)"
    else:
        tdist = None
        env = os.environ.get("MCR_GPU_DEVICES")
        devs = [int(d) for d in env.split(",")] if env else list(range(world))
        if len(devs) < world:
            raise SystemExit(f"--gpus {world} needs {world} devices (MCR_GPU_DEVICES={env})")
        devs = devs[:world]
        cl = Comm.local_group(world, devs)
        comms = dict(enumerate(cl))
        devices = dict(enumerate(devs))
        ranks = list(range(world))
        transport = f"in-process group on devices {devs}"
    res = {}
    errors = []

    def run_rank(r):
        try:
            torch.cuda.set_device(devices[r])
            dev = torch.device("cuda", devices[r])
            sh = ShardMatrix.from_matrix(comms[r], m)
            stream = torch.cuda.Stream(dev)
            sh.set_stream(stream.cuda_stream)
            sh.set_dots("tree" if args.dots == "tree" else "sequential")
            bl = torch.from_numpy(np.ascontiguousarray(b[sh.row0:sh.row0 + sh.n])).to(dev)
            xl = torch.empty(sh.n, dtype=torch.float64, device=dev)

            def step():
                out = []
                for method in ("jacobi", "bicgstab"):
                    rc, rep = sh.solve_device(method, bl.data_ptr(), None, 1e-10, 10_000, xl.data_ptr())
                    if rc not in (_lib.MCR_OK, _lib.MCR_NOT_CONVERGED):
                        raise RuntimeError(f"rank {r}: {method} rc={rc}: {_lib.last_error()}")
                    out.append(rep)
                return out

            with torch.cuda.stream(stream):
                for _ in range(args.warmup):
                    step()
                torch.cuda.synchronize(dev)
                ms_, reps_ = [], None
                for _ in range(args.steps):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    reps_ = step()
                    e1.record(stream)
                    torch.cuda.synchronize(dev)
                    ms_.append(e0.elapsed_time(e1))
                # end to end: host slice of b in, host slice of x out, every step
                e2e = []
                for i in range(1 + args.steps):
                    t0 = time.perf_counter()
                    for method in ("jacobi", "bicgstab"):
                        rc, _x, _rep = sh.solve(method, b[sh.row0:sh.row0 + sh.n], None, 1e-10, 10_000)
                    if i >= 1:
                        e2e.append(time.perf_counter() - t0)
            res[r] = {"ms": sum(ms_), "reps": reps_, "e2e": sum(e2e), "rows": sh.n,
                      "nnz": int(sh.info()["nnz"]), "launches": sum(int(x.kernel_launches) for x in reps_)}
            sh.close()
        except BaseException as e:  # noqa: BLE001
            errors.append(e)

    with ClockSampler(devices[ranks[0]]) as clocks:
        if torchrun:
            tdist.barrier()
            run_rank(ranks[0])
        else:
            ts = [threading.Thread(target=run_rank, args=(r,)) for r in ranks]
            for t in ts:
                t.start()
            for t in ts:
                t.join()
    for c in comms.values():
        c.close()
    if errors:
        raise errors[0]
    total_ms = max(v["ms"] for v in res.values())
    e2e_total = max(v["e2e"] for v in res.values())
    if torchrun:
        t = torch.tensor([total_ms, e2e_total], dtype=torch.float64, device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        total_ms, e2e_total = float(t[0].item()), float(t[1].item())
    r0 = res[ranks[0]]
    rj, rb = r0["reps"]
    rank0 = int(os.environ.get("RANK", "0")) if torchrun else 0
    line = {
        "metric": METRIC, "value": 2.0 * args.steps / (total_ms / 1e3), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference generator (bit-identical to mcreach.generate_dd_matrix)",
        "config": {"workload": desc + f", rows sharded over {world} GPU(s)", "n": n, "nnz": nnz,
                   "tolerance": 1e-10,
                   "solve_pair": ("jacobi + bicgstab from x0=0, both bit-identical to one GPU and the "
                                  "reference (BiCGStab dots: every shard sums the gathered vectors in the "
                                  "reference's order)" if args.dots != "tree" else
                                  "jacobi (bit-identical) + bicgstab (tree dots, rank-order) from x0=0"),
                   "l2": "inputs resident in HBM",
                   "parallelism": f"row shards x{world}: allgather of the iterate / p / s + "
                                  f"rank-order scalar exchange; {transport}"},
        "iterations": {"jacobi": int(rj.iterations), "bicgstab": int(rb.iterations)},
        "time_to_solution_ms": {"jacobi": rj.device_seconds * 1e3, "bicgstab": rb.device_seconds * 1e3},
        "per_rank": {str(r): {"rows": v["rows"], "nnz": v["nnz"], "ms_per_step": v["ms"] / args.steps}
                     for r, v in sorted(res.items())},
        "e2e": {"value": 2.0 * args.steps / e2e_total, "unit": UNIT,
                "h2d_bytes_per_step": 2 * 8 * n, "d2h_bytes_per_step": 2 * 8 * n,
                "note": "per rank: host slice of b in, host slice of x out (mcr_jacobi / mcr_bicgstab on the shard)"},
        "gpu_launches": r0["launches"],
        "clocks": clocks.summary(),
    }
    if rank0 == 0:
        print(json.dumps(line), flush=True)
    if tdist:
        tdist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c5"])
    ap.add_argument("--n", type=int, default=2 * 10 ** 8, help="C5 dimension")
    ap.add_argument("--gen", default="reference", choices=["reference", "rowkeyed"],
                    help="C5 inputs on one GPU: the reference's generator and stream (default) or the "
                         "row-keyed shard generator (always used at N > 1)")
    ap.add_argument("--p2p", action="store_true",
                    help="C5 at N > 1: fused exchange (producers store into peers' copies)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--storage", default="auto", choices=sorted(STORAGES),
                    help="C5 layout: auto (band-staged at this size), tiles or staged")
    ap.add_argument("--dots", default="sequential", choices=["sequential", "tree", "serial"],
                    help="BiCGStab inner products: the reference's order (default) or fused trees")
    args = ap.parse_args()
    env_world = int(os.environ.get("WORLD_SIZE", "1"))
    if env_world > 1 and env_world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={env_world}")
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.config == "c5":
        if args.gpus > 1 and env_world == 1:
            raise SystemExit("--config c5 at --gpus > 1 runs under torchrun (one process per GPU)")
        return run_c5(args)
    if args.gpus > 1:
        return run_sharded(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
