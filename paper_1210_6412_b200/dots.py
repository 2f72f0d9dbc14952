"""The reference's inner products on the GPU, stand-alone.

``dot_ascending(u, v)`` is ``_dot_ascending`` (solvers.py:136-141, ``np.cumsum(u * v)[-1]``)
and ``dot_blocks(u, v, k)`` is ``_ParOps.dot`` with ``parallel_dot_products`` (solvers.py:
384-396: each ``_row_blocks(n, k)`` block summed left to right, the block results added in
ascending order from 0.0), both bit for bit, computed by ``k_xdot`` (csrc/xdot.cuh) through
the C ABI ``mcr_xdot``. The BiCGStab solvers use the same kernel inside the solve.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

XDOT_STATS = ("hard_threads", "warp_tables", "cta_tables", "group_fallbacks", "cta_fallbacks",
              "warp_fallbacks", "thread_fallbacks", "serial_sums",
              # self-checks of a MCR_XDOT_DEBUG build
              "dbg_runs", "dbg_runs_bad", "dbg_tables", "dbg_tables_bad", "dbg_translations",
              "dbg_translations_bad", "dbg_spare",
              "why_hole", "why_sign", "why_binade", "why_slack", "why_modulus", "why_run_binade",
              "why_run_bounds",
              "t_load", "t_lookback", "t_runs_warps", "t_cta", "t_root_groups", "t_root_walk",
              "t_roots", "ns_skew", "ns_build", "ns_root", "ns_total", "_min_entry", "_max_entry",
              "_max_build", "_m_load", "_m_lookback", "_m_runs", "_m_cta", "maxns_load",
              "maxns_lookback", "maxns_runs", "maxns_cta", "lane_sims_warp", "lane_sims_cta",
              "_w_chain", "_w_merge", "_w_table", "maxns_chain", "maxns_merge", "maxns_table", "slowest_table")


def _run(u, v, nblocks: int, device: int, stats: bool):
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    if u.shape != v.shape or u.ndim != 1:
        raise ValueError(f"dot of shapes {u.shape} and {v.shape}")
    L = _lib.load()
    out = np.zeros(1 + nblocks)
    st = np.zeros(len(XDOT_STATS), dtype=np.uint64)
    rc = L.mcr_xdot(int(device), int(u.size), u.ctypes.data, v.ctypes.data, int(nblocks),
                    out.ctypes.data, st.ctypes.data if stats else None)
    if rc != _lib.MCR_OK:
        raise _lib.NativeLibraryError(f"libmcr error {rc}: {_lib.last_error()}")
    return out, dict(zip(XDOT_STATS, (int(x) for x in st)))


def dot_ascending(u, v, device: int = 0) -> float:
    """np.cumsum(u * v)[-1] (0.0 when empty), bit for bit."""
    return float(_run(u, v, 1, device, False)[0][0])


def dot_blocks(u, v, nblocks: int, device: int = 0):
    """(combined dot, [block dots]) of the reference's parallel_dot_products mode."""
    out, _ = _run(u, v, nblocks, device, False)
    return float(out[0]), [float(x) for x in out[1:]]


def dot_stats(u, v, nblocks: int = 1, device: int = 0):
    """(dot, fallback counters); the counters are filled when MCR_XDOT_STATS=1 was set
    before the library was first used."""
    out, st = _run(u, v, nblocks, device, True)
    return float(out[0]), st


CTA_MAX_N = 8192


def dot_ascending_cta(u, v, u2=None, v2=None, device: int = 0):
    """The same sum(s) by the one-CTA path of the small whole-solve BiCGStab kernel
    (n <= 8192; a second pair u2, v2 is summed in the same launch): a float, or a pair."""
    pairs = [(u, v)] + ([(u2, v2)] if u2 is not None else [])
    arrs = []
    for a, b in pairs:
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        if a.shape != b.shape or a.ndim != 1 or a.shape != np.shape(pairs[0][0]):
            raise ValueError("dot_ascending_cta: shapes")
        arrs += [a, b]
    if arrs[0].size > CTA_MAX_N:
        raise ValueError(f"dot_ascending_cta: n <= {CTA_MAX_N}")
    k = len(pairs)
    if k == 1:
        arrs += [arrs[0], arrs[1]]
    out = np.zeros(2)
    L = _lib.load()
    rc = L.mcr_xdot_cta(int(device), int(arrs[0].size), *(a.ctypes.data for a in arrs), k, out.ctypes.data)
    if rc != _lib.MCR_OK:
        raise _lib.NativeLibraryError(f"libmcr error {rc}: {_lib.last_error()}")
    return float(out[0]) if k == 1 else (float(out[0]), float(out[1]))

