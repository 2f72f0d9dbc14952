"""ctypes binding of libmcr.so (include/mcr.h).

The shared library is the only compute path: if it is missing or cannot be loaded, every
solver call raises ``NativeLibraryError``; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MCR_LIB") or os.path.join(_HERE, "libmcr.so")

MCR_OK = 0
MCR_NOT_CONVERGED = 1
MCR_BREAKDOWN = 2
MCR_ZERO_DIAGONAL = 3
MCR_DIMENSION = 4
MCR_CUDA_ERROR = 5
MCR_INVALID_ARGUMENT = 6

STORAGE_AUTO, STORAGE_CSR, STORAGE_DENSE, STORAGE_SELL, STORAGE_TILES, STORAGE_TILES_STREAM = 0, 1, 2, 3, 4, 5
STORAGE_STAGED = 6
BREAKDOWN_NAMES = {1: "y_prev*w", 2: "q*v", 3: "t*t"}

EXPORTS = (
    "mcr_version", "mcr_device_count", "mcr_matrix_create", "mcr_matrix_destroy",
    "mcr_matrix_info_get", "mcr_set_stream", "mcr_matvec", "mcr_matvec_device",
    "mcr_residual_inf", "mcr_jacobi", "mcr_jacobi_device", "mcr_bicgstab",
    "mcr_bicgstab_device", "mcr_last_error", "mcr_set_dot_mode",
    "mcr_shard_rows", "mcr_comm_unique_id", "mcr_comm_create_nccl", "mcr_comm_create_local",
    "mcr_comm_destroy", "mcr_comm_info", "mcr_shard_create", "mcr_generate",
    "mcr_generate_rhs", "mcr_matrix_export", "mcr_chain_create", "mcr_chain_destroy",
    "mcr_chain_info", "mcr_chain_export", "mcr_chain_matrix", "mcr_chain_solve",
    "mcr_shard_enable_p2p", "mcr_read_matrix", "mcr_read_vector", "mcr_read_dtmc",
    "mcr_text_info", "mcr_text_export", "mcr_text_destroy", "mcr_text_reason",
    "mcr_set_dot_blocks", "mcr_xdot", "mcr_xdot_stats", "mcr_xdot_bench", "mcr_xdot_cta",
    "mcr_refgen_matrix", "mcr_refgen_integers", "mcr_refgen_u64",
)
MCR_UNSUPPORTED_INPUT = 7
COMM_ID_BYTES = 128
DOTS_TREE, DOTS_SEQUENTIAL, DOTS_SERIAL = 0, 1, 2
DOT_MODES = {"tree": DOTS_TREE, "sequential": DOTS_SEQUENTIAL, "serial": DOTS_SERIAL}


class NativeLibraryError(RuntimeError):
    """libmcr.so is missing, failed to load, or a CUDA call inside it failed."""


class Report(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int64),
        ("converged", ctypes.c_int32),
        ("breakdown_which", ctypes.c_int32),
        ("breakdown_iteration", ctypes.c_int64),
        ("zero_diagonal_index", ctypes.c_int64),
        ("residual_inf", ctypes.c_double),
        ("device_seconds", ctypes.c_double),
        ("kernel_launches", ctypes.c_int64),
    ]


class MatrixInfo(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("storage", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("tiles", ctypes.c_int64),
        ("max_row_nnz", ctypes.c_int64),
        ("first_zero_diagonal", ctypes.c_int64),
        ("device_bytes", ctypes.c_int64),
        ("n_global", ctypes.c_int64),
        ("row0", ctypes.c_int64),
        ("world", ctypes.c_int32),
        ("rank", ctypes.c_int32),
    ]


_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as err:
        raise NativeLibraryError(f"cannot load {LIB_PATH}: {err}") from err
    vp = ctypes.c_void_p
    i64 = ctypes.c_int64
    dbl = ctypes.c_double
    L.mcr_version.restype = ctypes.c_int
    L.mcr_version.argtypes = []
    L.mcr_device_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
    L.mcr_matrix_create.argtypes = [i64, vp, vp, vp, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(vp)]
    L.mcr_matrix_destroy.argtypes = [vp]
    L.mcr_matrix_destroy.restype = None
    L.mcr_matrix_info_get.argtypes = [vp, ctypes.POINTER(MatrixInfo)]
    L.mcr_set_stream.argtypes = [vp, vp]
    L.mcr_set_dot_mode.argtypes = [vp, ctypes.c_int]
    L.mcr_set_dot_blocks.argtypes = [vp, ctypes.c_int]
    L.mcr_xdot.argtypes = [ctypes.c_int, i64, vp, vp, ctypes.c_int, vp, vp]
    L.mcr_xdot_stats.argtypes = [vp, vp, ctypes.c_int]
    L.mcr_xdot_bench.argtypes = [ctypes.c_int, i64, vp, vp, ctypes.c_int, ctypes.c_int, vp, vp, vp]
    L.mcr_xdot_cta.argtypes = [ctypes.c_int, i64, vp, vp, vp, vp, ctypes.c_int, vp]
    L.mcr_refgen_matrix.argtypes = [ctypes.c_int, i64, i64, i64, i64, vp, ctypes.c_int, ctypes.POINTER(vp)]
    L.mcr_refgen_integers.argtypes = [ctypes.c_int, i64, i64, i64, vp, vp]
    L.mcr_refgen_u64.argtypes = [ctypes.c_int, i64, ctypes.c_uint64, vp, vp]
    L.mcr_matvec.argtypes = [vp, vp, vp]
    L.mcr_matvec_device.argtypes = [vp, vp, vp]
    L.mcr_residual_inf.argtypes = [vp, vp, vp, ctypes.POINTER(dbl)]
    for name in ("mcr_jacobi", "mcr_jacobi_device", "mcr_bicgstab", "mcr_bicgstab_device"):
        getattr(L, name).argtypes = [vp, vp, vp, dbl, i64, vp, ctypes.POINTER(Report)]
    ip = ctypes.c_int
    pi64 = ctypes.POINTER(i64)
    pint = ctypes.POINTER(ctypes.c_int)
    L.mcr_shard_rows.argtypes = [i64, ip, ip, pi64, pi64]
    L.mcr_comm_unique_id.argtypes = [vp]
    L.mcr_comm_create_nccl.argtypes = [vp, ip, ip, ip, ctypes.POINTER(vp)]
    L.mcr_comm_create_local.argtypes = [ip, vp, ctypes.POINTER(vp)]
    L.mcr_comm_destroy.argtypes = [vp]
    L.mcr_comm_destroy.restype = None
    L.mcr_comm_info.argtypes = [vp, pint, pint, pint]
    L.mcr_shard_create.argtypes = [vp, i64, i64, i64, vp, vp, vp, ctypes.POINTER(vp)]
    L.mcr_generate.argtypes = [vp, ip, i64, dbl, ip, ip, ctypes.c_uint64, ip, ctypes.POINTER(vp)]
    L.mcr_generate_rhs.argtypes = [vp, ctypes.c_uint64, vp]
    L.mcr_matrix_export.argtypes = [vp, vp, vp, vp]
    L.mcr_shard_enable_p2p.argtypes = [vp]
    for name in ("mcr_read_matrix", "mcr_read_vector", "mcr_read_dtmc"):
        getattr(L, name).argtypes = [ctypes.c_char_p, ip, ctypes.POINTER(vp)]
    L.mcr_text_info.argtypes = [vp, pi64, pi64, pi64, pi64]
    L.mcr_text_export.argtypes = [vp, vp, vp, vp, vp]
    L.mcr_text_destroy.argtypes = [vp]
    L.mcr_text_destroy.restype = None
    L.mcr_text_reason.restype = ctypes.c_char_p
    L.mcr_text_reason.argtypes = []
    L.mcr_chain_create.argtypes = [i64, vp, vp, vp, vp, i64, ip, ctypes.POINTER(vp)]
    L.mcr_chain_destroy.argtypes = [vp]
    L.mcr_chain_destroy.restype = None
    L.mcr_chain_info.argtypes = [vp, pi64, pi64, pi64, pi64]
    L.mcr_chain_export.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.mcr_chain_matrix.argtypes = [vp, ctypes.POINTER(vp)]
    L.mcr_chain_solve.argtypes = [vp, ip, ip, dbl, i64, vp, vp, vp, ctypes.POINTER(Report)]
    L.mcr_last_error.restype = ctypes.c_char_p
    L.mcr_last_error.argtypes = []
    _lib = L
    return L


def last_error() -> str:
    return load().mcr_last_error().decode(errors="replace")


def device_count() -> int:
    c = ctypes.c_int(0)
    load().mcr_device_count(ctypes.byref(c))
    return c.value
