"""C-ABI checks that need no GPU: the library builds, loads, exports every symbol declared
in include/mcr.h, and fails loudly (no CPU fallback) when no device is present."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "mcr.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"MCR_API\s+[\w\s\*]+?\b(mcr_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("mcr_matrix_create", "mcr_jacobi", "mcr_bicgstab", "mcr_matvec",
              "mcr_residual_inf", "mcr_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1210_6412_b200 import _lib
    L = _lib.load()
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert set(_lib.EXPORTS) == set(declared_symbols())
    assert L.mcr_version() >= 100


def test_library_exports_nothing_else():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only",
                          os.path.join(ROOT, "paper_1210_6412_b200", "libmcr.so")],
                         capture_output=True, text=True, check=True).stdout
    ours = sorted({ln.split()[-1] for ln in out.splitlines() if " T mcr_" in ln})
    assert ours == declared_symbols()


def test_sm100a_code_in_library():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf",
                          os.path.join(ROOT, "paper_1210_6412_b200", "libmcr.so")],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_device_fails_loudly():
    from paper_1210_6412_b200 import _lib, solvers
    from paper_1210_6412_b200.sparse import csr_from_triplets
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible; covered by the gpu tests")
    m = csr_from_triplets(2, [(0, 0, 1.0), (1, 1, 1.0)])
    with pytest.raises(_lib.NativeLibraryError):
        solvers.jacobi_solve(m, np.ones(2))
    h = ctypes.c_void_p()
    rs = np.array([0, 1, 2], np.int64)
    rc = _lib.load().mcr_matrix_create(2, rs.ctypes.data, rs.ctypes.data,
                                       np.ones(2).ctypes.data, 0, 0, ctypes.byref(h))
    assert rc == _lib.MCR_CUDA_ERROR
    assert "device" in _lib.last_error()


def test_empty_system_needs_no_device():
    # solvers.py:216-217 -- n = 0 short-circuits before any device work
    from paper_1210_6412_b200 import solvers
    from paper_1210_6412_b200.sparse import csr_from_triplets
    empty = csr_from_triplets(0, [])
    for fn in solvers.SOLVERS.values():
        r = fn(empty, np.zeros(0))
        assert r.converged and r.iterations == 0


def test_config_validation():
    from paper_1210_6412_b200.solvers import SolverConfig
    with pytest.raises(ValueError):
        SolverConfig(tolerance=0.0)
    with pytest.raises(ValueError):
        SolverConfig(max_iterations=0)
    with pytest.raises(ValueError):
        SolverConfig(workers=0)
