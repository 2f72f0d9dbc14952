"""GPU: the reference's input generator on the device (csrc/refgen.cuh, mcr_refgen_*), drawing
numpy's default_rng stream: bounded draws against numpy itself (both Lemire widths, heavy
rejection, the pending 32-bit half across calls), generate_rhs, and whole matrices against the
SHA-256 pins of the reference's own arrays (tests/golden) and the golden-pinned host port."""

import ctypes

import numpy as np
import pytest

from golden_cases import manifest, sha

pytestmark = pytest.mark.gpu


def _u64(seed, n, rng_size):
    from paper_1210_6412_b200 import _lib
    from paper_1210_6412_b200.generator import pcg_words
    out = np.empty(n, dtype=np.uint64)
    rc = _lib.load().mcr_refgen_u64(0, n, ctypes.c_uint64(rng_size), pcg_words(seed).ctypes.data, out.ctypes.data)
    assert rc == 0, _lib.last_error()
    return out


@pytest.mark.parametrize("seed", [0, 1, 12345])
@pytest.mark.parametrize("size", [10 ** 6 * (10 ** 6 - 1), 3 * 2 ** 61, 2 ** 63 + 1, 2000 * 1999, 3 * 2 ** 30,
                                  2 ** 31 + 1, 2 ** 32, 10])
def test_bounded_draws_match_numpy(seed, size):
    n = 100_003
    want = np.random.default_rng(seed).integers(0, size, size=n, dtype=np.uint64)
    assert np.array_equal(_u64(seed, n, size), want), size


@pytest.mark.parametrize("seed", [0, 7, 2 ** 40 + 7])
def test_generate_rhs_matches_numpy(seed):
    from paper_1210_6412_b200.generator import generate_rhs, generate_rhs_device
    for n in (1, 2, 1001, 1_000_000):
        assert np.array_equal(generate_rhs_device(n, seed), generate_rhs(n, seed)), n


def _export(dm):
    from paper_1210_6412_b200 import _lib
    info = dm.info()
    n, nnz = int(info["n"]), int(info["nnz"])
    rs = np.empty(n + 1, dtype=np.int64)
    col = np.empty(nnz, dtype=np.int64)
    val = np.empty(nnz, dtype=np.float64)
    rc = _lib.load().mcr_matrix_export(dm.handle, rs.ctypes.data, col.ctypes.data, val.ctypes.data)
    assert rc == 0, _lib.last_error()
    return rs, col, val


SPEC_CASES = [name for name, c in manifest()["cases"].items() if c.get("spec") and c["n"] <= 20_000]


@pytest.mark.parametrize("name", SPEC_CASES)
def test_matrix_matches_reference_pins(name):
    """Every golden case built from a GenSpec: the device arrays hash to the reference's."""
    from paper_1210_6412_b200 import _lib
    from paper_1210_6412_b200.generator import GenSpec, generate_rhs_device
    from paper_1210_6412_b200.solvers import DeviceMatrix
    c = manifest()["cases"][name]
    s = c["spec"]
    spec = GenSpec(n=s["n"], nnz=s["nnz"], density=s["density"], seed=s["seed"])
    dm = DeviceMatrix.reference_generated(spec, 0, _lib.STORAGE_CSR)
    try:
        rs, col, val = _export(dm)
    finally:
        dm.close()
    assert sha(rs) == c["rstart_sha256"], name
    assert sha(col) == c["col_sha256"], name
    assert sha(val) == c["nonzero_sha256"], name
    assert sha(generate_rhs_device(s["n"], s["seed"])) == c["b_sha256"], name


@pytest.mark.parametrize("n,nnz,seed", [(70_000, 500_000, 5), (1, 1, 3), (2, 4, 1), (40, 40 * 40, 9),
                                        (65_000, 1_000_000, 4)])
def test_matrix_matches_host_port(n, nnz, seed):
    """64-bit code path (n (n - 1) > 2^32), the complete-matrix shortcut, tiny systems."""
    from paper_1210_6412_b200 import _lib
    from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix
    from paper_1210_6412_b200.solvers import DeviceMatrix
    spec = GenSpec(n=n, nnz=nnz, seed=seed)
    m = generate_dd_matrix(spec)
    dm = DeviceMatrix.reference_generated(spec, 0, _lib.STORAGE_CSR)
    try:
        rs, col, val = _export(dm)
    finally:
        dm.close()
    assert np.array_equal(rs, m.rstart) and np.array_equal(col, m.col) and np.array_equal(val, m.nonzero)


@pytest.mark.slow
def test_c2_matrix_matches_reference_pins():
    from paper_1210_6412_b200 import _lib
    from paper_1210_6412_b200.generator import GenSpec, generate_rhs_device
    from paper_1210_6412_b200.solvers import DeviceMatrix
    name = "c2_trial0"
    c = manifest()["cases"][name]
    s = c["spec"]
    dm = DeviceMatrix.reference_generated(GenSpec(n=s["n"], nnz=s["nnz"], density=s["density"], seed=s["seed"]),
                                          0, _lib.STORAGE_CSR)
    try:
        rs, col, val = _export(dm)
    finally:
        dm.close()
    assert sha(rs) == c["rstart_sha256"] and sha(col) == c["col_sha256"] and sha(val) == c["nonzero_sha256"]
    assert sha(generate_rhs_device(s["n"], s["seed"])) == c["b_sha256"]
