"""CPU: the restated numpy stream (oracle/pcg64.py, the device generator's checker) against
numpy itself and against the reference generator's arrays."""

import numpy as np
import pytest

from oracle import pcg64

RANGES = [  # (low, high, endpoint): 32-bit and 64-bit paths, heavy rejection, the 2^32 edge
    (0, 10 ** 6 * (10 ** 6 - 1), False), (1, 10, True), (0, 3 * 2 ** 30, False),
    (0, 2 ** 31 + 1, False), (5, 2 ** 32 + 5, False), (0, 2 ** 32, True), (0, 3 * 2 ** 61, False),
    (0, 2 ** 33, False), (7, 7, True), (0, 2000 * 1999, False)]


@pytest.mark.parametrize("seed", [0, 1, 12345, 2 ** 40 + 7])
def test_integers_match_numpy(seed):
    rng = np.random.default_rng(seed)
    g = pcg64.PCG64(seed)
    for lo, hi, ep in RANGES:
        for size in (1, 3, 257):  # odd sizes leave a 32-bit half pending across calls
            want = rng.integers(lo, hi, size=size, endpoint=ep).tolist()
            assert pcg64.integers(g, lo, hi, size, ep) == want, (lo, hi, ep, size)
    assert g.next64() == int(rng.bit_generator.random_raw())


@pytest.mark.parametrize("n,nnz,seed", [(92, 211, 3), (300, 5000, 11), (50, 50 * 49 + 50, 2)])
def test_generator_arrays_match_reference(n, nnz, seed):
    """The restated stream gives the reference's matrix (golden-pinned host port)."""
    from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix
    m = generate_dd_matrix(GenSpec(n=n, nnz=nnz, seed=seed))
    rows, cols, vals, diag = pcg64.generate_dd_arrays(n, nnz - n, 1, 10, seed)
    dense = np.zeros((n, n))
    dense[rows, cols] = vals
    dense[np.arange(n), np.arange(n)] = diag
    got = np.zeros((n, n))
    for r in range(n):
        for k in range(m.rstart[r], m.rstart[r + 1]):
            got[r, m.col[k]] = m.nonzero[k]
    assert np.array_equal(dense, got)
