"""GPU: the reference's inner products, bit for bit (S/solvers.py:136-141 `_dot_ascending`,
:384-396 `_ParOps.dot` with parallel_dot_products), through the C ABI:

* `dots.dot_ascending` / `dots.dot_blocks` -- k_xdot, the many-CTA kernel the BiCGStab solves
  of large systems use;
* `dots.dot_ascending_cta` -- the one-CTA path of the small whole-solve kernel
  (k_bicg_small<*, true>, n <= 8192), one and two dots per launch.

The checker is the reference's own expression, `np.cumsum(u * v)[-1]`, on adversarial inputs:
sums that wander through zero, ties to even, cancellation, subnormals, -0.0, inf / nan,
overflow, all sizes around the thread / warp / CTA boundaries.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def ref_dot(u, v):
    return float(np.cumsum(u * v)[-1]) if len(u) else 0.0


def ref_blocks(u, v, k):
    base, extra = divmod(len(u), k)
    acc, start, parts = 0.0, 0, []
    for i in range(k):
        size = base + (1 if i < extra else 0)
        p = ref_dot(u[start:start + size], v[start:start + size])
        parts.append(p)
        acc += p
        start += size
    return acc, parts


def bits(x):
    return np.float64(x).tobytes()


def adversarial(n, rng):
    yield "normal", rng.standard_normal(n), rng.standard_normal(n)
    yield "positive", np.abs(rng.standard_normal(n)), np.abs(rng.standard_normal(n))
    yield "drift", rng.standard_normal(n) + 0.01, rng.standard_normal(n)
    yield "ints", rng.integers(1, 11, n).astype(float), rng.integers(1, 11, n).astype(float)
    a = np.ones(n); a[0] = 2.0 ** 53
    yield "ties_even", a, np.ones(n)
    a = np.ones(n); a[0] = 2.0 ** 53 + 2
    yield "ties_odd", a, np.ones(n)
    yield "wide", rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n), rng.standard_normal(n)
    z = np.zeros(n); z[::7] = -0.0
    yield "zeros", z, np.full(n, -1.0)
    yield "negzero", np.full(n, -0.0), np.ones(n)
    a = rng.standard_normal(n); a[n // 2] = np.inf
    yield "inf", a, np.ones(n)
    a = rng.standard_normal(n); a[n // 3] = np.nan
    yield "nan", a, np.ones(n)
    yield "overflow", np.full(n, 1e300), np.full(n, 1e10)
    yield "subnormal", rng.standard_normal(n) * 1e-310, np.ones(n)
    a = rng.standard_normal(n); a[1::2] = -a[0::2][: n // 2]
    yield "cancel", a, np.ones(n)
    q = rng.integers(1, 11, n).astype(float)
    r = np.cumsum(rng.standard_normal(n)) * 1e-6 + 1e-5 * rng.standard_normal(n)
    yield "qr_like", q, r


SIZES_CTA = (0, 1, 2, 31, 33, 256, 384, 385, 1000, 2000, 4097, 7647, 8192)


@pytest.mark.parametrize("n", SIZES_CTA)
def test_cta_dot_bitwise(n):
    from paper_1210_6412_b200 import dots
    rng = np.random.default_rng(n)
    for name, u, v in adversarial(max(n, 1), rng):
        u, v = u[:n], v[:n]
        got = dots.dot_ascending_cta(u, v)
        assert bits(got) == bits(ref_dot(u, v)), (name, n, got, ref_dot(u, v))


@pytest.mark.parametrize("n", (385, 2000, 8192))
def test_cta_two_dots_in_one_launch(n):
    from paper_1210_6412_b200 import dots
    rng = np.random.default_rng(7 + n)
    cases = list(adversarial(n, rng))
    for (na, ua, va), (nb, ub, vb) in zip(cases, cases[1:] + cases[:1]):
        got = dots.dot_ascending_cta(ua, va, ub, vb)
        assert bits(got[0]) == bits(ref_dot(ua, va)), (na, nb)
        assert bits(got[1]) == bits(ref_dot(ub, vb)), (na, nb)


def test_cta_dot_bicgstab_like_walks():
    """Many sums that pass through zero over and over (the C4 regime): every segment of the
    walk's fast path and its element-by-element fallback."""
    from paper_1210_6412_b200 import dots
    rng = np.random.default_rng(3)
    for trial in range(40):
        n = int(rng.integers(385, 8193))
        u = rng.standard_normal(n)
        v = rng.standard_normal(n) * 10.0 ** rng.integers(-3, 3)
        got = dots.dot_ascending_cta(u, v)
        assert bits(got) == bits(ref_dot(u, v)), (trial, n)


@pytest.mark.parametrize("n", (0, 1, 511, 512, 513, 100_000))
def test_xdot_bitwise(n):
    from paper_1210_6412_b200 import dots
    rng = np.random.default_rng(11 + n)
    for name, u, v in adversarial(max(n, 1), rng):
        u, v = u[:n], v[:n]
        got = dots.dot_ascending(u, v)
        assert bits(got) == bits(ref_dot(u, v)), (name, n)


def test_xdot_million_walk_and_positive():
    from paper_1210_6412_b200 import dots
    rng = np.random.default_rng(5)
    n = 1_000_000
    for u, v in ((rng.standard_normal(n), rng.standard_normal(n)),
                 (np.abs(rng.standard_normal(n)), np.abs(rng.standard_normal(n)))):
        assert bits(dots.dot_ascending(u, v)) == bits(ref_dot(u, v))


@pytest.mark.parametrize("k", (2, 3, 16))
def test_xdot_blocks_bitwise(k):
    from paper_1210_6412_b200 import dots
    rng = np.random.default_rng(k)
    for name, u, v in adversarial(50_001, rng):
        got, parts = dots.dot_blocks(u, v, k)
        want, wparts = ref_blocks(u, v, k)
        assert bits(got) == bits(want), (name, k)
        assert [bits(x) for x in parts] == [bits(x) for x in wparts], (name, k)
