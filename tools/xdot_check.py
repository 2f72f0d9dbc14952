"""GPU check of the reference-order dot (k_xdot) against np.cumsum on adversarial inputs."""
import os, sys, time
os.environ.setdefault("MCR_XDOT_STATS", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1210_6412_b200 import dots


def ref(u, v, k=1):
    if k == 1:
        return np.cumsum(u * v)[-1] if len(u) else 0.0
    base, extra = divmod(len(u), k)
    acc, st = 0.0, 0
    parts = []
    for i in range(k):
        sz = base + (1 if i < extra else 0)
        p = np.cumsum(u[st:st + sz] * v[st:st + sz])[-1] if sz else 0.0
        parts.append(p)
        acc += p
        st += sz
    return acc, parts


def cases(rng):
    yield "empty", np.zeros(0), np.zeros(0)
    for n in (1, 2, 31, 32, 33, 255, 256, 257, 1000, 8191, 65537):
        yield f"normal{n}", rng.standard_normal(n), rng.standard_normal(n)
    n = 10**6
    yield "walk", rng.standard_normal(n), rng.standard_normal(n)
    yield "positive", np.abs(rng.standard_normal(n)), np.abs(rng.standard_normal(n))
    yield "drift", rng.standard_normal(n) + 0.01, rng.standard_normal(n)
    t = np.linspace(0, 20, n)
    yield "oscill", np.sin(t) + 1e-3 * rng.standard_normal(n), np.ones(n)
    yield "ints", rng.integers(1, 11, n).astype(float), rng.integers(1, 11, n).astype(float)
    a = np.ones(n); a[0] = 2.0**53
    yield "ties_even", a, np.ones(n)
    a = np.ones(n); a[0] = 2.0**53 + 2
    yield "ties_odd", a, np.ones(n)
    a = rng.choice([1.0, 3.0, 0.5], n); a[0] = 2.0**54 + 4
    yield "ties_mix", a, np.ones(n)
    yield "wide", rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n), rng.standard_normal(n)
    z = np.zeros(n); z[::7] = -0.0
    yield "zeros", z, np.full(n, -1.0)
    yield "negzero", np.full(1000, -0.0), np.ones(1000)
    a = rng.standard_normal(n); a[n // 2] = np.inf
    yield "inf", a, np.ones(n)
    a = rng.standard_normal(n); a[n // 3] = np.nan
    yield "nan", a, np.ones(n)
    yield "overflow", np.full(n, 1e300), np.full(n, 1e10)
    yield "subnormal", rng.standard_normal(n) * 1e-310, np.ones(n)
    a = rng.standard_normal(n); a[1::2] = -a[0::2]
    yield "cancel", a, np.ones(n)
    yield "near1", 1.0 + 1e-9 * rng.standard_normal(n), np.concatenate([[1.0], np.full(n - 1, 1e-7)])
    # BiCGStab-like: q positive integers, r mixed residual-ish with drift changes
    q = rng.integers(1, 11, n).astype(float)
    r = np.cumsum(rng.standard_normal(n)) * 1e-6 + 1e-5 * rng.standard_normal(n)
    yield "qr_like", q, r
    n2 = 20_000_000
    yield "walk20M", rng.standard_normal(n2), rng.standard_normal(n2)


def main():
    rng = np.random.default_rng(1)
    bad = 0
    for name, u, v in cases(rng):
        t0 = time.time()
        got, st = dots.dot_stats(u, v)
        dt = time.time() - t0
        want = ref(u, v)
        ok = np.float64(got).tobytes() == np.float64(want).tobytes() or (np.isnan(got) and np.isnan(want))
        bad += not ok
        nz = {k: x for k, x in st.items() if x}
        print(f"{'OK ' if ok else 'BAD'} {name:12s} n={len(u):9d} got={got!r} want={want!r} {dt*1e3:7.1f}ms {nz}", flush=True)
        for k in (3, 16):
            if len(u) < 100 or name in ("walk20M",):
                continue
            g, parts = dots.dot_blocks(u, v, k)
            w, wparts = ref(u, v, k)
            okb = (np.float64(g).tobytes() == np.float64(w).tobytes() or (np.isnan(g) and np.isnan(w))) and all(
                np.float64(a).tobytes() == np.float64(b).tobytes() or (np.isnan(a) and np.isnan(b)) for a, b in zip(parts, wparts))
            bad += not okb
            if not okb:
                print(f"BAD blocks{k} {name}: {g!r} vs {w!r}", flush=True)
    print("mismatches:", bad)
    return bad


if __name__ == "__main__":
    sys.exit(1 if main() else 0)
