"""Time k_xdot on the inner products of a real C2 BiCGStab run (captured from the reference
solver, run here) and on synthetic vectors: mean us per launch, result check, fallback stats."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref"))
sys.dont_write_bytecode = True
import numpy as np
from paper_1210_6412_b200 import _lib, dots
from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix, generate_rhs, trial_seed

L = _lib.load()


def bench(u, v, reps=20, nblocks=1):
    out = np.zeros(1 + nblocks)
    ms = np.zeros(1)
    st = np.zeros(len(dots.XDOT_STATS), dtype=np.uint64)
    rc = L.mcr_xdot_bench(0, u.size, u.ctypes.data, v.ctypes.data, nblocks, reps, out.ctypes.data,
                          ms.ctypes.data, st.ctypes.data)
    assert rc == 0, _lib.last_error()
    return out[0], ms[0] * 1e3, {k: int(x) for k, x in zip(dots.XDOT_STATS, st) if x}


def main():
    if os.environ.get("XB_SYNTH_ONLY"):
        return synth()
    import mcreach.solvers as S
    from mcreach.sparse import CsrMatrix
    n, nnz = 10**6, 10**7
    seed = trial_seed(0, n, None, nnz, 0)
    g = generate_dd_matrix(GenSpec(n=n, nnz=nnz, seed=seed))
    m = CsrMatrix(g.n, g.rstart, g.col, g.nonzero)
    b = generate_rhs(n, seed)
    rec = []
    orig = S._dot_ascending

    def dot(u, v):
        rec.append((u.copy(), v.copy()))
        return orig(u, v)
    S._dot_ascending = dot
    keep = set(range(0, 320, int(os.environ.get("XB_STRIDE", "9"))))
    if os.environ.get("XB_ONLY"):
        keep = {int(x) for x in os.environ["XB_ONLY"].split(",")}
    t = time.time()
    r = S.bicgstab_solve_parallel(m, b, S.SolverConfig(workers=os.cpu_count()))
    print(f"reference bicgstab-par: {r.iterations} iterations, {len(rec)} dots, {time.time()-t:.1f}s", flush=True)
    names = ["q.r", "q.v", "t.t", "t.s"]
    tot = []
    for i, (u, v) in enumerate(rec):
        if i not in keep:
            continue
        want = np.cumsum(u * v)[-1]
        got, us, st = bench(u, v, reps=int(os.environ.get("XB_REPS", "20")))
        ok = np.float64(got).tobytes() == np.float64(want).tobytes()
        tot.append(us)
        print(f"dot {i:3d} it {(i + 3) // 4:2d} {names[(i + 3) % 4]}: {'OK ' if ok else 'BAD'} {us:8.1f} us  {st}", flush=True)
    print(f"mean {np.mean(tot):.1f} us, median {np.median(tot):.1f} us over {len(tot)} dots")
    synth()


def synth():
    n = 10**6
    rng = np.random.default_rng(0)
    for name, (u, v) in {"positive": (np.abs(rng.standard_normal(n)), np.abs(rng.standard_normal(n))),
                         "ints": (rng.integers(1, 11, n).astype(float), rng.integers(1, 11, n).astype(float)),
                         "walk": (rng.standard_normal(n), rng.standard_normal(n)),
                         "pos_offset": (np.concatenate([[1e6], np.abs(rng.standard_normal(n - 1))]), np.ones(n))}.items():
        got, us, st = bench(u, v, reps=int(os.environ.get("XB_REPS", "20")))
        print(f"{name}: {us:.1f} us {st}", flush=True)


if __name__ == "__main__":
    main()
