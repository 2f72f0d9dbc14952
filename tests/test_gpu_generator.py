"""Device generator of the C5 family (csrc/generator.cuh) against its CPU restatement
(oracle/oracle.c orc_generate): identical arrays for the whole system and for every shard of
several world sizes; solves of a generated system match the oracle (Jacobi bit for bit)."""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from paper_1210_6412_b200 import _lib, dist, solvers
    _lib.load()
    assert _lib.device_count() >= 1, "no CUDA device visible"
    return dist, solvers


@pytest.mark.parametrize("n,mean,seed", [(100003, 7.0, 1), (4097, 0.0, 2), (3, 30.0, 3),
                                         (50000, 12.5, 4)])
def test_device_generator_matches_oracle(mods, n, mean, seed):
    from oracle import oracle
    dist, gs = mods
    dm = gs.DeviceMatrix.generated(n, mean, 1, 10, seed, storage=5)
    rs, col, val = dm.export()
    ref = oracle.generate(seed, n, mean)
    assert np.array_equal(rs, ref.rstart)
    assert np.array_equal(col, ref.col)
    assert np.array_equal(val, ref.nonzero)
    import torch
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    dm.generated_rhs(seed, b.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(b.cpu().numpy(), oracle.generate_rhs(seed, n))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_generation_matches_slices(mods, world):
    from oracle import oracle
    dist, gs = mods
    n, seed = 30011, 9
    ref = oracle.generate(seed, n, 7.0)
    comms = dist.Comm.local_group(world)
    try:
        for r in range(world):
            sh = dist.ShardMatrix.generated(comms[r], n, 7.0, 1, 10, seed)
            dm = gs.DeviceMatrix(None, _handle=sh.handle)
            rs, col, val = dm.export()
            dm._finalizer.detach()  # owned by the ShardMatrix
            e0, e1 = ref.rstart[sh.row0], ref.rstart[sh.row0 + sh.n]
            assert np.array_equal(rs, ref.rstart[sh.row0:sh.row0 + sh.n + 1] - e0)
            assert np.array_equal(col, ref.col[e0:e1])
            assert np.array_equal(val, ref.nonzero[e0:e1])
            sh.close()
    finally:
        for c in comms:
            c.close()


def test_generated_system_solves_like_oracle(mods):
    from oracle import oracle
    dist, gs = mods
    n, seed = 200000, 5
    ref = oracle.generate(seed, n, 7.0)
    b = oracle.generate_rhs(seed, n)
    dm = gs.DeviceMatrix.generated(n, 7.0, 1, 10, seed)
    rc, x, rep = dm.solve("jacobi", b, None, 1e-10, 10_000)
    oj = oracle.jacobi(ref, b)
    assert rc == 0 and rep.iterations == oj["iterations"]
    assert np.array_equal(x, oj["x"])
    assert float(rep.residual_inf).hex() == float(oj["residual_inf"]).hex()
    rc, xb, repb = dm.solve("bicgstab", b, None, 1e-10, 10_000)
    ob = oracle.bicgstab(ref, b)  # the reference's algorithm incl. its left-to-right dots
    assert rc == 0 and repb.iterations == ob["iterations"]
    assert np.array_equal(xb, ob["x"])


def test_sharded_generated_solve_bit_identical(mods):
    """World 3 on generated shards: Jacobi x identical to one GPU, device-pointer path."""
    import torch
    dist, gs = mods
    n, seed, world = 120001, 7, 3
    one = gs.DeviceMatrix.generated(n, 7.0, 1, 10, seed, storage=5)
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    one.generated_rhs(seed, b.data_ptr())
    torch.cuda.synchronize()
    rc, x1, rep1 = one.solve("jacobi", b.cpu().numpy(), None, 1e-10, 10_000)
    assert rc == 0
    comms = dist.Comm.local_group(world)
    xs, reps = [None] * world, [None] * world

    def run(r):
        sh = dist.ShardMatrix.generated(comms[r], n, 7.0, 1, 10, seed)
        bl = torch.empty(sh.n, dtype=torch.float64, device="cuda")
        xl = torch.empty(sh.n, dtype=torch.float64, device="cuda")
        sh.generated_rhs(seed, bl.data_ptr())
        rcr, rep = sh.solve_device("jacobi", bl.data_ptr(), None, 1e-10, 10_000, xl.data_ptr())
        assert rcr == 0
        torch.cuda.synchronize()
        xs[r], reps[r] = xl.cpu().numpy(), rep
        sh.close()

    try:
        ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    finally:
        for c in comms:
            c.close()
    assert all(r is not None for r in reps)
    assert all(r.iterations == rep1.iterations for r in reps)
    assert np.array_equal(np.concatenate(xs), x1)


def test_large_generated_staged_equals_tiles(mods):
    """Beyond L2 (n = 2e7, x = 160 MB) AUTO picks the band-staged layout; at full size its SpMV
    and Jacobi iterates are bit-identical to the tiled CSR kernels (a size-independent check:
    the oracle would take minutes here), and the BiCGStab solution agrees within 1e-9."""
    import ctypes
    import torch
    from paper_1210_6412_b200 import _lib
    dist, gs = mods
    n, seed = 20_000_000, 9
    L = _lib.load()
    staged = gs.DeviceMatrix.generated(n, 7.0, 1, 10, seed)
    tiles = gs.DeviceMatrix.generated(n, 7.0, 1, 10, seed, storage=_lib.STORAGE_TILES_STREAM)
    try:
        assert staged.info()["storage"] == _lib.STORAGE_STAGED
        assert tiles.info()["storage"] == _lib.STORAGE_TILES
        dev = torch.device("cuda", 0)
        x = torch.rand(n, dtype=torch.float64, device=dev, generator=torch.Generator(dev).manual_seed(3))
        ys = torch.empty_like(x)
        yt = torch.empty_like(x)
        for dm, y in ((staged, ys), (tiles, yt)):
            assert L.mcr_matvec_device(dm.handle, ctypes.c_void_p(x.data_ptr()),
                                       ctypes.c_void_p(y.data_ptr())) == _lib.MCR_OK
        torch.cuda.synchronize()
        assert torch.equal(ys, yt)
        b = torch.empty(n, dtype=torch.float64, device=dev)
        staged.generated_rhs(seed, b.data_ptr())
        out = []
        for dm in (staged, tiles):
            res = []
            for fn, it in ((L.mcr_jacobi_device, 25), (L.mcr_bicgstab_device, 10_000)):
                xo = torch.empty(n, dtype=torch.float64, device=dev)
                rep = _lib.Report()
                rc = fn(dm.handle, ctypes.c_void_p(b.data_ptr()), None, 1e-10, it,
                        ctypes.c_void_p(xo.data_ptr()), ctypes.byref(rep))
                assert rc in (_lib.MCR_OK, _lib.MCR_NOT_CONVERGED), _lib.last_error()
                res.append((rep.iterations, float(rep.residual_inf), xo))
            out.append(res)
        (js, bs), (jt, bt) = out
        assert js[0] == jt[0] and js[1] == jt[1] and torch.equal(js[2], jt[2])  # Jacobi: exact
        assert abs(bs[0] - bt[0]) <= 2                                           # BiCGStab: dots
        assert float((bs[2] - bt[2]).abs().max()) / max(1.0, float(bt[2].abs().max())) <= 1e-9
    finally:
        staged.close()
        tiles.close()
