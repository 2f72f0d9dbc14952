"""CPU: the multithreaded text readers (csrc/formats.cpp via paper_1210_6412_b200.formats)
against the reference's file semantics (mcreach/formats.py:89-232): values bit-identical to
Python's float() (17-digit round trips), csr_from_triplets order with zeros dropped, comments,
blank lines, CRLF, keyword lines anywhere in chain files; every malformed / non-plain file is
refused by the fast path (MCR_UNSUPPORTED_INPUT) and read by the package's own line-by-line
readers (textio.py), whose results and errors are compared here with the reference reader's
(the reference is the checker only; the package never calls it)."""

import ctypes
import os

import numpy as np
import pytest

from paper_1210_6412_b200 import _lib, formats
from paper_1210_6412_b200.chains import random_dtmc
from paper_1210_6412_b200.generator import GenSpec, generate_dd_matrix


def fmt(v):
    return format(float(v), ".17g")  # formats.py:58-59


def write_matrix(m, path, shuffle=None, extra=""):
    rows = np.repeat(np.arange(m.n), np.diff(m.rstart))
    order = np.arange(m.m) if shuffle is None else shuffle.permutation(m.m)
    lines = [f"matrix {m.n} {m.m}"] + [f"{rows[k]} {m.col[k]} {fmt(m.nonzero[k])}" for k in order]
    path.write_text(extra + "\n".join(lines) + "\n")


def expected_csr(n, triplets):
    r = np.array([t[0] for t in triplets], dtype=np.int64)
    c = np.array([t[1] for t in triplets], dtype=np.int64)
    v = np.array([t[2] for t in triplets], dtype=np.float64)
    keep = v != 0.0
    r, c, v = r[keep], c[keep], v[keep]
    o = np.lexsort((c, r))
    rs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=rs[1:])
    return rs, c[o], v[o]


def rc_of(fn, path):
    L = _lib.load()
    h = ctypes.c_void_p()
    rc = getattr(L, fn)(os.fsencode(str(path)), 0, ctypes.byref(h))
    if h.value:
        L.mcr_text_destroy(h)
    return rc


@pytest.mark.parametrize("seed", range(4))
def test_matrix_round_trip_bitwise(tmp_path, seed):
    rng = np.random.default_rng(seed)
    m = generate_dd_matrix(GenSpec(n=300 + 100 * seed, nnz=3000 + 500 * seed, seed=seed))
    m2 = type(m)(m.n, m.rstart, m.col, m.nonzero / 7.0)  # awkward fractions
    p = tmp_path / "m.txt"
    write_matrix(m2, p, shuffle=rng)
    a = formats.read_matrix(p)
    assert np.array_equal(a.rstart, m2.rstart)
    assert np.array_equal(a.col, m2.col)
    assert np.array_equal(a.nonzero, m2.nonzero)


def test_large_file_threads_agree(tmp_path):
    m = generate_dd_matrix(GenSpec(n=20000, nnz=200000, seed=9))
    p = tmp_path / "big.txt"
    write_matrix(m, p, shuffle=np.random.default_rng(1))
    assert p.stat().st_size > (1 << 20)  # several chunks
    a = formats.read_matrix(p)
    assert np.array_equal(a.col, m.col) and np.array_equal(a.nonzero, m.nonzero)


def test_matrix_plain_but_odd_tokens(tmp_path):
    p = tmp_path / "odd.txt"
    p.write_text("# leading comment\r\n\r\n  matrix\t3 6 # trailing\r\n"
                 "+2 0 .5\n"
                 "0 002 5.\n"
                 "1 1 1E-3   # comment\n"
                 "\t0 0 -0.0\n"          # explicit zero: dropped
                 "2 2 12345678901234.5\n"
                 "1 0 -1e+300\n")
    a = formats.read_matrix(p)
    rs, c, v = expected_csr(3, [(2, 0, float(".5")), (0, 2, float("5.")), (1, 1, float("1E-3")),
                                (0, 0, -0.0), (2, 2, float("12345678901234.5")),
                                (1, 0, float("-1e+300"))])
    assert np.array_equal(a.rstart, rs) and np.array_equal(a.col, c)
    assert np.array_equal(a.nonzero, v)


@pytest.mark.parametrize("body", [
    "matrix 2 1\n0 1 1_0.5\n",     # underscores: Python accepts, fast path defers
    "matrix 2 1\n0 1 inf\n",
    "matrix 2 2\n0 1 0.5\n0 1 0.5\n",  # duplicate
    "matrx 2 2\n",
    "matrix 2 3\n0 1 0.5\n",       # wrong count
    "matrix 2 1\n0 x 0.5\n",
    "matrix 2 1\n0 5 0.5\n",       # out of range
    "matrix 2 1\r0 1 0.5\n",       # lone carriage return
    "",
])
def test_matrix_outside_fast_subset_is_deferred(tmp_path, body):
    p = tmp_path / "bad.txt"
    p.write_bytes(body.encode())
    assert rc_of("mcr_read_matrix", p) == _lib.MCR_UNSUPPORTED_INPUT


def test_vector_round_trip(tmp_path):
    v = np.random.default_rng(4).uniform(-1, 1, 1000) / 3.0
    p = tmp_path / "v.txt"
    p.write_text(f"vector {len(v)}\n" + "".join(fmt(x) + "\n" for x in v))
    assert np.array_equal(formats.read_vector(p), v)
    p.write_text("vector 2\n1.5\n")
    assert rc_of("mcr_read_vector", p) == _lib.MCR_UNSUPPORTED_INPUT


DEMO = """\
dtmc
states 4
initial 0
goal 3
# transitions may come in any order
2 0 0.4
0 2 0.5
0 3 0.5
1 1 1
2 1 0.6
3 3 1
"""


def test_dtmc_demo(tmp_path):
    p = tmp_path / "demo.dtmc"
    p.write_text(DEMO)
    chain, goals = formats.read_dtmc(p)
    assert chain.n == 4 and chain.initial == 0
    assert set(getattr(goals, "members", goals)) == {3}
    t = chain.transitions
    assert t.rstart.tolist() == [0, 2, 3, 5, 6]
    assert t.col.tolist() == [2, 3, 1, 0, 1, 3]
    assert t.nonzero.tolist() == [0.5, 0.5, 1.0, 0.4, 0.6, 1.0]


def test_dtmc_random_chain_round_trip(tmp_path):
    d = random_dtmc(5000, 3)
    t = d.transitions
    rows = np.repeat(np.arange(d.n), np.diff(t.rstart))
    order = np.random.default_rng(0).permutation(t.m)
    body = [f"{rows[k]} {t.col[k]} {fmt(t.nonzero[k])}" for k in order]
    head = ["dtmc", f"states {d.n}", f"initial {d.initial}",
            "goal " + " ".join(str(g) for g in d.goals)]
    p = tmp_path / "c.dtmc"
    p.write_text("\n".join(head[:2] + body[:10] + head[2:] + body[10:]) + "\n")  # keywords late
    chain, goals = formats.read_dtmc(p)
    assert np.array_equal(chain.transitions.rstart, t.rstart)
    assert np.array_equal(chain.transitions.col, t.col)
    assert np.array_equal(chain.transitions.nonzero, t.nonzero)
    assert sorted(getattr(goals, "members", goals)) == d.goals.tolist()


@pytest.mark.parametrize("body", [
    "dtmc\nstates 2\ngoal 1\n0 1 1\n1 1 1\n",                      # missing initial
    "states 2\n",                                                  # dtmc not first
    "dtmc\nstates 2\ninitial 0\ngoal 1\n0 1 0.5\n0 1 0.5\n1 1 1\n",  # duplicate transition
    "dtmc\nstates 2\ninitial 0\ngoal 1\n0 1 0.9\n1 1 1\n",          # row sum
    "dtmc\nstates 2\ninitial 0\ngoal 5\n0 1 1\n1 1 1\n",            # goal out of range
    "dtmc\nstates 2\nstates 2\ninitial 0\ngoal 1\n0 1 1\n1 1 1\n",   # duplicate keyword
    "dtmc\nstates 2\ninitial 0\ngoal 1\n0 1 1.5\n1 1 1\n",          # probability > 1
])
def test_dtmc_outside_fast_subset_is_deferred(tmp_path, body):
    p = tmp_path / "bad.dtmc"
    p.write_text(body)
    assert rc_of("mcr_read_dtmc", p) == _lib.MCR_UNSUPPORTED_INPUT


def test_errors_are_the_references(tmp_path):
    mf = pytest.importorskip("mcreach.formats")
    p = tmp_path / "c.dtmc"
    p.write_text("dtmc\nstates 2\ninitial 0\ngoal 1\n0 1 0.5\n0 1 0.5\n1 1 1\n")
    with pytest.raises(mf.ParseError) as err:
        formats.read_dtmc(p)
    assert err.value.line == 6
    p.write_text("matrix 2 1\n0 1 1_0.5\n")    # valid for Python, deferred: same result
    assert formats.read_matrix(p).nonzero.tolist() == [10.5]


def test_against_reference_reader(tmp_path):
    mf = pytest.importorskip("mcreach.formats")
    m = generate_dd_matrix(GenSpec(n=400, nnz=4000, seed=2))
    p = tmp_path / "m.txt"
    write_matrix(m, p, shuffle=np.random.default_rng(3), extra="# made by the test\n")
    a, r = formats.read_matrix(p), mf.read_matrix(p)
    assert np.array_equal(a.rstart, r.rstart) and np.array_equal(a.col, r.col)
    assert np.array_equal(a.nonzero, r.nonzero)


MATRIX_BODIES = [
    "matrix 2 1\n0 1 1_0.5\n",
    "matrix 2 1\n0 1 inf\n",
    "matrix 2 1\n0 1 nan\n",
    "matrix 2 2\n0 1 0.5\n0 1 0.5\n",
    "matrx 2 2\n",
    "matrix 2 3\n0 1 0.5\n",
    "matrix 2 1\n0 x 0.5\n",
    "matrix 2 1\n0 1 0.5 7\n",
    "matrix 2 1\n0 5 0.5\n",
    "matrix -1 0\n",
    "matrix 2 1\r0 1 0.5\n",
    "matrix 3 2\n0 1 1e400\n2 2 -0\n",
    "",
    "# only a comment\n",
]
VECTOR_BODIES = ["vector 2\n1.5\n", "vector 1\n1 2\n", "vectr 1\n1\n", "vector 2\n1\ninf\n", ""]
DTMC_BODIES = [
    "dtmc\nstates 2\ngoal 1\n0 1 1\n1 1 1\n",
    "states 2\n",
    "dtmc\nstates 2\ninitial 0\ngoal 1\n0 1 0.5\n0 1 0.5\n1 1 1\n",
    "dtmc\nstates 2\ninitial 0\ngoal 1\n0 1 0.9\n1 1 1\n",
    "dtmc\nstates 2\ninitial 0\ngoal 5\n0 1 1\n1 1 1\n",
    "dtmc\nstates 2\nstates 2\ninitial 0\ngoal 1\n0 1 1\n1 1 1\n",
    "dtmc\nstates 2\ninitial 0\ngoal 1\n0 1 1.5\n1 1 1\n",
    "dtmc\nstates 2\ninitial 7\ngoal 1\n0 1 1\n1 1 1\n",
    "dtmc\nstates 2\ninitial 0\ngoal 1\n0 3 1\n1 1 1\n",
    "dtmc\nstates 2\ninitial 0\ngoal\n0 1 1\n1 1 1\n",
    "dtmc\nstates 2\ninitial 0\ngoal 1\n0 1 0.5 9\n1 1 1\n",
    "dtmc\nstates 0\ninitial 0\ngoal 0\n",
    "dtmc\nstates 3\ninitial 0\ngoal 2\n0 1 0.25\n0 2 0.75\n1 1 1\n2 2 1_0e-1\n",
    "dtmc\nstates 2\ninitial 0\ngoal 1\n0 1 -0.5\n0 0 1.5\n1 1 1\n",
    "",
]


def _outcome(fn, path):
    try:
        r = fn(path)
    except Exception as err:  # noqa: BLE001
        return ("error", type(err).__name__, str(err), getattr(err, "line", None))
    if isinstance(r, tuple):
        chain, goals = r
        t = chain.transitions
        return ("ok", t.rstart.tolist(), t.col.tolist(), np.asarray(t.nonzero).tobytes(),
                chain.initial, sorted(getattr(goals, "members", goals)))
    if hasattr(r, "rstart"):
        return ("ok", r.rstart.tolist(), r.col.tolist(), np.asarray(r.nonzero).tobytes())
    return ("ok", np.asarray(r, dtype=np.float64).tobytes())


@pytest.mark.parametrize("kind,body", [("matrix", b) for b in MATRIX_BODIES]
                         + [("vector", b) for b in VECTOR_BODIES]
                         + [("dtmc", b) for b in DTMC_BODIES])
def test_outside_fast_subset_same_as_reference(tmp_path, kind, body):
    """Files the C++ readers refuse: the package's own readers give the reference reader's
    result or its exact error (class, message, line number)."""
    mf = pytest.importorskip("mcreach.formats")
    p = tmp_path / f"f.{kind}"
    p.write_bytes(body.encode())
    ours = _outcome(getattr(formats, f"read_{kind}"), p)
    ref = _outcome(getattr(mf, f"read_{kind}"), p)
    assert ours == ref, (body, ours, ref)
    if ours[0] == "error":  # the reference's own exception classes
        try:
            getattr(formats, f"read_{kind}")(p)
        except Exception as err:  # noqa: BLE001
            assert type(err).__module__.startswith("mcreach"), type(err)


def test_mirrors_without_the_reference(tmp_path, monkeypatch):
    """Without mcreach importable the mirrors carry the same messages and fields."""
    from paper_1210_6412_b200 import textio
    monkeypatch.setattr(textio, "_ref", lambda module: None)
    p = tmp_path / "c.dtmc"
    p.write_text("dtmc\nstates 2\ninitial 0\ngoal 1\n0 1 0.5\n0 1 0.5\n1 1 1\n")
    with pytest.raises(textio.ParseError) as err:
        textio.read_dtmc_parts(p)
    assert err.value.line == 6 and "duplicate transition 0 -> 1 (first on line 5)" in str(err.value)
    p.write_text("dtmc\nstates 2\ninitial 0\ngoal 1\n0 1 0.9\n1 1 1\n")
    with pytest.raises(textio.RowSumError) as err:
        textio.read_dtmc_parts(p)
    assert err.value.state == 0 and str(err.value) == "row 0 sums to 0.9, expected 1"
    p.write_text("matrix 2 2\n0 1 0.5\n0 1 0.25\n")
    from paper_1210_6412_b200.sparse import DuplicateEntry
    with pytest.raises(DuplicateEntry):
        textio.read_matrix(p)


def test_row_sums_left_to_right():
    """validate's row sums add each row's entries in column order from 0.0 (scipy's
    csr_matvec with a vector of ones), not pairwise."""
    from paper_1210_6412_b200 import textio
    from paper_1210_6412_b200.sparse import csr_from_triplets
    rng = np.random.default_rng(3)
    for _ in range(20):
        n = int(rng.integers(1, 40))
        ent = [(i, j, float(rng.uniform(0, 1))) for i in range(n) for j in range(n) if rng.random() < 0.5]
        p = csr_from_triplets(n, ent)
        want = np.zeros(n)
        for i in range(n):
            acc = 0.0
            for k in range(p.rstart[i], p.rstart[i + 1]):
                acc = acc + float(p.nonzero[k])
            want[i] = acc
        assert np.array_equal(textio.row_sums(p), want)
