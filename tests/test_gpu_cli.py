"""`python -m paper_1210_6412_b200` = the reference CLI (mcreach.cli) with the GPU methods
(SURVEY.md 8f item 1). Modelled on the reference's own T/test_cli.py."""

import csv

import pytest

pytestmark = pytest.mark.gpu

DEMO_DTMC = """\
dtmc
states 4
initial 0
goal 3
0 2 0.5
0 3 0.5
1 1 1
2 0 0.4
2 1 0.6
3 3 1
"""


@pytest.fixture
def demo_file(tmp_path):
    pytest.importorskip("mcreach")
    path = tmp_path / "demo.dtmc"
    path.write_text(DEMO_DTMC)
    return path


def run(capsys, main, *argv):
    code = main([str(a) for a in argv])
    cap = capsys.readouterr()
    return code, cap.out, cap.err


@pytest.mark.parametrize("method", ["jacobi", "bicgstab"])
def test_solve_gpu_matches_reference_output(demo_file, capsys, method):
    from mcreach.cli import main as ref_main
    from paper_1210_6412_b200.__main__ import main
    code, out, _ = run(capsys, main, "solve", "--input", demo_file, "--method", method, "--gpu",
                       "--full-vector")
    rcode, rout, _ = run(capsys, ref_main, "solve", "--input", demo_file, "--method", method,
                         "--full-vector")
    assert code == rcode == 0
    assert out == rout            # x0 = 0.625 (PAPER.md demo chain), identical digits
    assert out.splitlines()[0] == "0.625"


def test_bench_csv_rows_for_gpu_methods(tmp_path, capsys):
    pytest.importorskip("mcreach")
    from paper_1210_6412_b200.__main__ import main
    out = tmp_path / "t1.csv"
    code, _, err = run(capsys, main, "bench", "--table1", "--trials", "1", "--methods",
                       "jacobi-seq,jacobi-gpu,bicgstab-seq,bicgstab-gpu", "--output", out)
    assert code == 0, err
    rows = list(csv.DictReader(open(out)))
    assert len(rows) == 18 * 4
    by = {}
    for r in rows:
        by.setdefault((r["n"], r["m"]), {})[r["method"]] = r
    for cell in by.values():
        # Jacobi on the GPU is bit-identical: same sweep count as the reference's jacobi-seq
        assert cell["jacobi-gpu"]["iterations"] == cell["jacobi-seq"]["iterations"]
        assert cell["jacobi-gpu"]["converged"].lower() == "true"
        assert cell["bicgstab-gpu"]["converged"].lower() == "true"
        # BiCGStab too: the GPU sums its inner products in the reference's order
        assert cell["bicgstab-gpu"]["iterations"] == cell["bicgstab-seq"]["iterations"]


def test_unknown_method_still_rejected(tmp_path, capsys):
    pytest.importorskip("mcreach")
    from paper_1210_6412_b200.__main__ import main
    with pytest.raises(SystemExit):
        main(["bench", "--methods", "jacobi-tpu", "--output", str(tmp_path / "x.csv")])
