"""Text ingest at C2' scale: write a 1e6-state random DTMC in the reference's
chain format, then time the multithreaded reader against the reference's read_dtmc, and the
whole `solve` command (read + build + solve) for both."""
import io, json, os, sys, time, contextlib
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "baseline", "_ref")]
import numpy as np
from paper_1210_6412_b200 import formats
from paper_1210_6412_b200.chains import random_dtmc
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
path = f"/tmp/chain_{n}.dtmc"
d = random_dtmc(n, 4)
t = d.transitions
rows = np.repeat(np.arange(n), np.diff(t.rstart))
with open(path, "w") as fh:
    fh.write(f"dtmc\nstates {n}\ninitial {d.initial}\ngoal {' '.join(map(str, d.goals))}\n")
    fh.writelines(f"{r} {c} {format(float(v), '.17g')}\n" for r, c, v in zip(rows, t.col, t.nonzero))
out = {"n": n, "transitions": int(t.m), "file_mb": os.path.getsize(path) / 1e6, "cores": os.cpu_count()}
t0 = time.perf_counter(); ch, g = formats.read_dtmc(path); out["fast_read_s"] = time.perf_counter() - t0
assert np.array_equal(ch.transitions.nonzero, t.nonzero)
from mcreach import formats as mf
from mcreach.cli import main as ref_main
from paper_1210_6412_b200.__main__ import main as gpu_main
t0 = time.perf_counter(); rc, rg = mf.read_dtmc(path); out["reference_read_s"] = time.perf_counter() - t0
assert np.array_equal(rc.transitions.nonzero, ch.transitions.nonzero)
for name, fn, argv in (("gpu_solve_cli_s", gpu_main, ["solve", "--input", path, "--gpu"]),
                       ("reference_solve_cli_s", ref_main, ["solve", "--input", path, "--parallel"])):
    buf = io.StringIO()
    t0 = time.perf_counter()
    with contextlib.redirect_stdout(buf):
        code = fn(argv)
    out[name] = time.perf_counter() - t0
    out[name[:-2] + "_stdout"] = buf.getvalue().strip()
print(json.dumps(out), flush=True)
