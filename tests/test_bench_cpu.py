"""CPU: bench.py's reference arm (the driver's `--impl reference`) and the JSON contract."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, check=True).stdout
    lines = [ln for ln in out.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "solves/s" and d["higher_is_better"]
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["iterations"]["jacobi"] == 3541          # C1 trial 0, as the reference


def test_algorithmic_bytes():
    sys.path.insert(0, ROOT)
    import bench
    ab = bench.alg_bytes(10 ** 6, 10 ** 7, 9 * 10 ** 6)
    assert ab["spmv"] == 12 * 10 ** 7 + 8 * (10 ** 6 + 1) + 16 * 10 ** 6
    assert ab["jacobi_sweep"] == 12 * 9 * 10 ** 6 + 8 * (10 ** 6 + 1) + 32 * 10 ** 6
    assert ab["bicgstab_iteration"] == 2 * (12 * 10 ** 7 + 8 * (10 ** 6 + 1)) + 152 * 10 ** 6


def test_gpus_flag_is_honoured(monkeypatch):
    """--gpus N > 1 runs the row-sharded workload (run_sharded, n_gpus = N) rather than a
    single GPU; a WORLD_SIZE that disagrees with --gpus is an error."""
    sys.path.insert(0, ROOT)
    import bench
    seen = {}
    monkeypatch.setattr(bench, "run_sharded", lambda args: seen.setdefault("sharded", args.gpus) and 0)
    monkeypatch.setattr(bench, "run_ours", lambda args: seen.setdefault("single", args.gpus) and 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2", "--steps", "1", "--warmup", "0"])
    bench.main()
    assert seen == {"sharded": 2}
    seen.clear()
    monkeypatch.setattr(sys, "argv", ["bench.py", "--steps", "1", "--warmup", "0"])
    bench.main()
    assert seen == {"single": 1}
    monkeypatch.setenv("WORLD_SIZE", "4")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2"])
    import pytest
    with pytest.raises(SystemExit):
        bench.main()
