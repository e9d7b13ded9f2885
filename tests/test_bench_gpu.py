"""bench.py checks its own benchmarked launch configuration against the CPU oracle after the
timed regions (check_outputs): run the default line (BASELINE config 2 at full size) and
config 5 (mixed lengths, request order) briefly and require the check to pass."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("workload", ["c2", "c5", "c1"])
def test_bench_checks_its_own_outputs(workload):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--workload", workload, "--steps", "2",
                        "--warmup", "3", "--no-e2e", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    chk = line["check"]
    assert chk["ok"] and chk["append_bit_exact"] and chk["pairs_per_rank"] >= 4, chk
    assert chk["max_abs"] <= chk["tol"]
