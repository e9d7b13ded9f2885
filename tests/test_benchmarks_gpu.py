"""The C++ benchmark harness (benchmarks/bench_attention_b200.cpp) runs on the GPU: the
reference's bench_attention cases through the drop-in plus device-timed BM_Decode lines."""
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def test_cpp_bench_runs(built):
    exe = ROOT / "benchmarks" / "bench_attention_b200"
    if not exe.exists():
        pytest.skip("benchmarks/bench_attention_b200 not built")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    for case in ("BM_ExactAttention/64/256", "BM_ExactAttention/128/8192", "BM_SplitMerge/4096",
                 "BM_Decode/c2_llama2_7b_B64_l4096", "BM_Decode/c3_llama2_70b_B128_l4096"):
        assert case in r.stdout, r.stdout
    gbs = [float(m) for m in re.findall(r"BM_Decode/\S+\s+[0-9.]+ us\s+([0-9.]+) GB/s", r.stdout)]
    assert len(gbs) == 3 and min(gbs) > 1000.0, r.stdout  # device-resident decode streams at TB/s
    assert "BM_MultiHeadAttention/C1" in r.stdout
