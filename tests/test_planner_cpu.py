"""Planner feedback (§8(f) rows 3-4) on CPU: the exported B200 catalog loads through the
reference's OWN loaders and validators (model.cpp), the restated capacity planner (perf.max_batch)
equals the reference's max_batch (perf.cpp:130-140) on every point, and the catalog's measured
numbers are those of the committed bench lines."""
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
CAT = ROOT / "integration" / "b200_catalog.json"
CHECK = ROOT / "oracle" / "_ref" / "catalog_check"


def _ref_lines():
    if not CHECK.exists():
        pytest.skip("oracle/_ref/catalog_check not built (needs /root/reference)")
    r = subprocess.run([str(CHECK), str(CAT)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr  # the reference's validators accept every entry
    return [json.loads(ln) for ln in r.stdout.splitlines()]


def test_catalog_loads_through_reference_loaders():
    lines = _ref_lines()
    cat = json.loads(CAT.read_text())
    devices = [ln for ln in lines if "device" in ln]
    assert [d["device"] for d in devices] == [d["name"] for d in cat["devices"]]
    assert devices[0]["mem_bytes"] == cat["devices"][0]["mem_bytes"]


def test_max_batch_matches_reference():
    from paper_2405_01814_b200 import perf as PF

    specs = {"llama-2-7b": PF.LLAMA2_7B, "llama-2-70b": PF.LLAMA2_70B}
    pts = [ln for ln in _ref_lines() if "model" in ln]
    assert len(pts) == 16
    for p in pts:
        spec = specs[p["model"]]
        assert p["kv_bytes_per_token"] == PF.kv_bytes_per_token(spec)
        assert PF.max_batch(p["gpus"] * PF.B200_MEM_BYTES, 0.0, spec, p["seq_len"]) == p["max_batch"]


def test_catalog_capacity_and_measurements_are_consistent():
    from paper_2405_01814_b200 import perf as PF

    cat = json.loads(CAT.read_text())
    specs = {"llama-2-7b": PF.LLAMA2_7B, "llama-2-70b": PF.LLAMA2_70B}
    for p in cat["capacity"]["points"]:
        assert p["max_batch"] == PF.max_batch(p["gpus"] * PF.B200_MEM_BYTES, 0.0, specs[p["model"]],
                                              p["seq_len"])
    for model, m in cat["measured"].items():
        if not isinstance(m, dict):
            continue
        line = json.loads([ln for ln in open(ROOT / m["source"]) if ln.startswith("{")][-1])
        assert m["attn_kv_gbs_per_gpu"] == pytest.approx(line["value"] / line["n_gpus"])
        assert m["attn_mbu"] == pytest.approx(line["value"] / line["n_gpus"] * 1e9 / 8e12, abs=1e-4)
        assert 0.8 <= m["attn_mbu"] <= 1.0  # measured, replacing the 0.80 knob
    nv = cat["net_presets"][0]
    assert nv["name"] == "NVLINK-PEER" and 0 < nv["base_latency_s"] < 16.5e-6
    assert nv["achievable_bw"] > 45.7e9  # vs the reference's FHBN


def test_max_batch_known_answers_and_errors():
    from paper_2405_01814_b200 import perf as PF

    # 2 e (d/G) L = 2*2*1024*80 = 327,680 B/token for LLaMA-2-70B; 0.95 * 180 GB / (327680 * 4096)
    assert PF.max_batch(180e9, 0.0, PF.LLAMA2_70B, 4096) == 127
    assert PF.max_batch(8 * 180e9, 0.0, PF.LLAMA2_70B, 32768) == 127
    with pytest.raises(RuntimeError):
        PF.max_batch(100e9, 138e9, PF.LLAMA2_70B, 4096)
    with pytest.raises(ValueError):
        PF.max_batch(180e9, 0.0, PF.LLAMA2_70B, 0)
