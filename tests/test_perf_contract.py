"""The byte/flop contract bench.py reports against is the reference's own
(perf.cpp:77-88,123-128,142-148); check it against the reference's test_perf.cpp answers."""
import pytest

from paper_2405_01814_b200 import perf as P

LLAMA3_70B = P.LlmSpec("llama3-70b", 8192, 80, 8, 2, 64)
LLAMA_65B = P.LlmSpec("llama-65b", 8192, 80, 1, 2, 64)


def test_kv_bytes_per_token_known_answers():
    assert P.kv_bytes_per_token(LLAMA3_70B) == 327680.0  # test_perf.cpp:146-150
    assert P.kv_bytes_per_token(LLAMA_65B) == 2621440.0


def test_attn_cost_intensity_is_2g_over_e():
    for b in (1, 7, 300):
        for l in (1, 512, 8192):
            c = P.attn_cost(LLAMA3_70B, b, l)
            assert c.flops / c.bytes == 8.0
            c = P.attn_cost(LLAMA_65B, b, l)
            assert c.flops / c.bytes == 1.0
    assert P.attn_cost(LLAMA3_70B, 300, 8192).bytes == pytest.approx(8.053e11, rel=1e-3)


def test_baseline_config_bytes():
    # BASELINE.md section 3
    assert P.attn_cost(P.LLAMA_7B_1L_F32, 8, 1024).bytes == 268435456
    assert P.attn_cost(P.LLAMA2_7B, 64, 4096).bytes == pytest.approx(137.44e9, rel=1e-4)
    assert P.attn_cost(P.LLAMA2_70B, 128, 4096).bytes == pytest.approx(171.8e9, rel=1e-3)
    assert P.attn_cost(P.LLAMA2_70B, 32, 32768).bytes == pytest.approx(343.6e9, rel=1e-3)
    assert P.LLAMA2_70B.kv_heads == 8 and P.LLAMA2_70B.head_dim == 128
    assert P.comm_volume(P.LLAMA2_70B, 128) / 80 == pytest.approx(4.5 * 2**20, rel=1e-6)


def test_validation():
    with pytest.raises(ValueError):
        P.attn_cost(LLAMA3_70B, 0, 1)
    with pytest.raises(ValueError):
        P.mbu(1.0, 0.0, 1.0)
