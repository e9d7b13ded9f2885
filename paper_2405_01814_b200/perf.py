"""The reference's analytic byte/flop contract for the attention operator
(reference core/src/perf.cpp:64-88,118-148; core/include/disagg/perf.hpp:59-94).

bench.py computes roofline.achieved from these formulas, so the reported bandwidth is the
reference's own definition of attention traffic: KV-cache reads only (perf.hpp:64-68).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class LlmSpec:
    """The fields of reference LlmSpec (model.hpp:46-61) the attention contract reads."""

    name: str
    hidden_dim: int       # d
    layers: int           # L
    gqa_group: int = 1    # G
    bytes_per_elem: int = 2  # e
    num_heads: int = 0    # query heads (0 => hidden_dim / 128, model.cpp:166-175)

    @property
    def q_heads(self) -> int:
        return self.num_heads or self.hidden_dim // 128

    @property
    def kv_heads(self) -> int:
        return self.q_heads // self.gqa_group

    @property
    def head_dim(self) -> int:
        return self.hidden_dim // self.q_heads


@dataclass(frozen=True)
class OpCost:
    flops: float
    bytes: float


def kv_bytes_per_token(spec: LlmSpec) -> float:
    """2 e (d/G) L (perf.cpp:123-128)."""
    return 2.0 * spec.bytes_per_elem * (spec.hidden_dim // spec.gqa_group) * spec.layers


def attn_cost(spec: LlmSpec, batch: int, seq_len: int) -> OpCost:
    """flops = 4 l d L B, bytes = kv_bytes_per_token * l * B (perf.cpp:77-88)."""
    if batch < 1:
        raise ValueError("batch must be >= 1")
    if seq_len < 1:
        raise ValueError("seq_len must be >= 1")
    return OpCost(4.0 * seq_len * spec.hidden_dim * spec.layers * batch,
                  kv_bytes_per_token(spec) * seq_len * batch)


def attn_cost_ragged(spec: LlmSpec, seq_lens) -> OpCost:
    """attn_cost summed over per-request lengths (mixed-length continuous batch)."""
    total = float(sum(int(x) for x in seq_lens))
    return OpCost(4.0 * total * spec.hidden_dim * spec.layers, kv_bytes_per_token(spec) * total)


def mbu(bytes_: float, seconds: float, mem_bw: float) -> float:
    """bytes / (t * bw) (perf.cpp:118-121)."""
    if seconds <= 0:
        raise ValueError("mbu requires time > 0")
    return bytes_ / (seconds * mem_bw)


def comm_volume(spec: LlmSpec, batch: int) -> float:
    """(2 + 2/G) e d B L bytes across the pool boundary per step (perf.cpp:142-148)."""
    if batch < 1:
        raise ValueError("batch must be >= 1")
    g = float(spec.gqa_group)
    return (2.0 + 2.0 / g) * spec.bytes_per_elem * spec.hidden_dim * batch * spec.layers


# The BASELINE.json configurations' model shapes.
LLAMA_7B_1L_F32 = LlmSpec("llama-7b-1layer-fp32", 4096, 1, 1, 4, 32)
LLAMA2_7B = LlmSpec("llama-2-7b", 4096, 32, 1, 2, 32)
LLAMA2_70B = LlmSpec("llama-2-70b", 8192, 80, 8, 2, 64)


def max_batch(pool_mem_bytes: float, reserved_weight_bytes: float, spec: LlmSpec, seq_len: int,
              headroom_frac: float = 0.05) -> int:
    """Requests of seq_len tokens whose KV fits a memory pool (perf.cpp:130-140):
    floor((pool - weights - headroom * pool) / (kv_bytes_per_token * seq_len))."""
    import math

    if seq_len < 1:
        raise ValueError("seq_len must be >= 1")
    if not 0 <= headroom_frac < 1:
        raise ValueError("headroom_frac must be in [0,1)")
    free = pool_mem_bytes - reserved_weight_bytes - headroom_frac * pool_mem_bytes
    if free <= 0:
        raise RuntimeError("model weights plus headroom exceed pool memory")
    return int(math.floor(free / (kv_bytes_per_token(spec) * seq_len)))


# B200 attention-worker memory as the planner sees it (DeviceSpec.mem_bytes, model.hpp:64-74):
# 180 GB of HBM3e per GPU; the paged pool the bench allocates is what remains after the
# framework's own buffers (bench.py keeps 6 GiB free).
B200_MEM_BYTES = 180e9
