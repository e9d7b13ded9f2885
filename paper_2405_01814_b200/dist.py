"""KV-head-sharded attention worker pool over torch.distributed (NCCL on GPUs, gloo on CPU).

The paper's attention-offload step (reference SPEC/PAPER; modeled analytically in
core/src/sim.cpp:286-346) on N GPUs of one box:

* head_partition (attention.cpp:164-177): rank j owns KV heads [j*Hkv/N, (j+1)*Hkv/N) of every
  request, and therefore q heads [j*Hq/N, (j+1)*Hq/N).  Sharding by heads needs no
  cross-GPU reduction: outputs concatenate by head exactly (test_attention.cpp:237-256).
* Every rank is also a model worker for B_local requests.  Per layer it scatters those
  requests' Q, K_new, V_new to the head owners and gathers the attention outputs back —
  the send-Q / send-KV / return-output messages of sim.cpp:310-316, (2 + 2/G) e d B per layer
  (perf.cpp:142-148), as NCCL all-to-alls.
* Two staggered micro-batches (the n = 2 rotational schedule, pipeline.cpp:30-33, 44-118):
  micro-batch 1's scatter and micro-batch 0's gather run on a communication stream while the
  other micro-batch's attention runs on the compute stream, so the step approaches
  max(attention, communication) (sim.cpp:374-379).

Layouts (all contiguous, micro-batch outermost so every collective moves one contiguous
buffer): inputs qkv_in [L, MB, N, Bh, W, D] with W = hq_l + 2 hkv_l — per destination head shard
(the N axis) each request's packed QKV-projection rows [q heads | k heads | v heads], the layout a
QKV GEMM produces — so one all-to-all per (layer, micro-batch) carries Q, K_new and V_new;
outputs out [L, MB, N, Bh, hq_l, D] where N is the source head shard.  The receiving side
decodes q and appends k/v straight out of the packed buffer (batch strides, no repacking).  On the attention side request r of micro-batch m from source s is row
m*N*Bh + s*Bh + i of the KV store, so a micro-batch is a contiguous slice of the page table.
The local append/attend ops are injected: the GPU path passes our kernels (lam_kv_append,
lam_decode); the CPU gloo test passes the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch


@dataclass
class ShardGeometry:
    rank: int
    world: int
    layers: int
    B_local: int
    Hq: int
    Hkv: int
    D: int
    micro_batches: int = 2

    def __post_init__(self):
        if self.Hkv % self.world:
            raise ValueError(
                f"head partition requires num_kv_heads divisible by num_devices "
                f"({self.Hkv} % {self.world} != 0)")
        if self.B_local % self.micro_batches:
            raise ValueError("B_local must split evenly into micro-batches")

    @property
    def hq_l(self) -> int:
        return self.Hq // self.world

    @property
    def hkv_l(self) -> int:
        return self.Hkv // self.world

    @property
    def Bh(self) -> int:
        return self.B_local // self.micro_batches

    @property
    def B_mb(self) -> int:
        """requests per micro-batch on the attention side"""
        return self.world * self.Bh

    @property
    def B_attn(self) -> int:
        return self.world * self.B_local

    def kv_row(self, src: int, b_local: int) -> int:
        """attention-side row of request b_local of model worker src"""
        m, i = divmod(b_local, self.Bh)
        return m * self.B_mb + src * self.Bh + i

    @property
    def W(self) -> int:
        """packed rows per request and shard: q heads, k heads, v heads"""
        return self.hq_l + 2 * self.hkv_l

    def q_shape(self):
        return (self.layers, self.micro_batches, self.world, self.Bh, self.hq_l, self.D)

    def qkv_shape(self):
        return (self.layers, self.micro_batches, self.world, self.Bh, self.W, self.D)


class HeadShardedAttention:
    """One rank of the attention worker pool.

    append(layer, mb, k[B_mb, hkv_l, D], v[...])          writes the new tokens
    attend(layer, mb, q[B_mb, hq_l, D], out[B_mb, hq_l, D])  local decode attention
    With append=None, attend(layer, mb, q, k, v, out) does both (the fused decode launch).
    """

    def __init__(self, geo: ShardGeometry, dist, append: Callable, attend: Callable,
                 device: torch.device, dtype: torch.dtype):
        self.geo, self.dist = geo, dist
        self.append_fn, self.attend_fn = append, attend
        self.device, self.dtype = device, dtype
        g = geo
        MB = g.micro_batches
        # attention-side receive / send buffers, one per micro-batch
        self.qkv_r = [torch.empty((g.world, g.Bh, g.W, g.D), dtype=dtype, device=device)
                      for _ in range(MB)]
        self.o_l = [torch.empty((g.world, g.Bh, g.hq_l, g.D), dtype=dtype, device=device)
                    for _ in range(MB)]
        self.cuda = device.type == "cuda"
        if self.cuda:
            self.comm = torch.cuda.Stream(device=device)
            self.compute = torch.cuda.current_stream(device)
            self.h2d = torch.cuda.Stream(device=device)  # copy engines: host inputs in ...
            self.d2h = torch.cuda.Stream(device=device)  # ... and outputs back out

    # ---- collectives ----
    def _a2a(self, out: torch.Tensor, inp: torch.Tensor):
        self.dist.all_to_all_single(out, inp)

    def step(self, qkv_in, out, ev=None, host_in=None, host_out=None):
        """One decode step over all layers; returns when the work is enqueued (CUDA) or done
        (CPU).  `ev`, if given, is a list of (start, end) CUDA event pairs, one per local
        attention launch, recorded on the compute stream.  With pinned `host_in` / `host_out`
        (shapes of qkv_in / out) the step starts from host memory: every layer's inputs are copied
        in on a copy stream ahead of their scatter and every layer's outputs copied back as soon
        as they are gathered, both hidden under the attention of other layers."""
        g = self.geo
        MB = g.micro_batches
        if not self.cuda:
            for layer in range(g.layers):
                for m in range(MB):
                    self._scatter(layer, m, qkv_in)
                    self._attend(layer, m, None)
                    self._a2a(out[layer, m], self.o_l[m])
            return
        comm, comp = self.comm, self.compute
        comm.wait_stream(comp)  # inputs produced on the compute stream are visible
        scat = [[torch.cuda.Event() for _ in range(MB)] for _ in range(g.layers)]
        done = [[torch.cuda.Event() for _ in range(MB)] for _ in range(g.layers)]
        gath = [torch.cuda.Event() for _ in range(MB)]
        arrived = None
        if host_in is not None:  # every layer has its own input slot: copy them all ahead
            self.h2d.wait_stream(comp)
            arrived = [torch.cuda.Event() for _ in range(g.layers)]
            with torch.cuda.stream(self.h2d):
                for layer in range(g.layers):
                    qkv_in[layer].copy_(host_in[layer], non_blocking=True)
                    arrived[layer].record(self.h2d)
        if host_out is not None:
            self.d2h.wait_stream(comp)

        def scatter(layer, m):
            with torch.cuda.stream(comm):
                if layer > 0:
                    # micro-batch m's next layer follows its previous output gather (data
                    # dependency through the model worker) and the reuse of its receive buffers
                    comm.wait_event(done[layer - 1][m])
                if arrived is not None and m == 0:
                    comm.wait_event(arrived[layer])
                self._scatter(layer, m, qkv_in)
                scat[layer][m].record(comm)

        def gather(layer, m):
            with torch.cuda.stream(comm):
                comm.wait_event(done[layer][m])
                self._a2a(out[layer, m], self.o_l[m])
                gath[m].record(comm)
            if host_out is not None:
                self.d2h.wait_event(gath[m])
                with torch.cuda.stream(self.d2h):
                    host_out[layer, m].copy_(out[layer, m], non_blocking=True)

        for m in range(MB):
            scatter(0, m)
        k = 0
        for layer in range(g.layers):
            for m in range(MB):
                comp.wait_event(scat[layer][m])
                if layer > 0:
                    comp.wait_event(gath_prev[m])  # o_l[m] free again
                e = ev[k] if ev is not None else None
                k += 1
                self._attend(layer, m, e)
                done[layer][m].record(comp)
                gather(layer, m)
                if layer + 1 < g.layers:
                    scatter(layer + 1, m)
            gath_prev = list(gath)
            gath = [torch.cuda.Event() for _ in range(MB)]
        comp.wait_stream(comm)
        if host_out is not None:
            comp.wait_stream(self.d2h)

    def _scatter(self, layer, m, qkv_in):
        self._a2a(self.qkv_r[m], qkv_in[layer, m])

    def _attend(self, layer, m, e):
        g = self.geo
        packed = self.qkv_r[m].view(g.B_mb, g.W, g.D)
        q = packed[:, : g.hq_l]
        k = packed[:, g.hq_l: g.hq_l + g.hkv_l]
        v = packed[:, g.hq_l + g.hkv_l:]
        out = self.o_l[m].view(g.B_mb, g.hq_l, g.D)
        if self.append_fn is not None:
            self.append_fn(layer, m, k, v)
        if e is not None:
            e[0].record(self.compute)
        if self.append_fn is None:
            self.attend_fn(layer, m, q, k, v, out)
        else:
            self.attend_fn(layer, m, q, out)
        if e is not None:
            e[1].record(self.compute)


def stitch_outputs(out: torch.Tensor) -> torch.Tensor:
    """[L, MB, N(src shard), Bh, hq_l, D] -> [L, B_local, Hq, D] head-major (test helper and
    the layout a consumer of concatenated heads expects)."""
    L, MB, N, Bh, hq_l, D = out.shape
    return out.permute(0, 1, 3, 2, 4, 5).reshape(L, MB * Bh, N * hq_l, D)


def shard_inputs(q: torch.Tensor, kn: torch.Tensor, vn: torch.Tensor, world: int,
                 micro_batches: int = 2) -> torch.Tensor:
    """[L, B_local, H, D] head-major model-worker tensors -> packed destination-major send
    layout [L, MB, N, Bh, hq_l + 2 hkv_l, D]."""
    L, B, Hq, D = q.shape
    Hkv = kn.shape[2]
    Bh = B // micro_batches

    def f(x, H):
        return x.view(L, micro_batches, Bh, world, H // world, D).permute(0, 1, 3, 2, 4, 5)

    return torch.cat([f(q, Hq), f(kn, Hkv), f(vn, Hkv)], dim=4).contiguous()
