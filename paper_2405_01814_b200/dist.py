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

import os
from dataclasses import dataclass
from typing import Callable

import torch


def local_batch(batch: int, world: int, scaling: str = "strong", micro_batches: int = 2) -> int:
    """Requests each model worker produces.  strong: a fixed global batch is dealt out (request
    g = rank * B_local + b), so T1 / (N * TN) is the parallel efficiency at a fixed global batch
    (BASELINE.md §3); weak: every rank brings `batch` requests (global batch N * batch)."""
    if scaling == "weak":
        b = batch
    elif scaling == "strong":
        if batch % world:
            raise ValueError(f"global batch {batch} does not split over {world} ranks")
        b = batch // world
    else:
        raise ValueError("scaling must be 'strong' or 'weak'")
    if b % micro_batches:
        raise ValueError(f"{b} requests per rank do not split into {micro_batches} micro-batches")
    return b


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
                    self._gather(layer, m, out)
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
                self._gather(layer, m, out)
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

    def _gather(self, layer, m, out):
        self._a2a(out[layer, m], self.o_l[m])

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


class RequestGeometry:
    """Request-level partition of the attention worker pool (§8(f) row 4): every rank owns ALL
    KV heads of the requests `request_partition` (attention.cpp:179-203, greedy longest-first
    bin packing over KV sizes) assigns to it.  This is the fallback when num_kv_heads is not
    divisible by the number of devices (head_partition's ValidationError, attention.cpp:167-170),
    and it balances mixed-length batches by KV bytes instead of by head count.

    Global request r = s * B_local + b lives on model worker s; micro-batch m of every model
    worker is its local requests [m * Bh, (m + 1) * Bh).  Per (layer, micro-batch):
      * scatter: model worker s sends each of its micro-batch requests' packed QKV-projection
        rows [Hq + 2 Hkv][D] to owner[r] (one variable-split all-to-all); its send order is
        `send_order[m]`, i.e. its requests grouped by destination;
      * the owner decodes the rows it received — grouped by source, in the senders' order —
        over its KV store, where micro-batch m occupies rows [row_off[m], row_off[m] + n_recv[m]);
      * gather: the reverse all-to-all returns the outputs [Hq][D] in the sender's send order.
    """

    def __init__(self, rank: int, world: int, layers: int, B_local: int, Hq: int, Hkv: int,
                 D: int, owner, micro_batches: int = 2):
        if Hq % Hkv:
            raise ValueError("query heads must be a multiple of KV heads")
        if B_local % micro_batches:
            raise ValueError("B_local must split evenly into micro-batches")
        owner = [int(x) for x in owner]
        if len(owner) != world * B_local or any(not 0 <= d < world for d in owner):
            raise ValueError("owner must map every global request to a rank")
        self.rank, self.world, self.layers = rank, world, layers
        self.B_local, self.Hq, self.Hkv, self.D = B_local, Hq, Hkv, D
        self.micro_batches, self.owner = micro_batches, owner
        Bh = self.Bh
        # model-worker side: this rank's micro-batch requests grouped by destination (stable)
        self.send_order, self.send_counts = [], []
        # attention side: requests received per micro-batch, grouped by source, sender order
        self.recv_reqs, self.recv_counts, self.row_off = [], [], []
        off = 0
        for m in range(micro_batches):
            mb = range(m * Bh, (m + 1) * Bh)
            order = sorted(mb, key=lambda b: (owner[rank * B_local + b], b))
            self.send_order.append(order)
            self.send_counts.append([sum(owner[rank * B_local + b] == d for b in mb)
                                     for d in range(world)])
            reqs, counts = [], []
            for s in range(world):
                got = [s * B_local + b for b in sorted(range(m * Bh, (m + 1) * Bh),
                                                        key=lambda b: (owner[s * B_local + b], b))
                       if owner[s * B_local + b] == rank]
                reqs += got
                counts.append(len(got))
            self.recv_reqs.append(reqs)
            self.recv_counts.append(counts)
            self.row_off.append(off)
            off += len(reqs)
        self.B_attn = off  # requests this rank attends to (all micro-batches)

    @property
    def Bh(self) -> int:
        return self.B_local // self.micro_batches

    @property
    def W(self) -> int:
        return self.Hq + 2 * self.Hkv

    @property
    def rows(self) -> list:
        """attention-side KV rows: global request of every row of this rank's store"""
        return [r for reqs in self.recv_reqs for r in reqs]

    def send_order_of(self, s: int, m: int) -> list:
        """model worker s's micro-batch m requests (local indices) grouped by destination"""
        return sorted(range(m * self.Bh, (m + 1) * self.Bh),
                      key=lambda b: (self.owner[s * self.B_local + b], b))

    @property
    def R(self) -> int:
        """rows per micro-batch of a step launch: the largest micro-batch's received rows"""
        return max(1, max(len(x) for x in self.recv_reqs))

    def padded_rows(self) -> list:
        """the step launch's rows: micro-batch m's received requests in rows
        [m * R, m * R + n_recv[m]), then -1 (an empty row: length 0, no work, a scratch output)"""
        return [r for reqs in self.recv_reqs for r in reqs + [-1] * (self.R - len(reqs))]

    def q_shape(self):
        return (self.layers, self.micro_batches, self.Bh, self.Hq, self.D)

    def qkv_shape(self):
        return (self.layers, self.micro_batches, self.Bh, self.W, self.D)


class RequestShardedAttention(HeadShardedAttention):
    """The attention worker pool partitioned by request (RequestGeometry) with the same two
    staggered micro-batches and streams as HeadShardedAttention; only the exchange differs:
    variable-split all-to-alls of whole requests instead of equal head shards.

    qkv_in [L, MB, Bh, Hq + 2 Hkv, D] and out [L, MB, Bh, Hq, D] are in each micro-batch's
    send order (geo.send_order; `pack_request_inputs` / `unpack_request_outputs` convert).
    attend(layer, m, q, k, v, out) (fused) or append + attend work on the n_recv[m] rows that
    start at geo.row_off[m] of the local store, with all Hq / Hkv heads.
    """

    def __init__(self, geo: RequestGeometry, dist, append: Callable, attend: Callable,
                 device: torch.device, dtype: torch.dtype):
        self.geo, self.dist = geo, dist
        self.append_fn, self.attend_fn = append, attend
        self.device, self.dtype = device, dtype
        g = geo
        self.qkv_r = [torch.empty((sum(g.recv_counts[m]), g.W, g.D), dtype=dtype, device=device)
                      for m in range(g.micro_batches)]
        self.o_l = [torch.empty((sum(g.recv_counts[m]), g.Hq, g.D), dtype=dtype, device=device)
                    for m in range(g.micro_batches)]
        self.cuda = device.type == "cuda"
        if self.cuda:
            self.comm = torch.cuda.Stream(device=device)
            self.compute = torch.cuda.current_stream(device)
            self.h2d = torch.cuda.Stream(device=device)
            self.d2h = torch.cuda.Stream(device=device)

    def _scatter(self, layer, m, qkv_in):
        g = self.geo
        self.dist.all_to_all_single(self.qkv_r[m], qkv_in[layer, m],
                                    output_split_sizes=g.recv_counts[m],
                                    input_split_sizes=g.send_counts[m])

    def _gather(self, layer, m, out):
        g = self.geo
        self.dist.all_to_all_single(out[layer, m], self.o_l[m],
                                    output_split_sizes=g.send_counts[m],
                                    input_split_sizes=g.recv_counts[m])

    def _attend(self, layer, m, e):
        g = self.geo
        if self.qkv_r[m].shape[0] == 0:
            return
        packed = self.qkv_r[m]
        q = packed[:, : g.Hq]
        k = packed[:, g.Hq: g.Hq + g.Hkv]
        v = packed[:, g.Hq + g.Hkv:]
        out = self.o_l[m]
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


def pack_request_inputs(geo: RequestGeometry, q: torch.Tensor, kn: torch.Tensor,
                        vn: torch.Tensor) -> torch.Tensor:
    """[L, B_local, H, D] model-worker tensors -> [L, MB, Bh, Hq + 2 Hkv, D] in send order."""
    idx = torch.tensor([b for m in range(geo.micro_batches) for b in geo.send_order[m]],
                       dtype=torch.long, device=q.device)
    x = torch.cat([q, kn, vn], dim=2).index_select(1, idx)
    return x.view(q.shape[0], geo.micro_batches, geo.Bh, geo.W, geo.D).contiguous()


def unpack_request_outputs(geo: RequestGeometry, out: torch.Tensor) -> torch.Tensor:
    """[L, MB, Bh, Hq, D] in send order -> [L, B_local, Hq, D] in local request order."""
    L = out.shape[0]
    flat = out.reshape(L, geo.B_local, geo.Hq, geo.D)
    idx = [b for m in range(geo.micro_batches) for b in geo.send_order[m]]
    inv = torch.empty(geo.B_local, dtype=torch.long)
    inv[torch.tensor(idx)] = torch.arange(geo.B_local)
    return flat.index_select(1, inv.to(out.device))


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


class _DevView:
    """Wraps a raw device pointer for torch.as_tensor (CUDA array interface)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


class PeerShardedAttention:
    """One rank of the attention worker pool with the collectives replaced by peer memory.

    The same step as HeadShardedAttention (head_partition sharding, two staggered
    micro-batches) without NCCL on the data path — the device-initiated transport of the
    paper's FHBN design on NVLink / NVSwitch:

    * every rank, as model worker, keeps its packed QKV rows `qkv_in` [L, MB, N, Bh, W, D] and
      its output rows `out` [L, MB, N, Bh, hq_l, D] in HBM exported over CUDA IPC
      (lam_peer_alloc / lam_peer_open);
    * every rank, as attention worker, runs one lam_decode_peer launch per (layer,
      micro-batch) that TMA-loads each request's q / k_new / v_new straight from its model
      worker's qkv_in over NVLink (no scatter), appends the new token and stores the output
      rows straight into the model worker's `out` (no gather);
    * readiness travels as 32-bit sequence numbers written by the GPU stream front-end
      (lam_stream_signal / lam_stream_wait: no SM time, no host round trip):
      qkv_ready[m][s] (the model worker s's rows of layer l are in place) and
      out_ready[m][j] (attention worker j stored layer l's outputs).

    `launch_args(layer, m)` returns the lam_decode_args of the local launch (pools, page table,
    seq_lens, order of micro-batch m's rows); q / out / k_new / v_new come from the peers.

    sync="kernel" (default): the decode kernel itself waits for qkv_ready (every CTA's producer
    polls before its first load) and publishes out_ready (the last CTA to finish, after a
    system-scope fence), so the compute stream carries nothing but back-to-back decode
    launches.  sync="stream": the same sequence numbers as stream operations around each launch.
    sync="step": one lam_decode_step per decode step (every layer and micro-batch).

    The model worker here is a zero-compute stand-in: layer l + 1's qkv_ready follows layer l's
    out_ready from every attention worker.  relay="stream": stream operations on one model stream
    per micro-batch (cuStreamWaitValue32 / cuStreamWriteValue32; ~15-20 us from the outputs'
    publication to the next layer's inputs on B200).  relay="kernel" (sync="step" only, device
    inputs): the step launch forwards it itself (lam_peer_io::n_relay, a few us).
    """

    def __init__(self, geo: ShardGeometry, dist, ctx, launch_args: Callable, device: torch.device,
                 dtype: torch.dtype, sync: str = "kernel", step_args: Callable | None = None,
                 relay: str = "stream"):
        import ctypes as C

        from . import _lib

        g = self.geo = geo
        if g.world > _lib.LAM_MAX_PEERS:
            raise ValueError(f"peer transport supports up to {_lib.LAM_MAX_PEERS} ranks")
        self.lib, self.ctx, self.device, self.dtype = _lib.load(), ctx, device, dtype
        self._C = C
        esz = torch.tensor([], dtype=dtype).element_size()
        align = lambda n: (n + 4095) // 4096 * 4096  # noqa: E731
        n_qkv = 1
        for x in g.qkv_shape():
            n_qkv *= x
        n_out = 1
        for x in g.q_shape():
            n_out *= x
        MB, N = g.micro_batches, g.world
        self.off_out = align(n_qkv * esz)
        self.off_flags = self.off_out + align(n_out * esz)
        total = self.off_flags + align(2 * MB * N * 4)
        base, handle = C.c_void_p(), (C.c_uint8 * _lib.LAM_IPC_HANDLE_BYTES)()
        _lib.check(self.lib.lam_peer_alloc(ctx.handle, total, C.byref(base), handle))
        self.base = base.value
        raw = torch.as_tensor(_DevView(self.base, total), device=device)
        self.qkv_in = raw[: n_qkv * esz].view(dtype).view(g.qkv_shape())
        self.out = raw[self.off_out: self.off_out + n_out * esz].view(dtype).view(g.q_shape())
        self.flags = raw[self.off_flags: self.off_flags + 2 * MB * N * 4].view(torch.int32).view(2, MB, N)
        # exchange handles; map every peer's buffer
        handles = [None] * N
        if dist is None:
            if N != 1:
                raise ValueError("more than one rank needs a process group to exchange handles")
            handles[0] = bytes(handle)
        else:
            dist.all_gather_object(handles, bytes(handle))
        self.peer = []
        for r in range(N):
            if r == g.rank:
                self.peer.append(self.base)
                continue
            hb = (C.c_uint8 * _lib.LAM_IPC_HANDLE_BYTES).from_buffer_copy(handles[r])
            p = C.c_void_p()
            _lib.check(self.lib.lam_peer_open(ctx.handle, hb, C.byref(p)))
            self.peer.append(p.value)
        if dist is not None:
            dist.barrier()
        self.compute = torch.cuda.current_stream(device)
        # model-worker side signalling, one stream per micro-batch: a micro-batch waiting for its
        # previous layer never holds up another micro-batch's signal
        self.models = [torch.cuda.Stream(device=device) for _ in range(geo.micro_batches)]
        self.model = self.models[0]
        self.h2d = torch.cuda.Stream(device=device)
        self.d2h = torch.cuda.Stream(device=device)
        self.epoch = 0
        # precomputed launch descriptors and flag address lists
        Ptrs = C.c_void_p * N
        qkv_elems_mb = g.Bh * g.W * g.D          # one (layer, mb, dest) block
        out_elems_mb = g.Bh * g.hq_l * g.D
        j = g.rank
        self.args, self.io = {}, {}
        for layer in range(g.layers):
            for m in range(MB):
                a = launch_args(layer, m)
                a.q_batch_stride = g.W * g.D
                a.new_batch_stride = g.W * g.D
                a.lse = None
                # consecutive launches of a step touch disjoint pools / page-table rows, so they
                # may overlap (lam_decode_peer + overlap_prev); the step's first launch follows
                # whatever the stream ran before it (e.g. a length update) in stream order
                a.overlap_prev = 0 if (layer, m) == (0, 0) else 1
                io = _lib.PeerIO()
                io.n_src, io.rows_per_src = N, g.Bh
                blk = (layer * MB + m) * N + j
                for s in range(N):
                    io.q_src[s] = self.peer[s] + blk * qkv_elems_mb * esz
                    io.out_dst[s] = self.peer[s] + self.off_out + blk * out_elems_mb * esz
                io.k_new_offset = g.hq_l * g.D
                io.v_new_offset = (g.hq_l + g.hkv_l) * g.D
                self.args[layer, m], self.io[layer, m] = a, io
        fl = lambda r, kind, m, i: self.peer[r] + self.off_flags + ((kind * MB + m) * N + i) * 4  # noqa: E731
        if sync not in ("kernel", "stream", "step"):
            raise ValueError("sync must be 'kernel', 'stream' or 'step'")
        # out_ready[m][rank] on every model worker; every worker's out_ready[m][*] is waited on
        self.sig_out = [Ptrs(*[fl(r, 1, m, j) for r in range(N)]) for m in range(MB)]
        self.wait_out = [Ptrs(*[fl(j, 1, m, s) for s in range(N)]) for m in range(MB)]
        if sync == "stream":
            # qkv_ready[m][rank] written into every attention worker (the compute stream's wait
            # polls local memory)
            self.sig_qkv = [Ptrs(*[fl(r, 0, m, j) for r in range(N)]) for m in range(MB)]
            self.wait_qkv = [Ptrs(*[fl(j, 0, m, s) for s in range(N)]) for m in range(MB)]
            self.n_sig_qkv = N
        else:
            # the model worker writes ONE local qkv_ready[m][rank] (each stream write costs a
            # system memory barrier, ~3 us on B200) and the kernels poll the sources' flags over
            # NVLink
            self.sig_qkv = [Ptrs(fl(j, 0, m, j)) for m in range(MB)]
            self.wait_qkv = [Ptrs(*[fl(s, 0, m, s) for s in range(N)]) for m in range(MB)]
            self.n_sig_qkv = 1
        self.sync = sync
        if relay not in ("stream", "kernel") or (relay == "kernel" and sync != "step"):
            raise ValueError("relay must be 'stream' or 'kernel' (the latter with sync='step')")
        self.relay = relay
        self.ahead = os.environ.get("LAM_PEER_AHEAD", "0") == "1"
        if sync == "step":
            # one persistent lam_decode_step launch per decode step: launch lm = layer * MB + m
            # of layer 0 / micro-batch 0's addressing, blocks lm * N apart in every model
            # worker's buffers, flags N apart per micro-batch
            if step_args is None:
                raise ValueError("sync='step' needs step_args")
            a, pool_layers, pool_layer_rows = step_args()
            a.q_batch_stride = g.W * g.D
            a.new_batch_stride = g.W * g.D
            a.lse = None
            a.overlap_prev = 0
            io = _lib.PeerIO()
            io.n_src, io.rows_per_src = N, g.Bh
            for s in range(N):
                io.q_src[s] = self.peer[s] + j * qkv_elems_mb * esz
                io.out_dst[s] = self.peer[s] + self.off_out + j * out_elems_mb * esz
            io.k_new_offset = g.hq_l * g.D
            io.v_new_offset = (g.hq_l + g.hkv_l) * g.D
            io.n_wait = io.n_done = N
            for i in range(N):
                io.wait_flags[i] = self.wait_qkv[0][i]
                io.done_flags[i] = self.sig_out[0][i]
            if relay == "kernel":  # this rank's qkv_ready follows its out_ready[*] in-kernel
                io.relay_flag = self.sig_qkv[0][0]
                for i in range(N):
                    io.relay_wait_flags[i] = self.wait_out[0][i]
            from .decode import step_layout

            self.step_a, self.step_io = a, io
            self.step_st = step_layout(L_ := g.layers, MB, g.B_mb, pool_layers=pool_layers,
                                       pool_layer_rows=pool_layer_rows,
                                       lm_q_stride=N * qkv_elems_mb, lm_out_stride=N * out_elems_mb,
                                       flag_mb_stride=N)
            del L_
            # LAM_STEP_TRACE (diagnostic): per-launch globaltimer stamps of the latest step
            self.trace_buf = None
            if os.environ.get("LAM_STEP_TRACE"):
                self.trace_buf = torch.empty(4 * g.layers * MB + 3 * 400 * 1024, dtype=torch.int64,
                                             device=device)
                self.step_st.trace = self.trace_buf.data_ptr()
        if sync == "kernel":
            for (layer, m), io in self.io.items():
                io.n_wait = io.n_done = N
                for i in range(N):
                    io.wait_flags[i] = self.wait_qkv[m][i]
                    io.done_flags[i] = self.sig_out[m][i]

    def close(self):
        if self.peer:
            torch.cuda.synchronize(self.device)
            for r, p in enumerate(self.peer):
                if r != self.geo.rank:
                    self.lib.lam_peer_close(self.ctx.handle, p)
            self.lib.lam_peer_free(self.ctx.handle, self.base)
            self.peer = []

    def step(self, ev=None, host_in=None, host_out=None):
        """One decode step over all layers on this rank (enqueue only).  Inputs are read from
        self.qkv_in (or copied there from pinned `host_in` first), outputs land in self.out
        (and are copied to pinned `host_out`).  `ev`: (start, end) CUDA event pairs, one per
        local launch, recorded on the compute stream."""
        from . import _lib

        g, lib, C = self.geo, self.lib, self._C
        MB, N, L = g.micro_batches, g.world, g.layers
        h = self.ctx.handle
        comp, model = self.compute, self.model
        e0 = self.epoch
        self.epoch += L
        for ms_ in self.models:
            ms_.wait_stream(comp)  # the previous step (and any input writes) are complete
        arrived = None
        if host_in is not None:
            self.h2d.wait_stream(comp)
            arrived = [torch.cuda.Event() for _ in range(L)]
            with torch.cuda.stream(self.h2d):
                for layer in range(L):
                    self.qkv_in[layer].copy_(host_in[layer], non_blocking=True)
                    arrived[layer].record(self.h2d)
        if host_out is not None:
            self.d2h.wait_stream(comp)
        cs = comp.cuda_stream
        if self.sync == "step":  # the whole step in one grid; it waits per (layer, micro-batch)
            self.step_st.epoch = e0 & 0xFFFFFFFF
            # in-kernel forwarding unless the inputs arrive from the host (their copies order
            # the model streams' signals)
            kernel_relay = self.relay == "kernel" and host_in is None
            self.step_io.n_relay = N if kernel_relay else 0
            if self.trace_buf is not None:
                with torch.cuda.stream(comp):
                    self.trace_buf.fill_(-1)
            if ev is not None:
                ev[0][0].record(comp)
            _lib.check(lib.lam_decode_step(h, self.step_a, self.step_st, self.step_io, cs))
            if ev is not None:
                ev[0][1].record(comp)
        k = 0
        for layer in range(L):
            ep = e0 + layer + 1
            for m in range(MB if layer == 0 or not (self.sync == "step" and kernel_relay) else 0):
                ms = self.models[m].cuda_stream
                if arrived is not None:
                    self.models[m].wait_event(arrived[layer])
                # model worker: layer l's rows need layer l-1's outputs of this micro-batch
                # (LAM_PEER_AHEAD=1, a diagnostic: publish every layer at once, no dependency)
                if layer > 0 and not self.ahead:
                    _lib.check(lib.lam_stream_wait(h, self.wait_out[m], N, ep - 1, ms))
                _lib.check(lib.lam_stream_signal(h, self.sig_qkv[m], self.n_sig_qkv, ep, ms))
            for m in range(MB if self.sync != "step" else 0):
                io = self.io[layer, m]
                in_kernel = self.sync == "kernel"
                if in_kernel:
                    io.wait_value = io.done_value = ep
                else:
                    _lib.check(lib.lam_stream_wait(h, self.wait_qkv[m], N, ep, cs))
                e = ev[k] if ev is not None else None
                k += 1
                if e is not None:
                    e[0].record(comp)
                _lib.check(lib.lam_decode_peer(h, self.args[layer, m], io, cs))
                if e is not None:
                    e[1].record(comp)
                if not in_kernel:
                    _lib.check(lib.lam_stream_signal(h, self.sig_out[m], N, ep, cs))
            for m in range(MB if host_out is not None else 0):
                ds = self.d2h.cuda_stream
                _lib.check(lib.lam_stream_wait(h, self.wait_out[m], N, ep, ds))
                with torch.cuda.stream(self.d2h):
                    host_out[layer, m].copy_(self.out[layer, m], non_blocking=True)
        # the step ends when this rank's outputs of the last layer have all arrived
        for m in range(MB):
            _lib.check(lib.lam_stream_wait(h, self.wait_out[m], N, e0 + L, cs))
        for ms_ in self.models:
            comp.wait_stream(ms_)
        if host_out is not None:
            comp.wait_stream(self.d2h)


class PeerRequestShardedAttention:
    """The request-level partition (RequestGeometry, attention.cpp:179-203) over the zero-copy
    peer transport: no collective and no copy kernel on the data path.

    Every rank, as model worker, exports qkv_in [L, MB, Bh, Hq + 2 Hkv, D] and out
    [L, MB, Bh, Hq, D] (both in its send order, `pack_request_inputs` /
    `unpack_request_outputs`; each (layer, micro-batch) block has one more scratch row) and a
    flag block [2][MB][N].  The owner of a request pulls its q / new K/V rows straight from the
    sender's qkv_in over NVLink, appends, attends with all heads and stores the outputs into the
    sender's out.  The launch's row map (lam_peer_io.row_src) names (source, row in the source's
    block) for each received row — any number per source.  The model worker writes its own
    qkv_ready[m] word, the kernels poll every source's word, and the last unit of a launch stores
    out_ready[m][owner] into every model worker.

    sync="step" (default): one lam_decode_step per decode step; every micro-batch has geo.R rows
    (geo.padded_rows(): pads are empty rows whose zero output goes to the owner's scratch row).
    `step_args()` returns (lam_decode_args over all MB * R rows — pools of layer 0, page table,
    seq_lens with 0 for pads, request_order local to each micro-batch —, pool_layers,
    pool_layer_rows).  sync="kernel": one lam_decode_peer per (layer, micro-batch) from
    `launch_args(layer, m)` over micro-batch m's received rows (an owner with none only
    publishes).
    """

    def __init__(self, geo: RequestGeometry, dist, ctx, launch_args: Callable | None,
                 device: torch.device, dtype: torch.dtype, sync: str = "step",
                 step_args: Callable | None = None):
        import ctypes as C

        from . import _lib

        g = self.geo = geo
        if g.world > _lib.LAM_MAX_PEERS:
            raise ValueError(f"peer transport supports up to {_lib.LAM_MAX_PEERS} ranks")
        if sync not in ("step", "kernel") or (sync == "step" and step_args is None) or \
                (sync == "kernel" and launch_args is None):
            raise ValueError("sync='step' needs step_args, sync='kernel' needs launch_args")
        self.sync = sync
        self.lib, self.ctx, self.device, self.dtype = _lib.load(), ctx, device, dtype
        self._C = C
        esz = torch.tensor([], dtype=dtype).element_size()
        align = lambda n: (n + 4095) // 4096 * 4096  # noqa: E731
        MB, N, L = g.micro_batches, g.world, g.layers
        Bb = g.Bh + 1  # rows per (layer, micro-batch) block: the requests and one scratch row
        n_qkv = L * MB * Bb * g.W * g.D
        n_out = L * MB * Bb * g.Hq * g.D
        self.off_out = align(n_qkv * esz)
        self.off_flags = self.off_out + align(n_out * esz)
        total = self.off_flags + align(2 * MB * N * 4)
        base, handle = C.c_void_p(), (C.c_uint8 * _lib.LAM_IPC_HANDLE_BYTES)()
        _lib.check(self.lib.lam_peer_alloc(ctx.handle, total, C.byref(base), handle))
        self.base = base.value
        raw = torch.as_tensor(_DevView(self.base, total), device=device)
        qkv = raw[: n_qkv * esz].view(dtype).view(L, MB, Bb, g.W, g.D)
        out = raw[self.off_out: self.off_out + n_out * esz].view(dtype).view(L, MB, Bb, g.Hq, g.D)
        self.qkv_in, self.out = qkv[:, :, : g.Bh], out[:, :, : g.Bh]  # (strided views)
        handles = [None] * N
        if dist is None:
            if N != 1:
                raise ValueError("more than one rank needs a process group to exchange handles")
            handles[0] = bytes(handle)
        else:
            dist.all_gather_object(handles, bytes(handle))
        self.peer = []
        for r in range(N):
            if r == g.rank:
                self.peer.append(self.base)
                continue
            hb = (C.c_uint8 * _lib.LAM_IPC_HANDLE_BYTES).from_buffer_copy(handles[r])
            p = C.c_void_p()
            _lib.check(self.lib.lam_peer_open(ctx.handle, hb, C.byref(p)))
            self.peer.append(p.value)
        if dist is not None:
            dist.barrier()
        self.compute = torch.cuda.current_stream(device)
        self.models = [torch.cuda.Stream(device=device) for _ in range(MB)]
        self.epoch = 0
        Ptrs = C.c_void_p * N
        fl = lambda r, kind, m, i: self.peer[r] + self.off_flags + ((kind * MB + m) * N + i) * 4  # noqa: E731
        j = g.rank
        self.sig_qkv = [Ptrs(fl(j, 0, m, j)) for m in range(MB)]          # own word
        self.wait_qkv = [[fl(s, 0, m, s) for s in range(N)] for m in range(MB)]  # polled remotely
        self.sig_out = [Ptrs(*[fl(r, 1, m, j) for r in range(N)]) for m in range(MB)]
        self.wait_out = [Ptrs(*[fl(j, 1, m, s) for s in range(N)]) for m in range(MB)]
        blk_qkv, blk_out = Bb * g.W * g.D, Bb * g.Hq * g.D  # elements per (layer, mb) block

        def src_row(r):  # global request -> (source, row in the source's block)
            s, b = divmod(r, g.B_local)
            m = b // g.Bh
            return (s << 24) | g.send_order_of(s, m).index(b)

        def io_for(layer, m, rows_map):
            io = _lib.PeerIO()
            io.n_src, io.rows_per_src = N, 1
            for s in range(N):
                io.q_src[s] = self.peer[s] + (layer * MB + m) * blk_qkv * esz
                io.out_dst[s] = self.peer[s] + self.off_out + (layer * MB + m) * blk_out * esz
            io.k_new_offset = g.Hq * g.D
            io.v_new_offset = (g.Hq + g.Hkv) * g.D
            io.n_wait = io.n_done = N
            for s in range(N):
                io.wait_flags[s] = self.wait_qkv[m][s]
                io.done_flags[s] = self.sig_out[m][s]
            io.row_src = rows_map.data_ptr()
            return io

        self.args, self.io = {}, {}
        if sync == "step":
            scratch = (j << 24) | g.Bh
            rmap = [src_row(r) if r >= 0 else scratch for r in g.padded_rows()]
            self.row_map = torch.tensor(rmap, dtype=torch.int32, device=device)
            a, pool_layers, pool_layer_rows = step_args()
            a.q_batch_stride = a.new_batch_stride = g.W * g.D
            a.lse = None
            a.overlap_prev = 0
            self.step_a, self.step_io = a, io_for(0, 0, self.row_map)
            from .decode import step_layout

            self.step_st = step_layout(L, MB, g.R, pool_layers=pool_layers,
                                       pool_layer_rows=pool_layer_rows, lm_q_stride=blk_qkv,
                                       lm_out_stride=blk_out, flag_mb_stride=N)
        else:
            self.row_maps = [torch.tensor([src_row(r) for r in g.recv_reqs[m]] or [0],
                                          dtype=torch.int32, device=device) for m in range(MB)]
            for layer in range(L):
                for m in range(MB):
                    if not g.recv_reqs[m]:
                        continue
                    a = launch_args(layer, m)
                    a.q_batch_stride = a.new_batch_stride = g.W * g.D
                    a.lse = None
                    a.overlap_prev = 0
                    self.args[layer, m], self.io[layer, m] = a, io_for(layer, m, self.row_maps[m])

    def close(self):
        if self.peer:
            torch.cuda.synchronize(self.device)
            for r, p in enumerate(self.peer):
                if r != self.geo.rank:
                    self.lib.lam_peer_close(self.ctx.handle, p)
            self.lib.lam_peer_free(self.ctx.handle, self.base)
            self.peer = []

    def step(self):
        """One decode step over all layers (enqueue only): inputs from self.qkv_in, outputs in
        self.out of every model worker."""
        from . import _lib

        g, lib = self.geo, self.lib
        MB, N, L = g.micro_batches, g.world, g.layers
        h = self.ctx.handle
        comp = self.compute
        e0 = self.epoch
        self.epoch += L
        for ms in self.models:
            ms.wait_stream(comp)
        cs = comp.cuda_stream
        if self.sync == "step":
            self.step_st.epoch = e0 & 0xFFFFFFFF
            _lib.check(lib.lam_decode_step(h, self.step_a, self.step_st, self.step_io, cs))
        for layer in range(L):
            ep = e0 + layer + 1
            for m in range(MB):  # model worker: layer l + 1 follows layer l's outputs
                ms = self.models[m].cuda_stream
                if layer > 0:
                    _lib.check(lib.lam_stream_wait(h, self.wait_out[m], N, ep - 1, ms))
                _lib.check(lib.lam_stream_signal(h, self.sig_qkv[m], 1, ep, ms))
            for m in range(MB if self.sync == "kernel" else 0):  # attention worker
                if (layer, m) in self.io:
                    io = self.io[layer, m]
                    io.wait_value = io.done_value = ep
                    _lib.check(lib.lam_decode_peer(h, self.args[layer, m], io, cs))
                else:  # nothing received: publish the (empty) outputs at once
                    _lib.check(lib.lam_stream_signal(h, self.sig_out[m], N, ep, cs))
        for m in range(MB):
            _lib.check(lib.lam_stream_wait(h, self.wait_out[m], N, e0 + L, cs))
        for ms in self.models:
            comp.wait_stream(ms)
