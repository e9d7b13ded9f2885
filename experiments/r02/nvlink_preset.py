"""Measure the NVLink peer transport as a reference NetPreset (net.hpp: one-way base latency +
achievable bandwidth): 2 ranks, torchrun.  Latency: ping-pong of 32-bit sequence numbers between
the two GPUs' streams (lam_stream_signal to the peer's flag, lam_stream_wait on the own flag) —
the signalling the attention-worker engine uses per layer.  Bandwidth: a 1 GiB copy into the
peer's buffer (IPC-mapped, NVLink)."""
import ctypes as C
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2405_01814_b200 import _lib  # noqa: E402
from paper_2405_01814_b200.dist import _DevView  # noqa: E402

rank = int(os.environ["RANK"])
dev = torch.device("cuda", rank)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
lib, ctx = _lib.load(), _lib.context(rank)
nbytes = 1 << 30
base, handle = C.c_void_p(), (C.c_uint8 * _lib.LAM_IPC_HANDLE_BYTES)()
_lib.check(lib.lam_peer_alloc(ctx.handle, nbytes + 4096, C.byref(base), handle))
hs = [None, None]
dist.all_gather_object(hs, bytes(handle))
peer = C.c_void_p()
_lib.check(lib.lam_peer_open(ctx.handle, (C.c_uint8 * _lib.LAM_IPC_HANDLE_BYTES).from_buffer_copy(hs[1 - rank]),
                             C.byref(peer)))
mine = torch.as_tensor(_DevView(base.value, nbytes + 4096), device=dev)
theirs = torch.as_tensor(_DevView(peer.value, nbytes + 4096), device=dev)
flag_mine = (C.c_void_p * 1)(base.value + nbytes)
flag_peer = (C.c_void_p * 1)(peer.value + nbytes)
s = torch.cuda.Stream()
dist.barrier()
torch.cuda.synchronize()
n = 2000
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for i in range(1, n + 1):
    if rank == 0:
        _lib.check(lib.lam_stream_signal(ctx.handle, flag_peer, 1, i, s.cuda_stream))
        _lib.check(lib.lam_stream_wait(ctx.handle, flag_mine, 1, i, s.cuda_stream))
    else:
        _lib.check(lib.lam_stream_wait(ctx.handle, flag_mine, 1, i, s.cuda_stream))
        _lib.check(lib.lam_stream_signal(ctx.handle, flag_peer, 1, i, s.cuda_stream))
e1.record(s)
torch.cuda.synchronize()
one_way = e0.elapsed_time(e1) * 1e-3 / (2 * n)
dist.barrier()
src = torch.empty(nbytes, dtype=torch.uint8, device=dev).fill_(rank)
bw = []
for rep in range(6):
    torch.cuda.synchronize()
    dist.barrier()
    e0.record(s)
    with torch.cuda.stream(s):
        theirs[:nbytes].copy_(src, non_blocking=True)
    e1.record(s)
    torch.cuda.synchronize()
    if rep:
        bw.append(nbytes / (e0.elapsed_time(e1) * 1e-3))
dist.barrier()
if rank == 0:
    print(json.dumps({"name": "NVLINK-PEER", "base_latency_s": one_way,
                      "achievable_bw": sorted(bw)[len(bw) // 2],
                      "how": "one-way = half the round trip of a stream-ordered sequence-number "
                             "ping-pong between two B200s (lam_stream_signal / lam_stream_wait, "
                             f"{n} round trips); bandwidth = median of 5 x 1 GiB copies into the "
                             "peer's IPC-mapped buffer (both directions at once)"}), flush=True)
lib.lam_peer_close(ctx.handle, peer)
dist.destroy_process_group()
