"""torchrun worker for tests/test_dist_gpu.py: the KV-head-sharded engine with the real kernels
(lam_kv_append + lam_decode over a paged store) over NCCL, checked against the CPU oracle."""
import math
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2405_01814_b200 import decode as dec  # noqa: E402
from paper_2405_01814_b200 import _lib  # noqa: E402
from paper_2405_01814_b200.dist import (HeadShardedAttention, PeerShardedAttention,  # noqa: E402
                                        ShardGeometry, shard_inputs, stitch_outputs)
from paper_2405_01814_b200.kvcache import PagedKVCache  # noqa: E402

L, B_LOCAL, HQ, HKV, D, MB, P = 3, 8, 64, 8, 128, 2, 64


def main_request():
    """Request-partitioned pool (dist.RequestShardedAttention): every rank holds all KV heads of
    the requests request_partition gives it; Hkv = 3 is not divisible by the world size."""
    from paper_2405_01814_b200.attention import request_partition
    from paper_2405_01814_b200.dist import (RequestGeometry, RequestShardedAttention,
                                            pack_request_inputs, unpack_request_outputs)

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    hq, hkv = 24, 3
    rng = np.random.default_rng(13)
    B = world * B_LOCAL
    lens = np.exp(rng.uniform(np.log(8), np.log(2000), B)).astype(np.int32)  # mixed lengths
    owner = request_partition((lens + 1).astype(np.float64), world).device_of
    geo = RequestGeometry(rank, world, L, B_LOCAL, hq, hkv, D, owner, MB)
    lmax = int(lens.max()) + 1
    bf = lambda x: torch.from_numpy(x).to(torch.bfloat16)  # noqa: E731
    ck = bf(rng.uniform(-1, 1, (L, B, hkv, lmax, D)).astype(np.float32))
    cv = bf(rng.uniform(-1, 1, (L, B, hkv, lmax, D)).astype(np.float32))
    q = bf(rng.uniform(-1, 1, (L, B, hq, D)).astype(np.float32))
    kn = bf(rng.uniform(-1, 1, (L, B, hkv, D)).astype(np.float32))
    vn = bf(rng.uniform(-1, 1, (L, B, hkv, D)).astype(np.float32))
    peer = os.environ.get("LAM_TEST_TRANSPORT", "nccl") == "peer"
    req_sync = os.environ.get("LAM_TEST_SYNC", "step") if peer else "-"
    # the step launch's rows are micro-batch-major with R rows each (-1: an empty pad row)
    rows = np.array(geo.padded_rows() if req_sync == "step" else geo.rows, np.int64)
    row_lens = np.where(rows >= 0, lens[np.maximum(rows, 0)] + 1, 0)
    n_rows = max(len(rows), 1)
    cache = PagedKVCache(L, hkv, D, P, int((-(-row_lens // P)).sum()) + 2, n_rows,
                         int(-(-row_lens.max() // P)) if len(rows) else 1, dtype=torch.bfloat16,
                         device=dev, shuffle_seed=rank)
    if len(rows):
        cache.set_lengths(row_lens)
    cache.sync()
    pt = cache.page_table_host
    for layer in range(L):
        for r, req in enumerate(rows):
            if req < 0:
                continue
            n = int(lens[req])
            for p0 in range(0, n, P):
                t1 = min(n, p0 + P)
                cache.k[layer, pt[r, p0 // P], :, : t1 - p0] = ck[layer, req, :, p0:t1].to(dev)
                cache.v[layer, pt[r, p0 // P], :, : t1 - p0] = cv[layer, req, :, p0:t1].to(dev)
    max_len = int(row_lens.max()) if len(rows) else 1

    def attend_fused(layer, m, qr, k, v, out):
        sl = slice(geo.row_off[m], geo.row_off[m] + qr.shape[0])
        dec.decode(qr, cache.k[layer], cache.v[layer], cache.seq_lens[sl],
                   page_table=cache.page_table[sl], max_len=max_len, out=out, k_new=k, v_new=v)

    mine = slice(rank * B_LOCAL, (rank + 1) * B_LOCAL)
    qkv_in = pack_request_inputs(geo, q[:, mine], kn[:, mine], vn[:, mine]).to(dev)
    if peer:
        # zero-copy: owners pull whole requests from the senders and store outputs back
        from paper_2405_01814_b200.dist import PeerRequestShardedAttention

        def launch_args(layer, m):
            n = len(geo.recv_reqs[m])
            sl = slice(geo.row_off[m], geo.row_off[m] + n)
            qd = torch.empty((n, hq, D), dtype=torch.bfloat16, device=dev)
            a, _ = dec.make_args(qd, cache.k[layer], cache.v[layer], cache.seq_lens[sl],
                                 page_table=cache.page_table[sl], max_len=max_len, out=qd)
            return a

        def step_args():
            qd = torch.empty((len(rows), hq, D), dtype=torch.bfloat16, device=dev)
            a, _ = dec.make_args(qd, cache.k[0], cache.v[0], cache.seq_lens,
                                 page_table=cache.page_table, max_len=max_len, out=qd)
            return a, L, cache.k[0].numel() // D

        eng = PeerRequestShardedAttention(geo, dist, _lib.context(dev.index), launch_args, dev,
                                          torch.bfloat16, sync=req_sync, step_args=step_args)
        eng.qkv_in.copy_(qkv_in)
        eng.out.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        eng.step()
        torch.cuda.synchronize()
        out = eng.out.clone()
        dist.barrier()
        eng.close()
    else:
        eng = RequestShardedAttention(geo, dist, None, attend_fused, dev, torch.bfloat16)
        out = torch.zeros(geo.q_shape(), dtype=torch.bfloat16, device=dev)
        eng.step(qkv_in, out)
        torch.cuda.synchronize()
    got = unpack_request_outputs(geo, out).float().cpu().numpy()
    worst = 0.0
    for layer in range(L):
        for b in range(B_LOCAL):
            req = rank * B_LOCAL + b
            k = ck[layer, req:req + 1].float().numpy().copy()
            v = cv[layer, req:req + 1].float().numpy().copy()
            k[0, :, lens[req]] = kn[layer, req].float().numpy()
            v[0, :, lens[req]] = vn[layer, req].float().numpy()
            want = O.decode_dense(q[layer, req:req + 1].float().numpy(), k, v, [lens[req] + 1],
                                  1 / math.sqrt(D))[0]
            worst = max(worst, float(np.abs(got[layer, b] - want).max()))
    ok = worst <= 2e-3 + 2 ** -9
    print(f"rank {rank} request-sharded worst max-abs {worst:.3e} {'OK' if ok else 'FAIL'}",
          flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


def main():
    if os.environ.get("LAM_TEST_SHARD", "head") == "request":
        return main_request()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    geo = ShardGeometry(rank, world, L, B_LOCAL, HQ, HKV, D, MB)
    rng = np.random.default_rng(11)
    B = world * B_LOCAL
    lens = rng.integers(1, 300, B).astype(np.int32)           # tokens cached before the step
    lmax = int(lens.max()) + 1
    bf = lambda x: torch.from_numpy(x).to(torch.bfloat16)  # noqa: E731
    ck = bf(rng.uniform(-1, 1, (L, B, HKV, lmax, D)).astype(np.float32))
    cv = bf(rng.uniform(-1, 1, (L, B, HKV, lmax, D)).astype(np.float32))
    q = bf(rng.uniform(-1, 1, (L, B, HQ, D)).astype(np.float32))
    kn = bf(rng.uniform(-1, 1, (L, B, HKV, D)).astype(np.float32))
    vn = bf(rng.uniform(-1, 1, (L, B, HKV, D)).astype(np.float32))

    h0, h1 = rank * geo.hkv_l, (rank + 1) * geo.hkv_l
    row_req = np.zeros(geo.B_attn, np.int64)
    for src in range(world):
        for b in range(B_LOCAL):
            row_req[geo.kv_row(src, b)] = src * B_LOCAL + b
    row_lens = lens[row_req] + 1
    cache = PagedKVCache(L, geo.hkv_l, D, P, int((-(-row_lens // P)).sum()) + 2, geo.B_attn,
                         int(-(-row_lens.max() // P)), dtype=torch.bfloat16, device=dev,
                         shuffle_seed=rank)
    cache.set_lengths(row_lens)
    cache.sync()
    pt = cache.page_table_host
    for layer in range(L):  # prefill the cached prefix (test infrastructure: torch indexing)
        for r, req in enumerate(row_req):
            for t in range(lens[req]):
                page, off = pt[r, t // P], t % P
                cache.k[layer, page, :, off] = ck[layer, req, h0:h1, t].to(dev)
                cache.v[layer, page, :, off] = cv[layer, req, h0:h1, t].to(dev)
    positions = torch.tensor(row_lens - 1, dtype=torch.int32, device=dev)

    fused = os.environ.get("LAM_TEST_FUSED", "1") == "1"

    def append(layer, m, k, v):
        sl = slice(m * geo.B_mb, (m + 1) * geo.B_mb)
        dec.kv_append(k, v, cache.k[layer], cache.v[layer], positions[sl], cache.page_table[sl])

    def attend(layer, m, qr, out):
        sl = slice(m * geo.B_mb, (m + 1) * geo.B_mb)
        dec.decode(qr, cache.k[layer], cache.v[layer], cache.seq_lens[sl],
                   page_table=cache.page_table[sl], max_len=int(row_lens.max()), out=out)

    def attend_fused(layer, m, qr, k, v, out):
        sl = slice(m * geo.B_mb, (m + 1) * geo.B_mb)
        dec.decode(qr, cache.k[layer], cache.v[layer], cache.seq_lens[sl],
                   page_table=cache.page_table[sl], max_len=int(row_lens.max()), out=out,
                   k_new=k, v_new=v)

    mine = slice(rank * B_LOCAL, (rank + 1) * B_LOCAL)
    qkv_in = shard_inputs(q[:, mine], kn[:, mine], vn[:, mine], world, MB).to(dev)
    if os.environ.get("LAM_TEST_TRANSPORT", "nccl") == "peer":
        # peer-memory transport: zero-copy pull of q/k/v, outputs stored into the model worker
        ctx = _lib.context(dev.index)

        def launch_args(layer, m):
            sl = slice(m * geo.B_mb, (m + 1) * geo.B_mb)
            qd = torch.empty((geo.B_mb, geo.hq_l, D), dtype=torch.bfloat16, device=dev)
            a, _ = dec.make_args(qd, cache.k[layer], cache.v[layer], cache.seq_lens[sl],
                                 page_table=cache.page_table[sl], max_len=int(row_lens.max()),
                                 out=qd)
            return a

        def step_args():  # sync="step": every row of every micro-batch, pool layer 0
            qd = torch.empty((geo.B_attn, geo.hq_l, D), dtype=torch.bfloat16, device=dev)
            a, _ = dec.make_args(qd, cache.k[0], cache.v[0], cache.seq_lens,
                                 page_table=cache.page_table, max_len=int(row_lens.max()), out=qd)
            return a, L, cache.k[0].numel() // D

        sync = os.environ.get("LAM_TEST_SYNC", "kernel")
        relay = "kernel" if sync == "step-relay" else "stream"
        sync = "step" if sync == "step-relay" else sync
        eng = PeerShardedAttention(geo, dist, ctx, launch_args, dev, torch.bfloat16,
                                   sync=sync, step_args=step_args, relay=relay)
        eng.qkv_in.copy_(qkv_in)
        eng.out.zero_()
        host_io = os.environ.get("LAM_TEST_HOST", "0") == "1"
        if host_io:  # from pinned host buffers, as the end-to-end bench runs it
            h_in = qkv_in.cpu().pin_memory()
            h_out = torch.zeros(geo.q_shape(), dtype=torch.bfloat16).pin_memory()
            eng.qkv_in.zero_()
            torch.cuda.synchronize()
            eng.step(host_in=h_in, host_out=h_out)
        else:
            eng.step()
        torch.cuda.synchronize()
        out = h_out if host_io else eng.out.clone()
        dist.barrier()
        eng.close()
    else:
        eng = (HeadShardedAttention(geo, dist, None, attend_fused, dev, torch.bfloat16) if fused
               else HeadShardedAttention(geo, dist, append, attend, dev, torch.bfloat16))
        out = torch.zeros(geo.q_shape(), dtype=torch.bfloat16, device=dev)
        eng.step(qkv_in, out)
        torch.cuda.synchronize()
    got = stitch_outputs(out).float().cpu().numpy()
    worst = 0.0
    for layer in range(L):
        for b in range(B_LOCAL):
            req = rank * B_LOCAL + b
            k = ck[layer, req:req + 1].float().numpy().copy()
            v = cv[layer, req:req + 1].float().numpy().copy()
            k[0, :, lens[req]] = kn[layer, req].float().numpy()
            v[0, :, lens[req]] = vn[layer, req].float().numpy()
            want = O.decode_dense(q[layer, req:req + 1].float().numpy(), k, v, [lens[req] + 1],
                                  1 / math.sqrt(D))[0]
            worst = max(worst, float(np.abs(got[layer, b] - want).max()))
    # bf16 output: kernel tolerance 2e-3 plus the final bf16 rounding of |out| <= 1
    ok = worst <= 2e-3 + 2 ** -9
    print(f"rank {rank} worst max-abs {worst:.3e} {'OK' if ok else 'FAIL'}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
