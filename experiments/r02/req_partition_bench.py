"""C5 (LLaMA-2-70B, B = 256, lengths log-uniform 128..16384, seed 2024, 80 layers) over the
request-level partition on the peer transport (dist.PeerRequestShardedAttention): every rank
owns ALL KV heads of the requests request_partition (attention.cpp:179-203) gives it.  Strong
scaling (the same 256 requests at every N); prints one JSON line from rank 0 with the whole
job's attn_cost GB/s (device-timed, max over ranks), to set beside bench.py --workload c5
(head partition).  Run under torchrun (127.0.0.1)."""
import json
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_2405_01814_b200 import _lib, decode as dec  # noqa: E402
from paper_2405_01814_b200.attention import request_partition  # noqa: E402
from paper_2405_01814_b200.dist import PeerRequestShardedAttention, RequestGeometry  # noqa: E402
from paper_2405_01814_b200.kvcache import PagedKVCache  # noqa: E402

L, B, HQ, HKV, D, P, MB = 80, 256, 64, 8, 128, 64, 2
STEPS, WARMUP = int(os.environ.get("STEPS", 5)), int(os.environ.get("WARMUP", 3))


def main():
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    r = np.random.default_rng(2024)
    lens = np.exp(r.uniform(math.log(128), math.log(16384), B)).astype(np.int32)  # bench c5 law
    owner = request_partition(lens.astype(np.float64), world).device_of
    B_local = B // world
    geo = RequestGeometry(rank, world, L, B_local, HQ, HKV, D, owner, MB)
    sync = os.environ.get("SYNC", "step")
    rows = np.array(geo.padded_rows() if sync == "step" else geo.rows, np.int64)
    row_lens = np.where(rows >= 0, lens[np.maximum(rows, 0)], 0).astype(np.int32)
    pages = int((-(-row_lens // P)).sum()) + 2
    cache = PagedKVCache(L, HKV, D, P, pages, max(len(rows), 1), int(-(-row_lens.max() // P)),
                         dtype=torch.bfloat16, device=dev, shuffle_seed=rank)
    cache.set_lengths(row_lens)
    cache.sync()
    cache.fill_random(torch.Generator(device=dev).manual_seed(rank))
    max_len = int(row_lens.max())
    orders = []
    for m in range(MB):  # longest request first within each launch (LPT), as bench.py does
        n = geo.R if sync == "step" else len(geo.recv_reqs[m])
        off = m * geo.R if sync == "step" else geo.row_off[m]
        sl = row_lens[off: off + n]
        orders.append(torch.tensor(np.argsort(-sl, kind="stable").astype(np.int32), device=dev))
    order_all = torch.cat(orders).contiguous()

    def step_args():
        qd = torch.empty((len(rows), HQ, D), dtype=torch.bfloat16, device=dev)
        a, _ = dec.make_args(qd, cache.k[0], cache.v[0], cache.seq_lens, page_table=cache.page_table,
                             max_len=max_len, out=qd, request_order=order_all)
        return a, L, cache.k[0].numel() // D

    def launch_args(layer, m):
        n = len(geo.recv_reqs[m])
        sl = slice(geo.row_off[m], geo.row_off[m] + n)
        qd = torch.empty((n, HQ, D), dtype=torch.bfloat16, device=dev)
        a, _ = dec.make_args(qd, cache.k[layer], cache.v[layer], cache.seq_lens[sl],
                             page_table=cache.page_table[sl], max_len=max_len, out=qd,
                             request_order=orders[m])
        return a

    ctx = _lib.context(dev.index)
    eng = PeerRequestShardedAttention(geo, dist, ctx, launch_args, dev, torch.bfloat16, sync=sync,
                                      step_args=step_args)
    eng.qkv_in.uniform_(-1, 1)
    torch.cuda.synchronize()
    for _ in range(WARMUP):
        eng.step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(STEPS):
        eng.step()
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / STEPS], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    mine = float(row_lens.sum()) * 2 * HKV * D * 2 * L  # this rank's KV bytes per step
    loads = [None] * world
    dist.all_gather_object(loads, mine)
    status = ctx.status()
    eng.close()
    if rank == 0:
        total = float(lens.sum()) * 2 * HKV * D * 2 * L
        print(json.dumps({
            "workload": "c5 (B=256 log-uniform 128..16384, seed 2024, 80 layers), request partition, peer transport",
            "sync": sync, "rows_per_microbatch": geo.R,
            "n_gpus": world, "ms_per_step": float(ms), "value_gbs": total / (float(ms) / 1e3) / 1e9,
            "per_gpu_gbs": total / (float(ms) / 1e3) / 1e9 / world,
            "kv_bytes_per_rank_share": [x / total for x in loads], "device_status": status}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
