"""One lam_decode_peer launch whose source rows live on ANOTHER GPU (single process, two
devices, peer access): a C3-at-N=2-shaped attention shard on cuda:0 (64 rows, 32 q / 4 KV
heads, l = 4096, paged bf16) pulls the packed q / new K/V rows from cuda:1 over NVLink and
stores its outputs there.  Checks the outputs and the appended rows against the same launch
with the rows local (bitwise), and prints the bytes the transport must move per launch
(perf.cpp:142-148, comm_volume) for the ncu NVLink counters to be set against.
Run: python experiments/r02/peer_nvlink.py   (2 visible GPUs; ncu with --devices 0)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_2405_01814_b200 import _lib, decode as dec  # noqa: E402
from paper_2405_01814_b200.kvcache import PagedKVCache  # noqa: E402

B, HQ, HKV, D, L, P = 64, 32, 4, 128, 4096, 64
W = HQ + 2 * HKV


def main():
    d0, d1 = torch.device("cuda:0"), torch.device("cuda:1")
    torch.cuda.set_device(d0)
    torch.empty(1, device=d0).copy_(torch.empty(1, device=d1))  # torch enables peer access
    torch.cuda.set_device(d1)
    torch.empty(1, device=d1).copy_(torch.empty(1, device=d0))
    torch.cuda.set_device(d0)
    g = torch.Generator(device=d0).manual_seed(0)
    cache = PagedKVCache(1, HKV, D, P, B * L // P + 1, B, L // P, dtype=torch.bfloat16, device=d0,
                         shuffle_seed=3)
    cache.set_lengths([L] * B)
    cache.sync()
    cache.fill_random(g)
    k0, v0 = cache.k[0].clone(), cache.v[0].clone()
    qkv_local = torch.empty((B, W, D), dtype=torch.bfloat16, device=d0).uniform_(-1, 1, generator=g)
    qkv_remote = qkv_local.to(d1)
    out_remote = torch.zeros((B, HQ, D), dtype=torch.bfloat16, device=d1)
    out_local = torch.zeros((B, HQ, D), dtype=torch.bfloat16, device=d0)
    qd = torch.empty((B, HQ, D), dtype=torch.bfloat16, device=d0)
    a, _ = dec.make_args(qd, cache.k[0], cache.v[0], cache.seq_lens, page_table=cache.page_table,
                         max_len=L, out=qd)
    a.q_batch_stride = a.new_batch_stride = W * D
    lib, ctx = _lib.load(), _lib.context(0)
    s = torch.cuda.current_stream(d0).cuda_stream

    def launch(src, dst):
        io = _lib.PeerIO()
        io.n_src, io.rows_per_src = 1, B
        io.q_src[0], io.out_dst[0] = src.data_ptr(), dst.data_ptr()
        io.k_new_offset, io.v_new_offset = HQ * D, (HQ + HKV) * D
        _lib.check(lib.lam_decode_peer(ctx.handle, a, io, s))

    # remote rows (the launch ncu profiles first: --launch-count 1 with the kernel filter)
    launch(qkv_remote, out_remote)
    torch.cuda.synchronize(d0)
    torch.cuda.synchronize(d1)
    k_remote, v_remote = cache.k[0].clone(), cache.v[0].clone()
    cache.k[0].copy_(k0)
    cache.v[0].copy_(v0)
    launch(qkv_local, out_local)
    torch.cuda.synchronize(d0)
    same_out = torch.equal(out_remote.to(d0), out_local)
    same_kv = torch.equal(k_remote, cache.k[0]) and torch.equal(v_remote, cache.v[0])
    esz = 2
    print(json.dumps({
        "launch": f"lam_decode_peer B={B} Hq={HQ} Hkv={HKV} l={L} bf16, rows on cuda:1, KV on cuda:0",
        "outputs_bitwise_equal_local": same_out, "append_bitwise_equal_local": same_kv,
        "pulled_bytes": B * W * D * esz, "stored_bytes": B * HQ * D * esz,
        "comm_volume_bytes": B * (2 * HQ + 2 * HKV) * D * esz,
        "kv_bytes_local_hbm": B * L * 2 * HKV * D * esz}))
    sys.exit(0 if same_out and same_kv else 1)


if __name__ == "__main__":
    main()
