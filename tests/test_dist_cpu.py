"""The multi-GPU exchange logic (paper_2405_01814_b200/dist.py) on CPU: world_size 2 over gloo.

Each rank is a model worker for B_local requests and the attention worker for half the KV
heads.  The local append/attend ops are the CPU oracle (injected), so this test checks the
sharding, the all-to-all layouts, the micro-batch row mapping and the output stitching; the
GPU kernels are covered by the -m gpu tests.  Result: every request's attention output equals
the single-process oracle over all heads, and appended tokens land where decode reads them.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parent.parent

L, B_LOCAL, HQ, HKV, D, WORLD, MB = 2, 4, 8, 4, 8, 2, 2


def _global_problem(seed=7):
    rng = np.random.default_rng(seed)
    B = WORLD * B_LOCAL
    lens = rng.integers(1, 20, B).astype(np.int32)       # cached tokens before this step
    lmax = int(lens.max()) + 1
    cache_k = rng.uniform(-1, 1, (L, B, HKV, lmax, D)).astype(np.float32)
    cache_v = rng.uniform(-1, 1, (L, B, HKV, lmax, D)).astype(np.float32)
    q = rng.uniform(-1, 1, (L, B, HQ, D)).astype(np.float32)
    kn = rng.uniform(-1, 1, (L, B, HKV, D)).astype(np.float32)
    vn = rng.uniform(-1, 1, (L, B, HKV, D)).astype(np.float32)
    return lens, lmax, cache_k, cache_v, q, kn, vn


def _expected(layer, req):
    from oracle import oracle as O

    lens, lmax, ck, cv, q, kn, vn = _global_problem()
    k = ck[layer, req:req + 1].copy()
    v = cv[layer, req:req + 1].copy()
    k[0, :, lens[req]] = kn[layer, req]
    v[0, :, lens[req]] = vn[layer, req]
    return O.decode_dense(q[layer, req:req + 1], k, v, [lens[req] + 1], 1 / np.sqrt(D))[0]


def _worker(rank, port, result_dir):
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2405_01814_b200.dist import (HeadShardedAttention, ShardGeometry, shard_inputs,
                                            stitch_outputs)

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    geo = ShardGeometry(rank, WORLD, L, B_LOCAL, HQ, HKV, D, MB)
    lens, lmax, ck, cv, q, kn, vn = _global_problem()
    h0, h1 = rank * geo.hkv_l, (rank + 1) * geo.hkv_l
    # attention-side store: rows in micro-batch-major order, this rank's KV heads only
    row_req = np.zeros(geo.B_attn, np.int64)
    for src in range(WORLD):
        for b in range(B_LOCAL):
            row_req[geo.kv_row(src, b)] = src * B_LOCAL + b
    store_k = ck[:, row_req, h0:h1].copy()
    store_v = cv[:, row_req, h0:h1].copy()
    pos = lens[row_req]                     # new token position of each row

    def append(layer, m, k, v):
        rows = range(m * geo.B_mb, (m + 1) * geo.B_mb)
        for i, r in enumerate(rows):
            store_k[layer, r, :, pos[r]] = k[i].contiguous().numpy()
            store_v[layer, r, :, pos[r]] = v[i].contiguous().numpy()

    def attend(layer, m, qr, out):
        sl = slice(m * geo.B_mb, (m + 1) * geo.B_mb)
        res = O.decode_dense(qr.contiguous().numpy(), store_k[layer, sl], store_v[layer, sl], pos[sl] + 1,
                             1 / np.sqrt(D))
        out.copy_(torch.from_numpy(res))

    eng = HeadShardedAttention(geo, dist, append, attend, torch.device("cpu"), torch.float32)
    mine = slice(rank * B_LOCAL, (rank + 1) * B_LOCAL)
    qkv_in = shard_inputs(torch.from_numpy(q[:, mine]), torch.from_numpy(kn[:, mine]),
                          torch.from_numpy(vn[:, mine]), WORLD, MB)
    out = torch.zeros(geo.q_shape())
    eng.step(qkv_in, out)
    np.save(Path(result_dir) / f"out{rank}.npy", stitch_outputs(out).numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_head_sharded_exchange_matches_oracle(tmp_path):
    import torch.multiprocessing as mp

    os.environ["PYTHONPATH"] = str(ROOT) + os.pathsep + os.environ.get("PYTHONPATH", "")
    mp.spawn(_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    for rank in range(WORLD):
        got = np.load(tmp_path / f"out{rank}.npy")          # [L, B_local, Hq, D]
        for layer in range(L):
            for b in range(B_LOCAL):
                want = _expected(layer, rank * B_LOCAL + b)
                assert np.allclose(got[layer, b], want, rtol=0, atol=1e-6)


def test_geometry_validation():
    from paper_2405_01814_b200.dist import ShardGeometry

    with pytest.raises(ValueError, match="divisible"):
        ShardGeometry(0, 3, 1, 4, 8, 8, 128)
    g = ShardGeometry(1, 4, 80, 128, 64, 8, 128)
    assert (g.hq_l, g.hkv_l, g.Bh, g.B_mb, g.B_attn) == (16, 2, 64, 256, 512)
    rows = sorted(g.kv_row(s, b) for s in range(4) for b in range(128))
    assert rows == list(range(512))


# ---- request-level partition (dist.RequestShardedAttention), KV heads not divisible by N ----
RQ_HQ, RQ_HKV = 6, 3  # head_partition would reject 3 KV heads over 2 ranks


def _req_problem(seed=11):
    rng = np.random.default_rng(seed)
    B = WORLD * B_LOCAL
    lens = rng.integers(1, 40, B).astype(np.int32)
    lmax = int(lens.max()) + 1
    ck = rng.uniform(-1, 1, (L, B, RQ_HKV, lmax, D)).astype(np.float32)
    cv = rng.uniform(-1, 1, (L, B, RQ_HKV, lmax, D)).astype(np.float32)
    q = rng.uniform(-1, 1, (L, B, RQ_HQ, D)).astype(np.float32)
    kn = rng.uniform(-1, 1, (L, B, RQ_HKV, D)).astype(np.float32)
    vn = rng.uniform(-1, 1, (L, B, RQ_HKV, D)).astype(np.float32)
    return lens, ck, cv, q, kn, vn


def _req_owner(lens):
    from paper_2405_01814_b200.attention import request_partition

    return request_partition((lens + 1).astype(np.float64), WORLD).device_of


def _req_worker(rank, port, result_dir):
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2405_01814_b200.dist import (RequestGeometry, RequestShardedAttention,
                                            pack_request_inputs, unpack_request_outputs)

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    lens, ck, cv, q, kn, vn = _req_problem()
    geo = RequestGeometry(rank, WORLD, L, B_LOCAL, RQ_HQ, RQ_HKV, D, _req_owner(lens), MB)
    rows = np.array(geo.rows, np.int64)
    store_k, store_v = ck[:, rows].copy(), cv[:, rows].copy()  # all heads of owned requests
    pos = lens[rows]

    def attend(layer, m, qr, k, v, out):  # fused: append the new token, then attend
        sl = slice(geo.row_off[m], geo.row_off[m] + qr.shape[0])
        for i, r in enumerate(range(sl.start, sl.stop)):
            store_k[layer, r, :, pos[r]] = k[i].contiguous().numpy()
            store_v[layer, r, :, pos[r]] = v[i].contiguous().numpy()
        res = O.decode_dense(qr.contiguous().numpy(), store_k[layer, sl], store_v[layer, sl],
                             pos[sl] + 1, 1 / np.sqrt(D))
        out.copy_(torch.from_numpy(res))

    eng = RequestShardedAttention(geo, dist, None, attend, torch.device("cpu"), torch.float32)
    mine = slice(rank * B_LOCAL, (rank + 1) * B_LOCAL)
    qkv_in = pack_request_inputs(geo, torch.from_numpy(q[:, mine]), torch.from_numpy(kn[:, mine]),
                                 torch.from_numpy(vn[:, mine]))
    out = torch.zeros(geo.q_shape())
    eng.step(qkv_in, out)
    np.save(Path(result_dir) / f"rq{rank}.npy", unpack_request_outputs(geo, out).numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_request_sharded_exchange_matches_oracle(tmp_path):
    import torch.multiprocessing as mp

    from oracle import oracle as O

    lens, ck, cv, q, kn, vn = _req_problem()
    owner = _req_owner(lens)
    assert sorted(set(owner)) == [0, 1]  # both ranks attend, with requests from both sources
    os.environ["PYTHONPATH"] = str(ROOT) + os.pathsep + os.environ.get("PYTHONPATH", "")
    mp.spawn(_req_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True)
    for rank in range(WORLD):
        got = np.load(tmp_path / f"rq{rank}.npy")          # [L, B_local, Hq, D]
        for layer in range(L):
            for b in range(B_LOCAL):
                req = rank * B_LOCAL + b
                k = ck[layer, req:req + 1].copy()
                v = cv[layer, req:req + 1].copy()
                k[0, :, lens[req]] = kn[layer, req]
                v[0, :, lens[req]] = vn[layer, req]
                want = O.decode_dense(q[layer, req:req + 1], k, v, [lens[req] + 1], 1 / np.sqrt(D))[0]
                assert np.allclose(got[layer, b], want, rtol=0, atol=1e-6)


def test_request_geometry():
    from paper_2405_01814_b200.attention import request_partition
    from paper_2405_01814_b200.dist import RequestGeometry

    # the reference's imbalance case (test_attention.cpp:271-282): sizes 8192 + 7 x 512 over 2
    sizes = [8192] + [512] * 7
    a = request_partition(sizes, 2)
    geos = [RequestGeometry(r, 2, 1, 4, 8, 1, 128, a.device_of) for r in range(2)]
    # every request is attended exactly once, and every send count meets a receive count
    assert sorted(r for g in geos for r in g.rows) == list(range(8))
    for m in range(2):
        for s in range(2):
            for d in range(2):
                assert geos[s].send_counts[m][d] == geos[d].recv_counts[m][s]
    with pytest.raises(ValueError):
        RequestGeometry(0, 2, 1, 4, 8, 1, 128, [0] * 7)


# ---- the head-sharded exchange at 8 ranks (the driver's largest scaling point), gloo ----
W8, HQ8, HKV8, B8 = 8, 16, 8, 2


def _w8_problem(seed=5):
    rng = np.random.default_rng(seed)
    B = W8 * B8
    lens = rng.integers(1, 12, B).astype(np.int32)
    lmax = int(lens.max()) + 1
    ck = rng.uniform(-1, 1, (1, B, HKV8, lmax, D)).astype(np.float32)
    cv = rng.uniform(-1, 1, (1, B, HKV8, lmax, D)).astype(np.float32)
    q = rng.uniform(-1, 1, (1, B, HQ8, D)).astype(np.float32)
    kn = rng.uniform(-1, 1, (1, B, HKV8, D)).astype(np.float32)
    vn = rng.uniform(-1, 1, (1, B, HKV8, D)).astype(np.float32)
    return lens, ck, cv, q, kn, vn


def _w8_worker(rank, port, result_dir):
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2405_01814_b200.dist import (HeadShardedAttention, ShardGeometry, shard_inputs,
                                            stitch_outputs)

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=W8)
    geo = ShardGeometry(rank, W8, 1, B8, HQ8, HKV8, D, 2)
    lens, ck, cv, q, kn, vn = _w8_problem()
    h0, h1 = rank * geo.hkv_l, (rank + 1) * geo.hkv_l
    row_req = np.zeros(geo.B_attn, np.int64)
    for src in range(W8):
        for b in range(B8):
            row_req[geo.kv_row(src, b)] = src * B8 + b
    sk, sv = ck[:, row_req, h0:h1].copy(), cv[:, row_req, h0:h1].copy()
    pos = lens[row_req]

    def attend(layer, m, qr, k, v, out):
        sl = slice(m * geo.B_mb, (m + 1) * geo.B_mb)
        for i, r in enumerate(range(sl.start, sl.stop)):
            sk[layer, r, :, pos[r]] = k[i].contiguous().numpy()
            sv[layer, r, :, pos[r]] = v[i].contiguous().numpy()
        out.copy_(torch.from_numpy(O.decode_dense(qr.contiguous().numpy(), sk[layer, sl],
                                                  sv[layer, sl], pos[sl] + 1, 1 / np.sqrt(D))))

    eng = HeadShardedAttention(geo, dist, None, attend, torch.device("cpu"), torch.float32)
    mine = slice(rank * B8, (rank + 1) * B8)
    qkv_in = shard_inputs(torch.from_numpy(q[:, mine]), torch.from_numpy(kn[:, mine]),
                          torch.from_numpy(vn[:, mine]), W8, 2)
    out = torch.zeros(geo.q_shape())
    eng.step(qkv_in, out)
    np.save(Path(result_dir) / f"w8_{rank}.npy", stitch_outputs(out).numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_head_sharded_exchange_8_ranks(tmp_path):
    import torch.multiprocessing as mp

    from oracle import oracle as O

    os.environ["PYTHONPATH"] = str(ROOT) + os.pathsep + os.environ.get("PYTHONPATH", "")
    mp.spawn(_w8_worker, args=(_free_port(), str(tmp_path)), nprocs=W8, join=True)
    lens, ck, cv, q, kn, vn = _w8_problem()
    for rank in range(W8):
        got = np.load(tmp_path / f"w8_{rank}.npy")
        for b in range(B8):
            req = rank * B8 + b
            k, v = ck[0, req:req + 1].copy(), cv[0, req:req + 1].copy()
            k[0, :, lens[req]] = kn[0, req]
            v[0, :, lens[req]] = vn[0, req]
            want = O.decode_dense(q[0, req:req + 1], k, v, [lens[req] + 1], 1 / np.sqrt(D))[0]
            assert np.allclose(got[0, b], want, rtol=0, atol=1e-6)


# ---- strong scaling: one fixed global batch dealt out over 2, 4 and 8 ranks (gloo) ----
BG, HQS, HKVS = 16, 16, 8


def _strong_problem(seed=9):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 12, BG).astype(np.int32)
    lmax = int(lens.max()) + 1
    ck = rng.uniform(-1, 1, (2, BG, HKVS, lmax, D)).astype(np.float32)
    cv = rng.uniform(-1, 1, (2, BG, HKVS, lmax, D)).astype(np.float32)
    q = rng.uniform(-1, 1, (2, BG, HQS, D)).astype(np.float32)
    kn = rng.uniform(-1, 1, (2, BG, HKVS, D)).astype(np.float32)
    vn = rng.uniform(-1, 1, (2, BG, HKVS, D)).astype(np.float32)
    return lens, ck, cv, q, kn, vn


def _strong_worker(rank, world, port, result_dir):
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2405_01814_b200.dist import (HeadShardedAttention, ShardGeometry, local_batch,
                                            shard_inputs, stitch_outputs)

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bl = local_batch(BG, world, "strong")
    geo = ShardGeometry(rank, world, 2, bl, HQS, HKVS, D, 2)
    assert geo.B_attn == BG  # every attention worker sees the whole global batch
    lens, ck, cv, q, kn, vn = _strong_problem()
    h0, h1 = rank * geo.hkv_l, (rank + 1) * geo.hkv_l
    row_req = np.zeros(geo.B_attn, np.int64)
    for src in range(world):
        for b in range(bl):
            row_req[geo.kv_row(src, b)] = src * bl + b
    sk, sv = ck[:, row_req, h0:h1].copy(), cv[:, row_req, h0:h1].copy()
    pos = lens[row_req]

    def attend(layer, m, qr, k, v, out):
        sl = slice(m * geo.B_mb, (m + 1) * geo.B_mb)
        for i, r in enumerate(range(sl.start, sl.stop)):
            sk[layer, r, :, pos[r]] = k[i].contiguous().numpy()
            sv[layer, r, :, pos[r]] = v[i].contiguous().numpy()
        out.copy_(torch.from_numpy(O.decode_dense(qr.contiguous().numpy(), sk[layer, sl],
                                                  sv[layer, sl], pos[sl] + 1, 1 / np.sqrt(D))))

    eng = HeadShardedAttention(geo, dist, None, attend, torch.device("cpu"), torch.float32)
    mine = slice(rank * bl, (rank + 1) * bl)
    qkv_in = shard_inputs(torch.from_numpy(q[:, mine]), torch.from_numpy(kn[:, mine]),
                          torch.from_numpy(vn[:, mine]), world, 2)
    out = torch.zeros(geo.q_shape())
    eng.step(qkv_in, out)
    np.save(Path(result_dir) / f"strong{world}_{rank}.npy", stitch_outputs(out).numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_strong_scaling_geometry_same_global_batch(tmp_path, world):
    """The bench's --scaling strong geometry: the same 16 requests dealt out over N ranks (8 KV
    heads, 1-4 per rank, two micro-batches) give, per global request, the single-process oracle
    over all heads — the same outputs at every N."""
    import torch.multiprocessing as mp

    from oracle import oracle as O

    os.environ["PYTHONPATH"] = str(ROOT) + os.pathsep + os.environ.get("PYTHONPATH", "")
    mp.spawn(_strong_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    lens, ck, cv, q, kn, vn = _strong_problem()
    bl = BG // world
    for rank in range(world):
        got = np.load(tmp_path / f"strong{world}_{rank}.npy")
        for layer in range(2):
            for b in range(bl):
                req = rank * bl + b
                k, v = ck[layer, req:req + 1].copy(), cv[layer, req:req + 1].copy()
                k[0, :, lens[req]] = kn[layer, req]
                v[0, :, lens[req]] = vn[layer, req]
                want = O.decode_dense(q[layer, req:req + 1], k, v, [lens[req] + 1], 1 / np.sqrt(D))[0]
                assert np.allclose(got[layer, b], want, rtol=0, atol=1e-6)


def test_local_batch():
    from paper_2405_01814_b200.dist import local_batch

    assert local_batch(128, 8) == 16 and local_batch(128, 1) == 128
    assert local_batch(64, 4, "weak") == 64
    with pytest.raises(ValueError):
        local_batch(32, 3)
    with pytest.raises(ValueError):
        local_batch(8, 8)  # one request per rank cannot form two micro-batches
