"""lam_decode_peer on one GPU: rows grouped by source with per-source q/k/v and output buffers,
in-kernel sequence-number wait / publish, and programmatic dependent launch — checked bitwise
against lam_decode on the same rows (identical arithmetic, only the addressing differs)."""
import ctypes as C
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup(n_src=2, Bh=4, Hq=8, Hkv=2, D=128, P=64, seed=0):
    from paper_2405_01814_b200.kvcache import PagedKVCache

    g = torch.Generator(device="cuda").manual_seed(seed)
    B = n_src * Bh
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 700, B).astype(np.int32)
    cache = PagedKVCache(1, Hkv, D, P, int((-(-lens // P)).sum()) + 1, B, int(-(-lens.max() // P)),
                         dtype=torch.bfloat16, device=torch.device("cuda"), shuffle_seed=seed)
    cache.set_lengths(lens)
    cache.sync()
    cache.fill_random(g)
    W = Hq + 2 * Hkv
    qkv = [torch.empty((Bh, W, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g)
           for _ in range(n_src)]
    return cache, lens, qkv, dict(n_src=n_src, Bh=Bh, Hq=Hq, Hkv=Hkv, D=D, W=W)


def _reference(cache, lens, qkv, s):
    """lam_decode with fused append over the concatenated rows."""
    from paper_2405_01814_b200 import decode as dec

    Hq, Hkv = s["Hq"], s["Hkv"]
    packed = torch.cat(qkv, 0)
    k = cache.k[0].clone()
    v = cache.v[0].clone()
    out = dec.decode(packed[:, :Hq], k, v, cache.seq_lens, page_table=cache.page_table,
                     max_len=int(lens.max()), k_new=packed[:, Hq:Hq + Hkv],
                     v_new=packed[:, Hq + Hkv:])
    return out, k, v


@pytest.mark.parametrize("sync", ["kernel", "none"])
def test_decode_peer_matches_decode(built, sync):
    from paper_2405_01814_b200 import _lib, decode as dec

    cache, lens, qkv, s = _setup()
    want, k_want, v_want = _reference(cache, lens, qkv, s)
    n_src, Bh, Hq, Hkv, D, W = (s[x] for x in ("n_src", "Bh", "Hq", "Hkv", "D", "W"))
    outs = [torch.zeros((Bh, Hq, D), dtype=torch.bfloat16, device="cuda") for _ in range(n_src)]
    flags = torch.zeros(2 * n_src, dtype=torch.int32, device="cuda")
    qd = torch.empty((n_src * Bh, Hq, D), dtype=torch.bfloat16, device="cuda")
    a, _ = dec.make_args(qd, cache.k[0], cache.v[0], cache.seq_lens, page_table=cache.page_table,
                         max_len=int(lens.max()), out=qd)
    a.q_batch_stride = a.new_batch_stride = W * D
    io = _lib.PeerIO()
    io.n_src, io.rows_per_src = n_src, Bh
    for i in range(n_src):
        io.q_src[i] = qkv[i].data_ptr()
        io.out_dst[i] = outs[i].data_ptr()
    io.k_new_offset, io.v_new_offset = Hq * D, (Hq + Hkv) * D
    lib, ctx = _lib.load(), _lib.context(0)
    Ptrs = C.c_void_p * n_src
    ready = Ptrs(*[flags.data_ptr() + 4 * i for i in range(n_src)])
    done = Ptrs(*[flags.data_ptr() + 4 * (n_src + i) for i in range(n_src)])
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    if sync == "kernel":
        io.n_wait = io.n_done = n_src
        io.wait_value = io.done_value = 1
        for i in range(n_src):
            io.wait_flags[i] = ready[i]
            io.done_flags[i] = done[i]
        torch.cuda.synchronize()
        # the launch is enqueued first and waits inside the kernel for the publication
        _lib.check(lib.lam_decode_peer(ctx.handle, a, io, main.cuda_stream))
        _lib.check(lib.lam_stream_signal(ctx.handle, ready, n_src, 1, side.cuda_stream))
        _lib.check(lib.lam_stream_wait(ctx.handle, done, n_src, 1, side.cuda_stream))
        side.synchronize()  # returns only once the kernel published its outputs
    else:
        _lib.check(lib.lam_decode_peer(ctx.handle, a, io, main.cuda_stream))
    torch.cuda.synchronize()
    got = torch.cat(outs, 0)
    assert torch.equal(got, want)
    assert torch.equal(cache.k[0], k_want) and torch.equal(cache.v[0], v_want)
    if sync == "kernel":
        assert flags.tolist() == [1] * (2 * n_src)


def test_decode_peer_back_to_back_overlapping_launches(built):
    """Many self-synchronising launches in a row (programmatic dependent launch, launch slots
    reused round-robin): every launch's outputs and publication are correct."""
    from paper_2405_01814_b200 import _lib, decode as dec

    cache, lens, qkv, s = _setup(n_src=1, Bh=16, Hq=8, Hkv=1)
    n_src, Bh, Hq, Hkv, D, W = (s[x] for x in ("n_src", "Bh", "Hq", "Hkv", "D", "W"))
    lib, ctx = _lib.load(), _lib.context(0)
    n = 12
    flags = torch.zeros(2, dtype=torch.int32, device="cuda")
    outs = [torch.zeros((Bh, Hq, D), dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    qd = torch.empty((Bh, Hq, D), dtype=torch.bfloat16, device="cuda")
    # every launch appends the same new token (idempotent), so all outputs must be equal
    a, _ = dec.make_args(qd, cache.k[0], cache.v[0], cache.seq_lens, page_table=cache.page_table,
                         max_len=int(lens.max()), out=qd)
    a.q_batch_stride = a.new_batch_stride = W * D
    a.overlap_prev = 1  # consecutive launches may overlap (programmatic dependent launch)
    want, _, _ = _reference(cache, lens, qkv, s)
    torch.cuda.synchronize()
    ready = C.c_void_p(flags.data_ptr())
    done = C.c_void_p(flags.data_ptr() + 4)
    side = torch.cuda.Stream()
    stream = torch.cuda.current_stream().cuda_stream
    ios = []
    for i in range(n):
        io = _lib.PeerIO()
        io.n_src, io.rows_per_src = 1, Bh
        io.q_src[0], io.out_dst[0] = qkv[0].data_ptr(), outs[i].data_ptr()
        io.k_new_offset, io.v_new_offset = Hq * D, (Hq + Hkv) * D
        io.n_wait = io.n_done = 1
        io.wait_value = io.done_value = i + 1
        io.wait_flags[0], io.done_flags[0] = ready.value, done.value
        ios.append(io)
        _lib.check(lib.lam_decode_peer(ctx.handle, a, io, stream))
    for i in range(n):  # publish inputs one launch at a time, in order
        arr = (C.c_void_p * 1)(ready.value)
        _lib.check(lib.lam_stream_signal(ctx.handle, arr, 1, i + 1, side.cuda_stream))
    torch.cuda.synchronize()
    for i in range(n):
        assert torch.equal(outs[i], want), i
    # overlapping launches may publish out of order; every launch published a value in range
    assert flags[0].item() == n and 1 <= flags[1].item() <= n
    del ios


def test_decode_peer_validation(built):
    from paper_2405_01814_b200 import _lib

    lib, ctx = _lib.load(), _lib.context(0)
    a = _lib.DecodeArgs()
    io = _lib.PeerIO()
    with pytest.raises(_lib.ValidationError):
        _lib.check(lib.lam_decode_peer(ctx.handle, a, None, None))
    cache, lens, qkv, s = _setup()
    from paper_2405_01814_b200 import decode as dec

    qd = torch.empty((8, 8, 128), dtype=torch.bfloat16, device="cuda")
    a, _ = dec.make_args(qd, cache.k[0], cache.v[0], cache.seq_lens, page_table=cache.page_table,
                         max_len=int(lens.max()), out=qd)
    io.n_src, io.rows_per_src = 3, 4  # 3 * 4 != batch 8
    with pytest.raises(_lib.ValidationError):
        _lib.check(lib.lam_decode_peer(ctx.handle, a, io, None))
    io.n_src, io.rows_per_src = 2, 4
    with pytest.raises(_lib.ValidationError, match="null"):
        _lib.check(lib.lam_decode_peer(ctx.handle, a, io, None))
    assert math.isfinite(1.0)


def _peer_io(n_src, Bh, Hq, Hkv, D, qkv, outs, flags=None, value=1):
    from paper_2405_01814_b200 import _lib

    io = _lib.PeerIO()
    io.n_src, io.rows_per_src = n_src, Bh
    for i in range(n_src):
        io.q_src[i] = qkv[i].data_ptr()
        io.out_dst[i] = outs[i].data_ptr()
    io.k_new_offset, io.v_new_offset = Hq * D, (Hq + Hkv) * D
    if flags is not None:
        io.n_wait = io.n_done = n_src
        io.wait_value = io.done_value = value
        for i in range(n_src):
            io.wait_flags[i] = flags.data_ptr() + 4 * i
            io.done_flags[i] = flags.data_ptr() + 4 * (n_src + i)
    return io


@pytest.mark.parametrize("n_src,Bh,G", [(2, 3, 8), (3, 2, 1), (5, 2, 8), (8, 2, 8), (8, 1, 4)])
def test_decode_peer_vs_oracle(built, n_src, Bh, G):
    """The peer-transport launch (rows grouped by source, q / k_new / v_new read from each
    source's packed rows, outputs stored into each source's buffer, in-kernel sequence numbers)
    against the CPU oracle: fused append bit-exact (the oracle's byte paging of the pool equals
    the dense cache with the new token at seq_len - 1) and attention within the bf16 bound
    (exact_attention<float> on the upcast values, attention.cpp:48-70)."""
    from oracle import oracle as O
    from paper_2405_01814_b200 import _lib, decode as dec
    from tests.helpers import oracle_decode

    Hkv, D = 2, 128
    Hq = Hkv * G
    cache, lens, qkv, s = _setup(n_src=n_src, Bh=Bh, Hq=Hq, Hkv=Hkv, D=D, seed=n_src * 10 + G)
    B, W, P = n_src * Bh, s["W"], cache.k.shape[3]
    lmax = int(lens.max())
    pt = cache.page_table.cpu().numpy()
    # the cache before the step, dense, with each request's new token written at len - 1
    k_dense = dec.kv_gather(cache.k[0], cache.page_table, cache.seq_lens, lmax).cpu()
    v_dense = dec.kv_gather(cache.v[0], cache.page_table, cache.seq_lens, lmax).cpu()
    packed = torch.cat(qkv, 0).cpu()
    for b in range(B):
        k_dense[b, :, lens[b] - 1] = packed[b, Hq:Hq + Hkv]
        v_dense[b, :, lens[b] - 1] = packed[b, Hq + Hkv:]
    outs = [torch.zeros((Bh, Hq, D), dtype=torch.float32, device="cuda") for _ in range(n_src)]
    flags = torch.zeros(2 * n_src, dtype=torch.int32, device="cuda")
    qd = torch.empty((B, Hq, D), dtype=torch.bfloat16, device="cuda")
    a, _ = dec.make_args(qd, cache.k[0], cache.v[0], cache.seq_lens, page_table=cache.page_table,
                         max_len=lmax, out=torch.empty((B, Hq, D), device="cuda"))
    a.q_batch_stride = a.new_batch_stride = W * D
    io = _peer_io(n_src, Bh, Hq, Hkv, D, qkv, outs, flags, value=7)
    lib, ctx = _lib.load(), _lib.context(0)
    torch.cuda.synchronize()
    _lib.check(lib.lam_decode_peer(ctx.handle, a, io, torch.cuda.current_stream().cuda_stream))
    side = torch.cuda.Stream()
    ready = (C.c_void_p * n_src)(*[flags.data_ptr() + 4 * i for i in range(n_src)])
    _lib.check(lib.lam_stream_signal(ctx.handle, ready, n_src, 7, side.cuda_stream))
    torch.cuda.synchronize()
    assert flags.tolist() == [7] * (2 * n_src)
    assert ctx.status() == _lib.LAM_STATUS_OK
    # append: byte-exact against the oracle's page gather of the pool the kernel wrote
    for pool, dense in ((cache.k[0], k_dense), (cache.v[0], v_dense)):
        pool_bytes = pool.view(torch.uint8).cpu().numpy().reshape(pool.shape[0], Hkv, P, D * 2)
        got = O.page_gather(pool_bytes, pt, lens, lmax)
        assert np.array_equal(got, dense.view(torch.uint8).numpy().reshape(got.shape))
    want = oracle_decode(packed[:, :Hq], k_dense, v_dense, lens, 1 / math.sqrt(D))
    got = torch.cat(outs, 0).cpu().numpy()
    assert float(np.abs(got - want).max()) <= 2e-3


def test_decode_peer_row_map_vs_oracle(built):
    """Row map (lam_peer_io.row_src, the request-level partition on the peer transport): the
    launch's rows come from the sources in any number and order — here 7 of 3 x 3 source rows,
    shuffled, one source row unused — and each row's q / new K/V are read from, and its output
    stored to, the (source, row) the map names.  Fused append bit-exact, attention vs the CPU
    oracle within the bf16 bound."""
    from oracle import oracle as O
    from paper_2405_01814_b200 import _lib, decode as dec
    from tests.helpers import oracle_decode

    n_src, Bh, G, Hkv, D = 3, 3, 8, 2, 128
    Hq = Hkv * G
    cache, lens, qkv, s = _setup(n_src=n_src, Bh=Bh, Hq=Hq, Hkv=Hkv, D=D, seed=77)
    W, P = s["W"], cache.k.shape[3]
    Bn = 7
    perm = np.random.default_rng(5).permutation(n_src * Bh)[:Bn]  # row b <- source row perm[b]
    lens = lens[:Bn]
    lmax = int(lens.max())
    pt = cache.page_table.cpu().numpy()[:Bn]
    k_dense = dec.kv_gather(cache.k[0], cache.page_table[:Bn], cache.seq_lens[:Bn], lmax).cpu()
    v_dense = dec.kv_gather(cache.v[0], cache.page_table[:Bn], cache.seq_lens[:Bn], lmax).cpu()
    packed = torch.cat(qkv, 0).cpu()[perm]  # the rows each attention row reads
    for b in range(Bn):
        k_dense[b, :, lens[b] - 1] = packed[b, Hq:Hq + Hkv]
        v_dense[b, :, lens[b] - 1] = packed[b, Hq + Hkv:]
    outs = [torch.zeros((Bh, Hq, D), dtype=torch.float32, device="cuda") for _ in range(n_src)]
    flags = torch.zeros(2 * n_src, dtype=torch.int32, device="cuda")
    qd = torch.empty((Bn, Hq, D), dtype=torch.bfloat16, device="cuda")
    a, _ = dec.make_args(qd, cache.k[0], cache.v[0], cache.seq_lens[:Bn],
                         page_table=cache.page_table[:Bn], max_len=lmax,
                         out=torch.empty((Bn, Hq, D), device="cuda"))
    a.q_batch_stride = a.new_batch_stride = W * D
    io = _peer_io(n_src, Bh, Hq, Hkv, D, qkv, outs, flags, value=9)
    io.rows_per_src = 1  # ignored with a row map
    row_src = torch.tensor([(int(r) // Bh) << 24 | (int(r) % Bh) for r in perm], dtype=torch.int32,
                           device="cuda")
    io.row_src = row_src.data_ptr()
    lib, ctx = _lib.load(), _lib.context(0)
    torch.cuda.synchronize()
    _lib.check(lib.lam_decode_peer(ctx.handle, a, io, torch.cuda.current_stream().cuda_stream))
    side = torch.cuda.Stream()
    ready = (C.c_void_p * n_src)(*[flags.data_ptr() + 4 * i for i in range(n_src)])
    _lib.check(lib.lam_stream_signal(ctx.handle, ready, n_src, 9, side.cuda_stream))
    torch.cuda.synchronize()
    assert flags.tolist() == [9] * (2 * n_src)
    assert ctx.status() == _lib.LAM_STATUS_OK
    for pool, dense in ((cache.k[0], k_dense), (cache.v[0], v_dense)):
        pool_bytes = pool.view(torch.uint8).cpu().numpy().reshape(pool.shape[0], Hkv, P, D * 2)
        got = O.page_gather(pool_bytes, pt, lens, lmax)
        assert np.array_equal(got, dense.view(torch.uint8).numpy().reshape(got.shape))
    want = oracle_decode(packed[:, :Hq], k_dense, v_dense, lens, 1 / math.sqrt(D))
    got_src = torch.cat(outs, 0).cpu().numpy()
    assert float(np.abs(got_src[perm] - want).max()) <= 2e-3
    unused = sorted(set(range(n_src * Bh)) - set(int(r) for r in perm))
    assert not got_src[unused].any()  # rows no attention row maps to are never written


def test_spin_timeout_reports_status_instead_of_trapping(built):
    """A launch whose inputs are never published gives up after the context's spin timeout:
    it records LAM_STATUS_INPUT_TIMEOUT, still publishes its done flags, and the context stays
    usable for the next launch."""
    from paper_2405_01814_b200 import _lib, decode as dec

    cache, lens, qkv, s = _setup(n_src=2, Bh=2, Hq=8, Hkv=2)
    n_src, Bh, Hq, Hkv, D, W = (s[x] for x in ("n_src", "Bh", "Hq", "Hkv", "D", "W"))
    ctx = _lib.Context(0)  # own context: its timeout does not leak into other tests
    try:
        ctx.set_spin_timeout(20_000_000)  # 20 ms
        outs = [torch.zeros((Bh, Hq, D), dtype=torch.bfloat16, device="cuda") for _ in range(n_src)]
        flags = torch.zeros(2 * n_src, dtype=torch.int32, device="cuda")
        qd = torch.empty((n_src * Bh, Hq, D), dtype=torch.bfloat16, device="cuda")
        a, _ = dec.make_args(qd, cache.k[0].clone(), cache.v[0].clone(), cache.seq_lens,
                             page_table=cache.page_table, max_len=int(lens.max()), out=qd)
        a.q_batch_stride = a.new_batch_stride = W * D
        io = _peer_io(n_src, Bh, Hq, Hkv, D, qkv, outs, flags, value=3)
        lib = _lib.load()
        _lib.check(lib.lam_decode_peer(ctx.handle, a, io, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()  # returns: the kernel gave up instead of hanging or trapping
        assert ctx.status() == _lib.LAM_STATUS_INPUT_TIMEOUT
        assert flags[n_src:].tolist() == [3] * n_src
        assert ctx.status() == _lib.LAM_STATUS_OK  # cleared by the read
        # the context still works: publish and rerun
        flags[:n_src] = 4
        io.wait_value = io.done_value = 4
        want, _, _ = _reference(cache, lens, qkv, s)
        a2, _ = dec.make_args(qd, cache.k[0], cache.v[0], cache.seq_lens,
                              page_table=cache.page_table, max_len=int(lens.max()), out=qd)
        a2.q_batch_stride = a2.new_batch_stride = W * D
        _lib.check(lib.lam_decode_peer(ctx.handle, a2, io, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        assert ctx.status() == _lib.LAM_STATUS_OK
        assert torch.equal(torch.cat(outs, 0), want)
    finally:
        ctx.close()


@pytest.mark.parametrize("G", [8, 1])
def test_eager_q_new_rows_awaited_separately(built, G):
    """Eager q (lam_peer_io.n_wait_kv): q published alone lets the launch attend over the cached
    tokens but not finish — it cannot publish its outputs until the new K / V rows are announced;
    once they are, the result equals the fused launch bitwise."""
    import time

    from paper_2405_01814_b200 import _lib, decode as dec

    n_src, Bh, Hkv, D = 2, 3, 2, 128
    Hq = Hkv * G
    cache, lens, qkv, s = _setup(n_src=n_src, Bh=Bh, Hq=Hq, Hkv=Hkv, D=D, seed=31 + G)
    W = s["W"]
    want, k_want, v_want = _reference(cache, lens, qkv, s)
    outs = [torch.zeros((Bh, Hq, D), dtype=torch.bfloat16, device="cuda") for _ in range(n_src)]
    flags = torch.zeros(3 * n_src, dtype=torch.int32, device="cuda")  # q ready | kv ready | done
    qd = torch.empty((n_src * Bh, Hq, D), dtype=torch.bfloat16, device="cuda")
    a, _ = dec.make_args(qd, cache.k[0], cache.v[0], cache.seq_lens, page_table=cache.page_table,
                         max_len=int(lens.max()), out=qd)
    a.q_batch_stride = a.new_batch_stride = W * D
    io = _peer_io(n_src, Bh, Hq, Hkv, D, qkv, outs)
    fp = flags.data_ptr()
    io.n_wait = io.n_done = io.n_wait_kv = n_src
    io.wait_value = io.done_value = io.kv_wait_value = 5
    for i in range(n_src):
        io.wait_flags[i] = fp + 4 * i
        io.kv_wait_flags[i] = fp + 4 * (n_src + i)
        io.done_flags[i] = fp + 4 * (2 * n_src + i)
    lib, ctx = _lib.load(), _lib.context(0)
    side = torch.cuda.Stream()  # (created before the launch occupies the GPU)
    P = C.c_void_p * n_src
    torch.cuda.synchronize()
    _lib.check(lib.lam_decode_peer(ctx.handle, a, io, torch.cuda.current_stream().cuda_stream))
    _lib.check(lib.lam_stream_signal(ctx.handle, P(*[fp + 4 * i for i in range(n_src)]), n_src, 5,
                                     side.cuda_stream))
    side.synchronize()
    time.sleep(0.05)
    with torch.cuda.stream(side):  # (the launch's own stream is still busy)
        done = flags[2 * n_src:].cpu().tolist()
    assert done == [0] * n_src  # q alone does not finish the launch
    _lib.check(lib.lam_stream_signal(ctx.handle, P(*[fp + 4 * (n_src + i) for i in range(n_src)]),
                                     n_src, 5, side.cuda_stream))
    torch.cuda.synchronize()
    assert ctx.status() == _lib.LAM_STATUS_OK
    assert flags[2 * n_src:].tolist() == [5] * n_src
    assert torch.equal(torch.cat(outs, 0), want)
    assert torch.equal(cache.k[0], k_want) and torch.equal(cache.v[0], v_want)
