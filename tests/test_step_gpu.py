"""The step launch (lam_decode_step): every layer and micro-batch of a decode step in one
persistent grid.  Checked bitwise against one lam_decode launch per (layer, micro-batch) — the
same items with the same arithmetic, only scheduled across launch boundaries — and, for the
peer transport, with in-kernel per-layer sequence numbers driven by a model-worker stream."""
import ctypes as C

import numpy as np
import pytest
import torch

from tests.helpers import oracle_decode

pytestmark = pytest.mark.gpu


def _problem(L, MB, rows, Hq, Hkv, D=128, P=64, seed=0, pool_layers=None):
    from paper_2405_01814_b200.kvcache import PagedKVCache

    g = torch.Generator(device="cuda").manual_seed(seed)
    B = MB * rows
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 700, B).astype(np.int32)
    lens[0] = 1
    cache = PagedKVCache(pool_layers or L, Hkv, D, P, int((-(-lens // P)).sum()) + 2, B,
                         int(-(-lens.max() // P)), dtype=torch.bfloat16,
                         device=torch.device("cuda"), shuffle_seed=seed)
    cache.set_lengths(lens)
    cache.sync()
    cache.fill_random(g)
    W = Hq + 2 * Hkv
    x = torch.empty((L, B, W, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g)
    order = torch.cat([torch.argsort(cache.seq_lens[m * rows:(m + 1) * rows], descending=True,
                                     stable=True) for m in range(MB)]).to(torch.int32)
    return cache, lens, x, order


def _reference(cache, lens, x, order, L, MB, rows, Hq, Hkv, kernel, layer0=0, split=0):
    """One lam_decode per (layer, micro-batch), S = 1 (or the given split), on cloned pools."""
    from paper_2405_01814_b200 import decode as dec

    k, v = cache.k.clone(), cache.v.clone()
    out = torch.empty((L, MB * rows, Hq, x.shape[-1]), dtype=x.dtype, device="cuda")
    for layer in range(L):
        pl = (layer0 + layer) % k.shape[0]
        for m in range(MB):
            sl = slice(m * rows, (m + 1) * rows)
            xs = x[layer, sl]
            out[layer, sl] = dec.decode(xs[:, :Hq], k[pl], v[pl], cache.seq_lens[sl],
                                        page_table=cache.page_table[sl], max_len=int(lens.max()),
                                        k_new=xs[:, Hq:Hq + Hkv], v_new=xs[:, Hq + Hkv:],
                                        request_order=order[sl], kernel=kernel,
                                        split_tokens=split or int(lens.max()))
    return out, k, v


@pytest.mark.parametrize("kernel,G", [("auto", 8), ("gqa_tc", 8), ("auto", 1), ("gqa_mma", 1),
                                      ("simt", 2)])
@pytest.mark.parametrize("L,MB,layer0,pool_layers,split", [(3, 2, 0, None, 0), (3, 1, 2, 3, 0),
                                                           (3, 2, 1, 4, 128)])
def test_step_launch_equals_per_layer_launches(built, kernel, G, L, MB, layer0, pool_layers, split):
    from paper_2405_01814_b200 import decode as dec

    rows, Hkv = 5, 2
    Hq = Hkv * G
    cache, lens, x, order = _problem(L, MB, rows, Hq, Hkv, seed=G + L, pool_layers=pool_layers)
    want, k_want, v_want = _reference(cache, lens, x, order, L, MB, rows, Hq, Hkv, kernel, layer0,
                                      split)
    got = dec.decode_step(x[:, :, :Hq], cache.k, cache.v, cache.seq_lens, n_mb=MB,
                          page_table=cache.page_table, max_len=int(lens.max()),
                          k_new=x[:, :, Hq:Hq + Hkv], v_new=x[:, :, Hq + Hkv:],
                          request_order=order, kernel=kernel, layer0=layer0, split_tokens=split)
    torch.cuda.synchronize()
    assert torch.equal(got, want)
    assert torch.equal(cache.k, k_want) and torch.equal(cache.v, v_want)
    # and against the oracle for one (layer, request, head)
    b, h = int(np.argmax(lens)), Hq - 1
    pl = (layer0 + L - 1) % cache.k.shape[0]
    kd = dec.kv_gather(cache.k[pl], cache.page_table, cache.seq_lens, int(lens.max()))
    vd = dec.kv_gather(cache.v[pl], cache.page_table, cache.seq_lens, int(lens.max()))
    ref = oracle_decode(x[L - 1, b:b + 1, h:h + 1], kd[b:b + 1, h // G:h // G + 1],
                        vd[b:b + 1, h // G:h // G + 1], [int(lens[b])], 128 ** -0.5)
    assert float(np.abs(got[L - 1, b, h].float().cpu().numpy() - ref[0, 0]).max()) <= 2e-3 + 2 ** -9


@pytest.mark.parametrize("mode", ["stream", "ahead", "relay"])
@pytest.mark.parametrize("kernel", ["auto", "gqa_tc"])
def test_step_launch_peer_sequence_numbers(built, kernel, mode):
    """Peer-io step launch: two sources, two micro-batches, three layers.  The kernel is enqueued
    first; a model-worker stream then publishes layer l of micro-batch m only after the kernel
    published layer l - 1 of m (the data dependency through the model) — so the grid must wait
    per (layer, micro-batch) inside the kernel and publish per (layer, micro-batch).
    mode="ahead": every layer published before the launch; mode="relay": the launch forwards
    layers 1.. itself (lam_peer_io.n_relay: one qkv flag, awaited for both sources)."""
    ahead = mode == "ahead"
    from paper_2405_01814_b200 import _lib, decode as dec

    L, MB, n_src, Bh, Hq, Hkv, D = 3, 2, 2, 3, 16, 2, 128
    rows = n_src * Bh
    cache, lens, x, order = _problem(L, MB, rows, Hq, Hkv, seed=5)
    W = Hq + 2 * Hkv
    want, k_want, v_want = _reference(cache, lens, x, order, L, MB, rows, Hq, Hkv, kernel)
    # model-worker buffers: source s holds [L][MB][Bh][W][D] rows and [L][MB][Bh][Hq][D] outputs
    xs = x.view(L, MB, n_src, Bh, W, D)
    qkv = [xs[:, :, s].contiguous() for s in range(n_src)]
    outs = [torch.zeros((L, MB, Bh, Hq, D), dtype=torch.bfloat16, device="cuda") for _ in range(n_src)]
    flags = torch.zeros((2, MB, n_src), dtype=torch.int32, device="cuda")  # [qkv_ready | out_ready]
    qd = torch.empty((MB * rows, Hq, D), dtype=torch.bfloat16, device="cuda")
    a, _ = dec.make_args(qd, cache.k[0], cache.v[0], cache.seq_lens, page_table=cache.page_table,
                         max_len=int(lens.max()), out=qd, kernel=kernel)
    a.q_batch_stride = a.new_batch_stride = W * D
    a.request_order = order.data_ptr()
    a.split_tokens = int(lens.max())  # S = 1, as the reference (bitwise comparison)
    io = _lib.PeerIO()
    io.n_src, io.rows_per_src = n_src, Bh
    for s in range(n_src):
        io.q_src[s] = qkv[s].data_ptr()
        io.out_dst[s] = outs[s].data_ptr()
    io.k_new_offset, io.v_new_offset = Hq * D, (Hq + Hkv) * D
    io.n_wait = io.n_done = n_src
    fp = flags.data_ptr()
    for s in range(n_src):
        io.wait_flags[s] = fp + 4 * (s if mode != "relay" else 0)  # qkv_ready[mb 0][s]
        io.done_flags[s] = fp + 4 * (MB * n_src + s)     # out_ready[mb 0][s]
    epoch = 100
    if mode == "relay":
        io.n_relay = n_src
        io.relay_flag = fp
        for s in range(n_src):
            io.relay_wait_flags[s] = fp + 4 * (MB * n_src + s)
        flags[0, :, 0] = epoch + 1  # layer 0's inputs; the launch forwards the rest
    st = dec.step_layout(L, MB, rows, pool_layer_rows=cache.k[0].numel() // D, lm_q_stride=Bh * W * D,
                         lm_out_stride=Bh * Hq * D, flag_mb_stride=n_src, epoch=epoch)
    lib, ctx = _lib.load(), _lib.context(0)
    # (streams are created before the persistent grid occupies the GPU: creating one lazily can
    # wait for the running kernel)
    model = torch.cuda.Stream()
    P = C.c_void_p * n_src
    if ahead:  # every layer's inputs published before the launch: layers may finish out of order
        flags[0] = epoch + L
    torch.cuda.synchronize()
    _lib.check(lib.lam_decode_step(ctx.handle, a, st, io, torch.cuda.current_stream().cuda_stream))
    for layer in range(L if mode == "stream" else 0):
        for m in range(MB):
            if layer > 0:
                done = P(*[fp + 4 * ((MB + m) * n_src + s) for s in range(n_src)])
                _lib.check(lib.lam_stream_wait(ctx.handle, done, n_src, epoch + layer, model.cuda_stream))
            ready = P(*[fp + 4 * (m * n_src + s) for s in range(n_src)])
            _lib.check(lib.lam_stream_signal(ctx.handle, ready, n_src, epoch + layer + 1, model.cuda_stream))
    torch.cuda.synchronize()
    assert ctx.status() == _lib.LAM_STATUS_OK
    if mode == "relay":
        assert flags.tolist() == [[[epoch + L, 0]] * MB, [[epoch + L] * n_src] * MB]
    else:
        assert flags.tolist() == [[[epoch + L] * n_src] * MB] * 2
    got = torch.stack(outs, 2).view(L, MB * rows, Hq, D)
    assert torch.equal(got, want)
    assert torch.equal(cache.k, k_want) and torch.equal(cache.v, v_want)


@pytest.mark.parametrize("L", [1, 4])
def test_step_from_host_matches_device_step(built, L):
    """lam_decode_step_from_host (host buffers in and out, per-layer sequence numbers between the
    copy stream and the step launch), called twice so the sequence numbers carry across calls,
    equals the device-resident step launch bitwise — outputs and appended pools.  L = 1 is an
    ordinary launch that waits for, and publishes, the same sequence numbers."""
    from paper_2405_01814_b200 import _lib, decode as dec

    rows, Hq, Hkv, D = 6, 16, 2, 128
    cache, lens, x, order = _problem(L, 1, rows, Hq, Hkv, seed=9)
    k0, v0 = cache.k.clone(), cache.v.clone()
    want = dec.decode_step(x[:, :, :Hq], cache.k, cache.v, cache.seq_lens, page_table=cache.page_table,
                           max_len=int(lens.max()), k_new=x[:, :, Hq:Hq + Hkv], v_new=x[:, :, Hq + Hkv:],
                           request_order=order)
    k_want, v_want = cache.k.clone(), cache.v.clone()
    hq = x[:, :, :Hq].contiguous().cpu().pin_memory()
    hk = x[:, :, Hq:Hq + Hkv].contiguous().cpu().pin_memory()
    hv = x[:, :, Hq + Hkv:].contiguous().cpu().pin_memory()
    ho = torch.zeros((L, rows, Hq, D), dtype=torch.bfloat16).pin_memory()
    dq = torch.empty((rows, Hq, D), dtype=torch.bfloat16, device="cuda")
    a, _ = dec.make_args(dq, cache.k[0], cache.v[0], cache.seq_lens, page_table=cache.page_table,
                         max_len=int(lens.max()), out=torch.empty_like(dq), request_order=order)
    st = dec.step_layout(L, 1, rows, pool_layers=L, pool_layer_rows=cache.k[0].numel() // D)
    lib, ctx = _lib.load(), _lib.context(0)
    stage = torch.empty(int(lib.lam_decode_step_from_host_stage_bytes(a, L)), dtype=torch.uint8,
                        device="cuda")
    P = C.c_void_p * L
    s, xs = torch.cuda.current_stream(), torch.cuda.Stream()
    for rep in range(2):
        cache.k.copy_(k0)
        cache.v.copy_(v0)
        ho.zero_()
        torch.cuda.synchronize()
        _lib.check(lib.lam_decode_step_from_host(
            ctx.handle, a, st, P(*[hq[i].data_ptr() for i in range(L)]),
            P(*[hk[i].data_ptr() for i in range(L)]), P(*[hv[i].data_ptr() for i in range(L)]),
            P(*[ho[i].data_ptr() for i in range(L)]), stage.data_ptr(), s.cuda_stream, xs.cuda_stream))
        torch.cuda.synchronize()
        assert ctx.status() == _lib.LAM_STATUS_OK
        assert torch.equal(ho, want.cpu()), rep
        assert torch.equal(cache.k, k_want) and torch.equal(cache.v, v_want)
