"""Parity of the production decode path (lam_decode, lam_kv_append, lam_kv_gather) against
the CPU oracle on identical inputs.

Tolerances (north star): fp32 KV max-abs <= 1e-5 against exact_attention<float>;
bf16/fp16 KV max-abs <= 2e-3 against exact_attention<float> on the exactly upcast values
(fp32 output, so the bound measures the kernel, not the final rounding).  Paging and
appends are bit-exact.
"""
import math

import numpy as np
import pytest
import torch

from tests.helpers import make_dense, oracle_decode, page_table_for, to_paged

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-5, torch.bfloat16: 2e-3, torch.float16: 2e-3}


def _decode(*a, **kw):
    from paper_2405_01814_b200 import decode as dec

    return dec.decode(*a, **kw)


def _lens_t(lens):
    return torch.tensor(np.asarray(lens, np.int32), device="cuda")


def _maxabs(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))))


def test_config1_fp32_mha_full_parity(built):
    """BASELINE config 1: B=8, 32 heads, d=128, l=1024, fp32 — every head vs the oracle."""
    B, H, D, L = 8, 32, 128, 1024
    q, k, v = make_dense(B, H, H, D, L, torch.float32, seed=1)
    lens = [L] * B
    scale = 1 / math.sqrt(D)
    want = oracle_decode(q, k, v, lens, scale)
    for split in (0, 256, 96):
        out = _decode(q, k, v, _lens_t(lens), scale=scale, split_tokens=split)
        torch.cuda.synchronize()
        assert _maxabs(out.cpu().numpy(), want) <= 1e-5, split


def test_golden_fixtures(built, golden):
    for name, dtype in (("decode_mha_f32.npz", torch.float32), ("decode_gqa_bf16.npz", torch.bfloat16)):
        g = golden(name)
        q = torch.tensor(g["q"], device="cuda").to(dtype)
        k = torch.tensor(g["k"], device="cuda").to(dtype)
        v = torch.tensor(g["v"], device="cuda").to(dtype)
        out = _decode(q, k, v, _lens_t(g["lens"]), scale=float(g["scale"]), out_dtype=torch.float32)
        assert _maxabs(out.cpu().numpy(), g["out_f32"]) <= TOL[dtype], name


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("paged", [False, True])
@pytest.mark.parametrize("kernel", ["auto", "simt", "gqa_mma", "gqa_tc"])
def test_decode_vs_oracle(built, dtype, G, paged, kernel):
    if kernel in ("gqa_mma", "gqa_tc") and dtype == torch.float32:
        pytest.skip("tensor-core kernel is 16-bit only")
    B, Hkv, D = 3, 2, 128
    Hq = Hkv * G
    lens = [1, 77, 300]
    lmax = 320
    q, k, v = make_dense(B, Hq, Hkv, D, lmax, dtype, seed=G * 10 + int(paged))
    for b, l in enumerate(lens):  # poison rows past the sequence end
        k[b, :, l:] = float("nan")
        v[b, :, l:] = float("nan")
    scale = 1 / math.sqrt(D)
    want, want_lse = oracle_decode(q, k, v, lens, scale, want_lse=True)
    if paged:
        P = 64
        pt, npages = page_table_for(lens, P, seed=G)
        kp, vp = to_paged(k, lens, P, pt, npages), to_paged(v, lens, P, pt, npages)
        ptt = torch.tensor(pt, device="cuda")
    else:
        kp, vp, ptt = k, v, None
    for split in (0, 64, 128):
        out, lse = _decode(q, kp, vp, _lens_t(lens), page_table=ptt, max_len=max(lens),
                           scale=scale, out_dtype=torch.float32, split_tokens=split,
                           return_lse=True, kernel=kernel)
        torch.cuda.synchronize()
        assert _maxabs(out.cpu().numpy(), want) <= TOL[dtype], (split,)
        assert _maxabs(lse.cpu().numpy(), want_lse) <= 1e-3, (split,)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_paged_equals_dense_bitwise(built, dtype):
    B, Hq, Hkv, D = 4, 16, 2 if dtype == torch.bfloat16 else 16, 128
    lens = [64, 640, 1000, 5]
    lmax = 1024
    q, k, v = make_dense(B, Hq, Hkv, D, lmax, dtype, seed=7)
    pt, npages = page_table_for(lens, 64, seed=3)
    kp, vp = to_paged(k, lens, 64, pt, npages), to_paged(v, lens, 64, pt, npages)
    for split in (128, 0):
        a = _decode(q, k, v, _lens_t(lens), split_tokens=split, max_len=max(lens))
        b = _decode(q, kp, vp, _lens_t(lens), page_table=torch.tensor(pt, device="cuda"),
                    split_tokens=split, max_len=max(lens))
        assert torch.equal(a, b)
        c = _decode(q, k, v, _lens_t(lens), split_tokens=split, max_len=max(lens))
        assert torch.equal(a, c)  # deterministic


def test_bf16_output_is_rounded_fp32_output(built):
    q, k, v = make_dense(2, 16, 2, 128, 200, torch.bfloat16, seed=5)
    lens = _lens_t([200, 150])
    a = _decode(q, k, v, lens, out_dtype=torch.float32)
    b = _decode(q, k, v, lens)
    assert b.dtype == torch.bfloat16
    assert torch.equal(a.to(torch.bfloat16), b)


def test_empty_sequence_gives_zeros(built):
    q, k, v = make_dense(2, 4, 4, 128, 64, torch.float32, seed=9)
    out, lse = _decode(q, k, v, _lens_t([0, 64]), return_lse=True)
    assert torch.all(out[0] == 0) and torch.all(torch.isinf(lse[0]))
    want = oracle_decode(q[1:], k[1:], v[1:], [64], 1 / math.sqrt(128))
    assert _maxabs(out[1:].cpu().numpy(), want) <= 1e-5


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_kv_append_and_gather_are_bit_exact(built, dtype):
    from oracle import oracle as O
    from paper_2405_01814_b200 import decode as dec

    B, Hkv, D, P = 3, 4, 128, 32
    lens = [70, 1, 33]
    pt, npages = page_table_for(lens, P, seed=11)
    ptt = torch.tensor(pt, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(0)
    kp = torch.zeros((npages, Hkv, P, D), dtype=dtype, device="cuda")
    vp = torch.zeros_like(kp)
    dense_k = torch.randn((B, Hkv, max(lens), D), generator=g, device="cuda").to(dtype)
    dense_v = torch.randn((B, Hkv, max(lens), D), generator=g, device="cuda").to(dtype)
    for b in range(B):
        dense_k[b, :, lens[b]:] = 0
        dense_v[b, :, lens[b]:] = 0
    # append token by token (all requests at once, positions per request)
    for t in range(max(lens)):
        active = [b for b in range(B) if t < lens[b]]
        pos = torch.tensor([t if b in active else lens[b] - 1 for b in range(B)],
                           dtype=torch.int32, device="cuda")
        kn = torch.stack([dense_k[b, :, min(t, lens[b] - 1)] for b in range(B)])
        vn = torch.stack([dense_v[b, :, min(t, lens[b] - 1)] for b in range(B)])
        dec.kv_append(kn.contiguous(), vn.contiguous(), kp, vp, pos, ptt)
    lens_t = _lens_t(lens)
    gk = dec.kv_gather(kp, ptt, lens_t, max(lens))
    gv = dec.kv_gather(vp, ptt, lens_t, max(lens))
    assert torch.equal(gk, dense_k) and torch.equal(gv, dense_v)
    # the oracle's byte-level paging agrees with the pool the kernel wrote
    rb = D * kp.element_size()
    pool_bytes = kp.view(torch.uint8).cpu().numpy().reshape(npages, Hkv, P, rb)
    dense_bytes = O.page_gather(pool_bytes, pt, np.array(lens, np.int32), max(lens))
    assert np.array_equal(dense_bytes, dense_k.view(torch.uint8).cpu().numpy().reshape(dense_bytes.shape))


def test_dense_append(built):
    from paper_2405_01814_b200 import decode as dec

    k = torch.zeros((2, 3, 16, 64), dtype=torch.bfloat16, device="cuda")
    v = torch.zeros_like(k)
    kn = torch.randn((2, 3, 64), device="cuda").to(torch.bfloat16)
    vn = torch.randn((2, 3, 64), device="cuda").to(torch.bfloat16)
    dec.kv_append(kn, vn, k, v, torch.tensor([5, 15], dtype=torch.int32, device="cuda"))
    assert torch.equal(k[0, :, 5], kn[0]) and torch.equal(k[1, :, 15], kn[1])
    assert torch.equal(v[0, :, 5], vn[0]) and float(k.float().abs().sum() - kn.float().abs().sum()) == 0


def test_validation_errors(built):
    from paper_2405_01814_b200 import _lib
    from paper_2405_01814_b200 import decode as dec

    q, k, v = make_dense(1, 6, 4, 128, 64, torch.bfloat16)
    with pytest.raises(_lib.ValidationError):
        dec.decode(q, k, v, _lens_t([64]))  # 6 % 4 != 0
    q, k, v = make_dense(1, 8, 8, 96, 64, torch.float32)
    with pytest.raises(_lib.ValidationError):
        dec.decode(q, k, v, _lens_t([64]))  # head_dim 96 unsupported on this path
    q, k, v = make_dense(1, 8, 1, 128, 64, torch.bfloat16)
    with pytest.raises(_lib.ValidationError):
        dec.decode(q, k[:, :, :32].contiguous(), v[:, :, :32].contiguous(), _lens_t([64]),
                   max_len=64)  # dense: length exceeds the row capacity


@pytest.mark.slow
@pytest.mark.parametrize("kernel", ["auto", "gqa_tc"])
@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_llama2_70b_layer_subset_parity(built, cfg, kernel):
    """BASELINE configs 3/4 at full size for one layer (paged bf16, GQA 64/8): a seeded
    subset of (request, q head) pairs against the oracle, all heads finite and bounded."""
    B, L = (128, 4096) if cfg == "c3" else (32, 32768)
    Hq, Hkv, D, P = 64, 8, 128, 64
    npages = B * L // P
    g = torch.Generator(device="cuda").manual_seed(3)
    kp = torch.empty((npages, Hkv, P, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g)
    vp = torch.empty_like(kp).uniform_(-1, 1, generator=g)
    q = torch.empty((B, Hq, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g)
    perm = torch.randperm(npages, generator=torch.Generator().manual_seed(5)).to(torch.int32)
    pt = perm.view(B, L // P).cuda()
    lens = _lens_t([L] * B)
    out = _decode(q, kp, vp, lens, page_table=pt, out_dtype=torch.float32, kernel=kernel)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all() and out.abs().max() <= 1.0
    rng = np.random.default_rng(0)
    bs = rng.choice(B, 3, replace=False)
    scale = 1 / math.sqrt(D)
    for b in bs:
        kd = kp[pt[b].long()].permute(1, 0, 2, 3).reshape(1, Hkv, L, D)
        vd = vp[pt[b].long()].permute(1, 0, 2, 3).reshape(1, Hkv, L, D)
        heads = rng.choice(Hq, 4, replace=False)
        want = oracle_decode(q[b:b + 1], kd, vd, [L], scale, pairs=[(0, int(h)) for h in heads])
        for h in heads:
            assert _maxabs(out[b, h].cpu().numpy(), want[0, h]) <= 2e-3


@pytest.mark.parametrize("dtype,G,kernel", [(torch.bfloat16, 8, "auto"), (torch.bfloat16, 1, "auto"),
                                            (torch.float32, 1, "auto"), (torch.bfloat16, 8, "gqa_tc")])
def test_many_splits_combine(built, dtype, G, kernel):
    """More than 32 live splits per head exercises the long combine path."""
    B, Hkv, D, L = 2, 2, 128, 4000
    q, k, v = make_dense(B, Hkv * G, Hkv, D, L, dtype, seed=21)
    lens = [L, 2100]
    scale = 1 / math.sqrt(D)
    want = oracle_decode(q, k, v, lens, scale)
    out = _decode(q, k, v, _lens_t(lens), scale=scale, out_dtype=torch.float32,
                  split_tokens=128 if kernel == "gqa_tc" else 64, kernel=kernel)
    torch.cuda.synchronize()
    assert _maxabs(out.cpu().numpy(), want) <= TOL[dtype]


@pytest.mark.parametrize("G", [1, 8])
def test_packed_qkv_strides(built, G):
    """q / k_new / v_new taken straight out of a packed QKV projection output
    [B, Hq + 2 Hkv, D] (batch strides) give exactly the contiguous results."""
    from paper_2405_01814_b200 import decode as dec

    B, Hkv, D, P, L = 3, 2, 128, 64, 200
    Hq = Hkv * G
    q, k, v = make_dense(B, Hq, Hkv, D, L, torch.bfloat16, seed=31)
    lens = [200, 64, 129]
    pt, npages = page_table_for(lens, P, seed=5)
    ptt = torch.tensor(pt, device="cuda")
    kp, vp = to_paged(k, lens, P, pt, npages, fill=0.0), to_paged(v, lens, P, pt, npages, fill=0.0)
    kp2, vp2 = kp.clone(), vp.clone()
    packed = torch.randn((B, Hq + 2 * Hkv, D), device="cuda").to(torch.bfloat16)
    qv, kv_, vv = packed[:, :Hq], packed[:, Hq:Hq + Hkv], packed[:, Hq + Hkv:]
    pos = torch.tensor([l - 1 for l in lens], dtype=torch.int32, device="cuda")
    dec.kv_append(kv_, vv, kp, vp, pos, ptt)
    dec.kv_append(kv_.contiguous(), vv.contiguous(), kp2, vp2, pos, ptt)
    assert torch.equal(kp, kp2) and torch.equal(vp, vp2)
    a = dec.decode(qv, kp, vp, _lens_t(lens), page_table=ptt, max_len=max(lens))
    b = dec.decode(qv.contiguous(), kp, vp, _lens_t(lens), page_table=ptt, max_len=max(lens))
    assert torch.equal(a, b)


@pytest.mark.parametrize("mode", ["events", "flags", "zero_copy"])
@pytest.mark.parametrize("L", [1, 3, 6])
def test_decode_layers_host_matches_device_path(built, monkeypatch, L, mode):
    """lam_decode_layers_host (host buffers: staged copies synchronised by events or by sequence
    numbers, or zero-copy launches that read q / new rows from and store outputs into the
    pinned host buffers) == append + decode per layer; called twice, so the sequence numbers
    carry across calls."""
    import ctypes as C

    from paper_2405_01814_b200 import _lib
    from paper_2405_01814_b200 import decode as dec

    monkeypatch.setenv("LAM_HOST_FLAGS", "1" if mode == "flags" else "0")
    monkeypatch.setenv("LAM_HOST_ZERO_COPY", "1" if mode == "zero_copy" else "0")
    B, Hq, Hkv, D, P = 4, 16, 2, 128, 64
    lens = [130, 64, 300, 1]
    pt, npages = page_table_for(lens, P, seed=2)
    ptt = torch.tensor(pt, device="cuda")
    lens_t = _lens_t(lens)
    pos = (lens_t - 1).contiguous()
    g = torch.Generator(device="cuda").manual_seed(4)
    pools = [[torch.empty((npages, Hkv, P, D), device="cuda").uniform_(-1, 1, generator=g)
              .to(torch.bfloat16) for _ in range(2)] for _ in range(L)]
    ref_pools = [[t.clone() for t in pl] for pl in pools]
    init_pools = [[t.clone() for t in pl] for pl in pools]
    hq = torch.empty((L, B, Hq, D)).uniform_(-1, 1).to(torch.bfloat16).pin_memory()
    hk = torch.empty((L, B, Hkv, D)).uniform_(-1, 1).to(torch.bfloat16).pin_memory()
    hv = torch.empty((L, B, Hkv, D)).uniform_(-1, 1).to(torch.bfloat16).pin_memory()
    ho = torch.zeros((L, B, Hq, D), dtype=torch.bfloat16).pin_memory()
    dq = torch.empty((B, Hq, D), dtype=torch.bfloat16, device="cuda")
    arr = (dec.DecodeArgs * L)()
    for l in range(L):
        a, _ = dec.make_args(dq, pools[l][0], pools[l][1], lens_t, page_table=ptt, max_len=max(lens),
                             out=torch.empty_like(dq))
        arr[l] = a
    lib = _lib.load()
    stage = torch.empty(int(lib.lam_decode_layers_host_stage_bytes(arr)), dtype=torch.uint8,
                        device="cuda")
    Pt = C.c_void_p * L
    s, xs = torch.cuda.current_stream(), torch.cuda.Stream()
    wants = []
    for l in range(L):
        kp, vp = ref_pools[l]
        dec.kv_append(hk[l].cuda(), hv[l].cuda(), kp, vp, pos, ptt)
        wants.append(dec.decode(hq[l].cuda(), kp, vp, lens_t, page_table=ptt, max_len=max(lens)).cpu())
    for rep in range(2):
        for pl, init in zip(pools, init_pools):
            for t, t0 in zip(pl, init):
                t.copy_(t0)
        ho.zero_()
        torch.cuda.synchronize()
        _lib.check(lib.lam_decode_layers_host(
            _lib.context(0).handle, arr, L, Pt(*[hq[l].data_ptr() for l in range(L)]),
            Pt(*[hk[l].data_ptr() for l in range(L)]), Pt(*[hv[l].data_ptr() for l in range(L)]),
            Pt(*[ho[l].data_ptr() for l in range(L)]), stage.data_ptr(), pos.data_ptr(),
            s.cuda_stream, xs.cuda_stream))
        torch.cuda.synchronize()
        for l in range(L):
            assert torch.equal(ho[l], wants[l]), (rep, l)
            assert torch.equal(pools[l][0], ref_pools[l][0]) and torch.equal(pools[l][1], ref_pools[l][1])
        assert torch.equal(pools[l][0], kp) and torch.equal(pools[l][1], vp)


@pytest.mark.parametrize("dtype,G,paged,kernel", [
    (torch.bfloat16, 8, True, "auto"), (torch.bfloat16, 1, True, "auto"), (torch.float32, 1, False, "auto"),
    (torch.float16, 4, True, "auto"), (torch.float32, 4, True, "auto"), (torch.bfloat16, 8, True, "gqa_tc"),
    (torch.float16, 1, True, "gqa_tc"), (torch.bfloat16, 2, False, "gqa_tc")])
def test_fused_append_equals_append_then_decode(built, dtype, G, paged, kernel):
    """decode(..., k_new, v_new) == kv_append + decode: bitwise outputs and pools, for the
    last tile, split boundaries and single-token requests (new token at seq_lens - 1)."""
    from paper_2405_01814_b200 import decode as dec

    B, Hkv, D = 5, 2, 128
    lens = [1, 64, 65, 300, 129]
    lmax = 320
    q, k, v = make_dense(B, Hkv * G, Hkv, D, lmax, dtype, seed=41 + G)
    kn = torch.randn((B, Hkv, D), device="cuda").to(dtype)
    vn = torch.randn((B, Hkv, D), device="cuda").to(dtype)
    if paged:
        pt, npages = page_table_for(lens, 64, seed=9)
        ptt = torch.tensor(pt, device="cuda")
        kp, vp = to_paged(k, lens, 64, pt, npages, fill=7.0), to_paged(v, lens, 64, pt, npages, fill=7.0)
    else:
        ptt, kp, vp = None, k.clone(), v.clone()
    kp2, vp2 = kp.clone(), vp.clone()
    lt = _lens_t(lens)
    for split in (0, 128 if kernel == "gqa_tc" else 64):
        a = dec.decode(q, kp, vp, lt, page_table=ptt, max_len=max(lens), split_tokens=split,
                       k_new=kn, v_new=vn, out_dtype=torch.float32, kernel=kernel)
        dec.kv_append(kn, vn, kp2, vp2, (lt - 1).contiguous(), ptt)
        b = dec.decode(q, kp2, vp2, lt, page_table=ptt, max_len=max(lens), split_tokens=split,
                       out_dtype=torch.float32, kernel=kernel)
        torch.cuda.synchronize()
        assert torch.equal(a, b), split
        assert torch.equal(kp, kp2) and torch.equal(vp, vp2), split


def test_request_order_is_transparent(built):
    """Longest-first item ordering changes only the schedule, never the result."""
    from paper_2405_01814_b200 import decode as dec

    rng = np.random.default_rng(3)
    lens = rng.integers(1, 2000, 24).tolist()
    B, Hkv, G, D = len(lens), 2, 8, 128
    q, k, v = make_dense(B, Hkv * G, Hkv, D, 2048, torch.bfloat16, seed=13)
    pt, npages = page_table_for(lens, 64, seed=4)
    ptt = torch.tensor(pt, device="cuda")
    kp, vp = to_paged(k, lens, 64, pt, npages), to_paged(v, lens, 64, pt, npages)
    lt = _lens_t(lens)
    for split in (0, 256):
        for kernel in ("auto", "gqa_tc"):
            a = dec.decode(q, kp, vp, lt, page_table=ptt, max_len=max(lens), split_tokens=split,
                           kernel=kernel)
            b = dec.decode(q, kp, vp, lt, page_table=ptt, max_len=max(lens), split_tokens=split,
                           request_order=dec.longest_first(lt), kernel=kernel)
            assert torch.equal(a, b)
    want = oracle_decode(q, k, v, lens, 1 / math.sqrt(D))
    out = dec.decode(q, kp, vp, lt, page_table=ptt, max_len=max(lens), out_dtype=torch.float32,
                     request_order=dec.longest_first(lt))
    assert _maxabs(out.cpu().numpy(), want) <= 2e-3


@pytest.mark.parametrize("kernel,G,dtype", [("simt", 1, torch.bfloat16), ("simt", 1, torch.float32),
                                            ("gqa_mma", 8, torch.bfloat16), ("simt", 4, torch.float16),
                                            ("gqa_tc", 8, torch.bfloat16), ("gqa_tc", 1, torch.float16)])
@pytest.mark.parametrize("tail,splits", [(1, 2), (3, 4), (100, 3)])
def test_split_tail_vs_oracle(built, monkeypatch, kernel, G, dtype, tail, splits):
    """Split tail: the last `tail` units run as `splits` short items merged in split order, the
    others whole (LAM_TAIL_UNITS / LAM_TAIL_SPLITS)."""
    monkeypatch.setenv("LAM_TAIL_UNITS", str(tail))
    monkeypatch.setenv("LAM_TAIL_SPLITS", str(splits))
    B, Hkv, D = 5, 2, 128
    Hq = Hkv * G
    lens = [1, 700, 0, 333, 1024]
    q, k, v = make_dense(B, Hq, Hkv, D, 1024, dtype, seed=tail * 7 + splits)
    scale = 1 / math.sqrt(D)
    want, want_lse = oracle_decode(q, k, v, lens, scale, want_lse=True)
    P = 64
    pt, npages = page_table_for(lens, P, seed=splits)
    kp, vp = to_paged(k, lens, P, pt, npages), to_paged(v, lens, P, pt, npages)
    out, lse = _decode(q, kp, vp, _lens_t(lens), page_table=torch.tensor(pt, device="cuda"),
                       max_len=max(lens), scale=scale, out_dtype=torch.float32, return_lse=True,
                       kernel=kernel)
    torch.cuda.synchronize()
    assert _maxabs(out.cpu().numpy(), want) <= TOL[dtype]
    finite = np.isfinite(want_lse)
    assert _maxabs(lse.cpu().numpy()[finite], want_lse[finite]) <= 1e-3


@pytest.mark.parametrize("kernel,dtype,G", [("gqa_mma", torch.bfloat16, 8), ("gqa_mma", torch.bfloat16, 1),
                                            ("simt", torch.float32, 1), ("simt", torch.bfloat16, 2),
                                            ("gqa_tc", torch.bfloat16, 8), ("gqa_tc", torch.bfloat16, 1)])
@pytest.mark.parametrize("lmax", [40, 300, 3000])
def test_overlap_prev_orders_inputs_after_preceding_kernel(built, kernel, dtype, G, lmax):
    """overlap_prev (programmatic dependent launch): a chain of launches over different pools
    where each launch's q and fused new K/V rows are the PRECEDING launch's output — so they
    must be read only after it completes — equals the same chain with ordinary stream order,
    bitwise.  Covers first items shorter than the ring (all inputs deferred to the end of the
    item) and longer ones (deferred at the ring boundary)."""
    from paper_2405_01814_b200 import decode as dec

    B, Hkv, D, P, L = 24, 4, 128, 64, 6
    Hq = Hkv * G
    g = torch.Generator(device="cuda").manual_seed(3)
    lens = torch.randint(1, lmax, (B,), generator=g, device="cuda", dtype=torch.int32)
    lens[0] = lmax
    npg = (lmax + P - 1) // P
    pools = [(torch.empty((B * npg, Hkv, P, D), device="cuda").uniform_(-1, 1, generator=g).to(dtype),
              torch.empty((B * npg, Hkv, P, D), device="cuda").uniform_(-1, 1, generator=g).to(dtype))
             for _ in range(L)]
    pt = torch.randperm(B * npg, generator=g, device="cuda").to(torch.int32).view(B, npg)
    q0 = torch.empty((B, Hq, D), device="cuda").uniform_(-1, 1, generator=g).to(dtype)

    def chain(overlap):
        kv = [(k.clone(), v.clone()) for k, v in pools]
        outs, q = [], q0
        for layer in range(L):
            out = torch.empty((B, Hq, D), dtype=dtype, device="cuda")
            dec.decode(q, kv[layer][0], kv[layer][1], lens, page_table=pt, max_len=lmax, out=out,
                       kernel=kernel, k_new=q[:, :Hkv], v_new=q[:, Hkv - 1: 2 * Hkv - 1]
                       if Hq >= 2 * Hkv else q[:, :Hkv], overlap_prev=overlap and layer > 0)
            outs.append(out)
            q = out
        torch.cuda.synchronize()
        return outs, kv

    want, kv_want = chain(False)
    for _ in range(3):
        got, kv_got = chain(True)
        for layer in range(L):
            assert torch.equal(got[layer], want[layer]), layer
            assert torch.equal(kv_got[layer][0], kv_want[layer][0])
            assert torch.equal(kv_got[layer][1], kv_want[layer][1])


@pytest.mark.parametrize("name,B,Hq,Hkv,L,dtype,paged,want", [
    # (kernel, splits, CTAs) the planner picks for the BASELINE launch shapes, measured best on
    # B200 (profiles/r01b/SUMMARY.md §2, §7): C4 split 4 ways, the 512-unit sharded GQA launch
    # unsplit on 128 CTAs (2 even rounds), the rest unsplit on the full grid — C1 too since its
    # 64-token fp32 tiles (profiles/r02/final3/c1_simt_variants.txt).
    ("c1", 8, 32, 32, 1024, torch.float32, False, ("simt", 1, 148)),
    ("c2", 64, 32, 32, 4096, torch.bfloat16, True, ("gqa_tc", 1, 148)),
    ("c3", 128, 64, 8, 4096, torch.bfloat16, True, ("gqa_tc", 1, 148)),
    ("c4", 32, 64, 8, 32768, torch.bfloat16, True, ("gqa_tc", 4, 148)),
    ("c3n8", 512, 8, 1, 4096, torch.bfloat16, True, ("gqa_tc", 1, 128)),
])
def test_planner_choices_for_baseline_shapes(built, name, B, Hq, Hkv, L, dtype, paged, want):
    from paper_2405_01814_b200 import decode as dec

    if torch.cuda.get_device_properties(0).multi_processor_count != 148:
        pytest.skip("choices are pinned for the 148-SM B200")
    D, P = 128, 64
    q = torch.empty((B, Hq, D), dtype=dtype, device="cuda")
    lens = torch.full((B,), L, dtype=torch.int32, device="cuda")
    if paged:
        npg = B * L // P
        pool = torch.empty((npg, Hkv, P, D), dtype=dtype, device="cuda")
        pt = torch.zeros((B, L // P), dtype=torch.int32, device="cuda")
        kw = dict(page_table=pt, max_len=L)
    else:
        pool = torch.empty((B, Hkv, L, D), dtype=dtype, device="cuda")
        kw = dict(max_len=L)
    kern, splits, _ = dec.plan(q, pool, pool, lens, **kw)
    ctas = dec.plan_grid(q, pool, pool, lens, **kw)
    assert (kern, splits, ctas) == want


def _request_kv(pool, pt, b, kvh, ln, P):
    pages = pt[b, : -(-ln // P)].long()
    return pool[pages, kvh].reshape(-1, pool.shape[-1])[:ln]


@pytest.mark.slow
def test_c2_full_shape_overlap_chain_vs_oracle(built):
    """BASELINE config 2 exactly as the bench launches it — B=64, l=4096, 32/32 heads, bf16,
    paged P=64, the tensor-core kernel at G=1, fused append, overlap_prev — as a chain of three
    layers where each layer's q and new K/V rows are the previous layer's output (so the
    programmatic-dependent-launch ordering is load-bearing), against the oracle on seeded
    (request, head) pairs of every layer; appends bit-exact."""
    from paper_2405_01814_b200 import decode as dec

    B, H, D, L, P, layers = 64, 32, 128, 4096, 64, 3
    npg = B * L // P
    g = torch.Generator(device="cuda").manual_seed(12)
    perm = torch.randperm(npg, generator=torch.Generator().manual_seed(2)).to(torch.int32)
    pt = perm.view(B, L // P).cuda()
    lens = _lens_t([L] * B)
    pools = [(torch.empty((npg, H, P, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g),
              torch.empty((npg, H, P, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g))
             for _ in range(layers)]
    x0 = torch.empty((B, 3 * H, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g)
    kern, splits, _ = dec.plan(x0[:, :H], pools[0][0], pools[0][1], lens, page_table=pt, max_len=L)
    assert kern == "gqa_tc" and splits == 1  # the bench's C2 launch
    # layer 0 reads packed QKV rows; layer l > 0 reads q = k_new = v_new = layer l-1's output,
    # straight from the launch before it (no kernel in between)
    ins = [(x0[:, :H], x0[:, H:2 * H], x0[:, 2 * H:])]
    outs = []
    for layer in range(layers):
        q, kn, vn = ins[layer]
        o = dec.decode(q, pools[layer][0], pools[layer][1], lens, page_table=pt, max_len=L,
                       k_new=kn, v_new=vn, overlap_prev=layer > 0)
        outs.append(o)
        ins.append((o, o, o))
    torch.cuda.synchronize()
    rng = np.random.default_rng(4)
    ptc = pt
    for layer in range(layers):
        kp, vp = pools[layer]
        for _ in range(4):
            b, h = int(rng.integers(B)), int(rng.integers(H))
            kd = _request_kv(kp, ptc, b, h, L, P)
            vd = _request_kv(vp, ptc, b, h, L, P)
            q, kn, vn = ins[layer]
            assert torch.equal(kd[L - 1], kn[b, h]) and torch.equal(vd[L - 1], vn[b, h])
            want = oracle_decode(q[b:b + 1, h:h + 1], kd[None, None], vd[None, None], [L], 1 / math.sqrt(D))
            got = outs[layer][b, h].float().cpu().numpy()
            assert _maxabs(got, want[0, 0]) <= 2e-3 + 2.0 ** -9, (layer, b, h)


@pytest.mark.slow
def test_c5_full_shape_request_order_vs_oracle(built):
    """BASELINE config 5's launch as the bench runs it (one micro-batch launch of the global
    B=256 batch's first half is what the engine issues; here the whole batch in one launch):
    LLaMA-2-70B GQA 64/8, bf16, log-uniform lengths on [128, 16384] (mt-seeded), paged,
    fused append and longest-first request_order, against the oracle on seeded pairs that
    include the longest and the shortest request."""
    from paper_2405_01814_b200 import decode as dec

    B, Hq, Hkv, D, P = 256, 64, 8, 128, 64
    r = np.random.default_rng(2024)
    lens = np.exp(r.uniform(math.log(128), math.log(16384), B)).astype(np.int32)
    pt_np, npages = page_table_for(lens, P, seed=8)
    pt = torch.tensor(pt_np, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(5)
    kp = torch.empty((npages, Hkv, P, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g)
    vp = torch.empty_like(kp).uniform_(-1, 1, generator=g)
    x = torch.empty((B, Hq + 2 * Hkv, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g)
    lt = _lens_t(lens)
    out = dec.decode(x[:, :Hq], kp, vp, lt, page_table=pt, max_len=int(lens.max()),
                     k_new=x[:, Hq:Hq + Hkv], v_new=x[:, Hq + Hkv:], out_dtype=torch.float32,
                     request_order=dec.longest_first(lt))
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    rng = np.random.default_rng(6)
    bs = [int(np.argmax(lens)), int(np.argmin(lens))] + [int(b) for b in rng.choice(B, 6, replace=False)]
    for b in bs:
        ln = int(lens[b])
        kvh = int(rng.integers(Hkv))
        kd = _request_kv(kp, pt, b, kvh, ln, P)
        vd = _request_kv(vp, pt, b, kvh, ln, P)
        assert torch.equal(kd[ln - 1], x[b, Hq + kvh]) and torch.equal(vd[ln - 1], x[b, Hq + Hkv + kvh])
        heads = list(range(kvh * 8, kvh * 8 + 8))
        want = oracle_decode(x[b:b + 1, heads], kd[None, None], vd[None, None], [ln],
                             1 / math.sqrt(D))  # 8 q heads on one KV head (G = 8)
        assert _maxabs(out[b, heads].cpu().numpy(), want[0]) <= 2e-3, b
