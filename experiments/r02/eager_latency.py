"""Eager q (§8(f) row 1): per-layer latency of one C3-shaped decode launch (B=128, 64/8 heads,
l=4096, bf16, paged, peer io with one local source) when the model worker's K/V projection
takes X us after q: the fused protocol publishes q, K and V together after X; the eager protocol
publishes q at once and K/V after X.  Latency = model-worker start -> outputs published."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2405_01814_b200 import _lib, decode as dec  # noqa: E402
from paper_2405_01814_b200.kvcache import PagedKVCache  # noqa: E402

B, Hq, Hkv, D, L, P = 128, 64, 8, 128, 4096, 64
W = Hq + 2 * Hkv
cache = PagedKVCache(1, Hkv, D, P, B * L // P, B, L // P, dtype=torch.bfloat16,
                     device=torch.device("cuda"), shuffle_seed=1)
cache.set_lengths([L] * B)
cache.sync()
cache.fill_random(torch.Generator(device="cuda").manual_seed(0))
qkv = torch.empty((B, W, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
out = torch.empty((B, Hq, D), dtype=torch.bfloat16, device="cuda")
flags = torch.zeros(3, dtype=torch.int32, device="cuda")  # q, kv, done
a, _ = dec.make_args(out, cache.k[0], cache.v[0], cache.seq_lens, page_table=cache.page_table,
                     max_len=L, out=out)
a.q_batch_stride = a.new_batch_stride = W * D
lib, ctx = _lib.load(), _lib.context(0)
model = torch.cuda.Stream()
fp = flags.data_ptr()
one = lambda x: (C.c_void_p * 1)(x)  # noqa: E731


def run(eager, x_us, seq):
    io = _lib.PeerIO()
    io.n_src, io.rows_per_src = 1, B
    io.q_src[0], io.out_dst[0] = qkv.data_ptr(), out.data_ptr()
    io.k_new_offset, io.v_new_offset = Hq * D, (Hq + Hkv) * D
    io.n_wait = io.n_done = 1
    io.wait_value = io.done_value = seq
    io.wait_flags[0], io.done_flags[0] = fp, fp + 8
    if eager:
        io.n_wait_kv, io.kv_wait_value, io.kv_wait_flags[0] = 1, seq, fp + 4
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _lib.check(lib.lam_decode_peer(ctx.handle, a, io, torch.cuda.current_stream().cuda_stream))
    t0.record(model)
    if eager:
        _lib.check(lib.lam_stream_signal(ctx.handle, one(fp), 1, seq, model.cuda_stream))
    with torch.cuda.stream(model):  # the K/V projection (on the model stream)
        torch.cuda._sleep(int(x_us * 1e-6 * 1.9e9))
    _lib.check(lib.lam_stream_signal(ctx.handle, one(fp + 4), 1, seq, model.cuda_stream))
    if not eager:
        _lib.check(lib.lam_stream_signal(ctx.handle, one(fp), 1, seq, model.cuda_stream))
    _lib.check(lib.lam_stream_wait(ctx.handle, one(fp + 8), 1, seq, model.cuda_stream))
    t1.record(model)
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) * 1e3


seq = 0
for x in (0, 50, 100, 200):
    res = {}
    for eager in (False, True):
        vals = []
        for rep in range(6):
            seq += 1
            vals.append(run(eager, x, seq))
        res[eager] = sorted(vals)[len(vals) // 2]
    print(f"K/V projection {x:4d} us: fused {res[False]:7.1f} us, eager q {res[True]:7.1f} us, "
          f"gain {res[False] - res[True]:6.1f} us", flush=True)
print("status", ctx.status())
