import ctypes as C, sys
import torch
sys.path.insert(0, ".")
from tests.test_step_gpu import _problem, _reference
from paper_2405_01814_b200 import _lib, decode as dec
kernel = sys.argv[1] if len(sys.argv) > 1 else "auto"
L, MB, n_src, Bh, Hq, Hkv, D = 3, 2, 2, 3, 16, 2, 128
rows = n_src * Bh
cache, lens, x, order = _problem(L, MB, rows, Hq, Hkv, seed=5)
W = Hq + 2 * Hkv
want, k_want, v_want = _reference(cache, lens, x, order, L, MB, rows, Hq, Hkv, kernel)
xs = x.view(L, MB, n_src, Bh, W, D)
qkv = [xs[:, :, s].contiguous() for s in range(n_src)]
outs = [torch.zeros((L, MB, Bh, Hq, D), dtype=torch.bfloat16, device="cuda") for _ in range(n_src)]
flags = torch.zeros((2, MB, n_src), dtype=torch.int32, device="cuda")
qd = torch.empty((MB * rows, Hq, D), dtype=torch.bfloat16, device="cuda")
a, _ = dec.make_args(qd, cache.k[0], cache.v[0], cache.seq_lens, page_table=cache.page_table,
                     max_len=int(lens.max()), out=qd, kernel=kernel)
a.q_batch_stride = a.new_batch_stride = W * D
a.request_order = order.data_ptr()
io = _lib.PeerIO()
io.n_src, io.rows_per_src = n_src, Bh
for s in range(n_src):
    io.q_src[s] = qkv[s].data_ptr()
    io.out_dst[s] = outs[s].data_ptr()
io.k_new_offset, io.v_new_offset = Hq * D, (Hq + Hkv) * D
io.n_wait = io.n_done = n_src
fp = flags.data_ptr()
for s in range(n_src):
    io.wait_flags[s] = fp + 4 * s
    io.done_flags[s] = fp + 4 * (MB * n_src + s)
epoch = 100
st = dec.step_layout(L, MB, rows, pool_layer_rows=cache.k[0].numel() // D, lm_q_stride=Bh * W * D,
                     lm_out_stride=Bh * Hq * D, flag_mb_stride=n_src, epoch=epoch)
lib = _lib.load()
ctx = _lib.Context(0)
ctx.set_spin_timeout(300_000_000)
mode = sys.argv[2] if len(sys.argv) > 2 else "after"
P = C.c_void_p * n_src
if mode == "before":  # publish everything first, no dependency
    for layer in range(L):
        for m in range(MB):
            flags[0, m] = epoch + L
model = torch.cuda.Stream()
dummy = torch.zeros(1, dtype=torch.int32, device="cuda")
if mode == "after":  # warm the stream memory ops up before the kernel occupies the GPU
    _lib.check(lib.lam_stream_signal(ctx.handle, (C.c_void_p * 1)(dummy.data_ptr()), 1, 1, model.cuda_stream))
    _lib.check(lib.lam_stream_wait(ctx.handle, (C.c_void_p * 1)(dummy.data_ptr()), 1, 1, model.cuda_stream))
torch.cuda.synchronize()
_lib.check(lib.lam_decode_step(ctx.handle, a, st, io, torch.cuda.current_stream().cuda_stream))
if mode == "host":  # relay through host copies on a side stream (no stream memory ops)
    side = torch.cuda.Stream()
    import time
    t0 = time.time()
    for layer in range(L):
        for m in range(MB):
            if layer > 0:
                while True:
                    with torch.cuda.stream(side):
                        d = flags[1, m].cpu()
                    if int(d.min()) >= epoch + layer:
                        break
            with torch.cuda.stream(side):
                flags[0, m].fill_(epoch + layer + 1)
            side.synchronize()
    print("host relay done in", time.time() - t0)
if mode in ("after", "cold"):
    for layer in range(L):
        for m in range(MB):
            if layer > 0:
                done = P(*[fp + 4 * ((MB + m) * n_src + s) for s in range(n_src)])
                _lib.check(lib.lam_stream_wait(ctx.handle, done, n_src, epoch + layer, model.cuda_stream))
            ready = P(*[fp + 4 * (m * n_src + s) for s in range(n_src)])
            _lib.check(lib.lam_stream_signal(ctx.handle, ready, n_src, epoch + layer + 1, model.cuda_stream))
torch.cuda.synchronize()
print(kernel, mode, "status", ctx.status(), "flags", flags.tolist())
got = torch.stack(outs, 2).view(L, MB * rows, Hq, D)
for layer in range(L):
    for m in range(MB):
        sl = slice(m * rows, (m + 1) * rows)
        print(layer, m, "equal", torch.equal(got[layer, sl], want[layer, sl]), float((got[layer, sl].float() - want[layer, sl].float()).abs().max()))
