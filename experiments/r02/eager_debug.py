import ctypes as C, sys, time
import torch
sys.path.insert(0, ".")
from tests.test_peer_gpu import _setup, _reference, _peer_io
from paper_2405_01814_b200 import _lib, decode as dec
for G, kern in ((8, "auto"), (8, "gqa_mma"), (1, "simt")):
    n_src, Bh, Hkv, D = 2, 3, 2, 128
    Hq = Hkv * G
    cache, lens, qkv, s = _setup(n_src=n_src, Bh=Bh, Hq=Hq, Hkv=Hkv, D=D, seed=31 + G)
    W = s["W"]
    outs = [torch.zeros((Bh, Hq, D), dtype=torch.bfloat16, device="cuda") for _ in range(n_src)]
    flags = torch.zeros(3 * n_src, dtype=torch.int32, device="cuda")
    qd = torch.empty((n_src * Bh, Hq, D), dtype=torch.bfloat16, device="cuda")
    a, _ = dec.make_args(qd, cache.k[0], cache.v[0], cache.seq_lens, page_table=cache.page_table,
                         max_len=int(lens.max()), out=qd, kernel=kern)
    a.q_batch_stride = a.new_batch_stride = W * D
    io = _peer_io(n_src, Bh, Hq, Hkv, D, qkv, outs)
    fp = flags.data_ptr()
    io.n_wait = io.n_done = io.n_wait_kv = n_src
    io.wait_value = io.done_value = io.kv_wait_value = 5
    for i in range(n_src):
        io.wait_flags[i] = fp + 4 * i
        io.kv_wait_flags[i] = fp + 4 * (n_src + i)
        io.done_flags[i] = fp + 4 * (2 * n_src + i)
    print("io fields", io.n_wait_kv, io.kv_wait_value, io.kv_wait_flags[0], fp + 4 * n_src, C.sizeof(_lib.PeerIO))
    lib, ctx = _lib.load(), _lib.Context(0)
    side = torch.cuda.Stream()
    P = C.c_void_p * n_src
    torch.cuda.synchronize()
    t0 = time.time()
    _lib.check(lib.lam_decode_peer(ctx.handle, a, io, torch.cuda.current_stream().cuda_stream))
    _lib.check(lib.lam_stream_signal(ctx.handle, P(*[fp + 4 * i for i in range(n_src)]), n_src, 5, side.cuda_stream))
    side.synchronize()
    for k in range(5):
        time.sleep(0.01)
        with torch.cuda.stream(side):
            f = flags.cpu().tolist()
        print(G, kern, f"{time.time()-t0:.3f}s", f)
    _lib.check(lib.lam_stream_signal(ctx.handle, P(*[fp + 4 * (n_src + i) for i in range(n_src)]), n_src, 5, side.cuda_stream))
    torch.cuda.synchronize()
    print("final", flags.tolist(), "status", ctx.status())
    ctx.close()
