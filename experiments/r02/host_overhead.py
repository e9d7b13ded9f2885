"""Host cost of one lam_decode call on the C1 shape (dense fp32 MHA, B=8, 32 heads, l=1024):
host enqueue time per call against GPU time per launch (diagnostic for the C1 step)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2405_01814_b200 import _lib, decode as dec  # noqa: E402

B, H, D, L = 8, 32, 128, 1024
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
sets = [(torch.empty((B, H, L, D), device=dev).uniform_(-1, 1, generator=g),
         torch.empty((B, H, L, D), device=dev).uniform_(-1, 1, generator=g)) for _ in range(4)]
q = torch.empty((B, H, D), device=dev).uniform_(-1, 1, generator=g)
kn = torch.empty((B, H, D), device=dev).uniform_(-1, 1, generator=g)
vn = torch.empty((B, H, D), device=dev).uniform_(-1, 1, generator=g)
out = torch.empty((B, H, D), device=dev)
lens = torch.full((B,), L, dtype=torch.int32, device=dev)
ctx = _lib.context(0)
lib = _lib.load()
args = [dec.make_args(q, k, v, lens, max_len=L, out=out, k_new=kn, v_new=vn)[0] for k, v in sets]
s = torch.cuda.current_stream().cuda_stream
for rep in range(3):
    for i in range(20):
        _lib.check(lib.lam_decode(ctx.handle, args[i % 4], s))
    torch.cuda.synchronize()
    n = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for i in range(n):
        lib.lam_decode(ctx.handle, args[i % 4], s)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    gpu = e0.elapsed_time(e1) * 1e3 / n
    host = (t1 - t0) * 1e6 / n
    # host cost alone: the same calls while the GPU is busy with a long queue already
    print(f"rep {rep}: host enqueue {host:.1f} us/call, GPU {gpu:.1f} us/launch "
          f"({B * H * L * D * 4 * 2 / gpu / 1e3:.0f} GB/s)", flush=True)
    # CUDA graph of 20 launches
    gs = torch.cuda.Stream()
    gs.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(gs):
        graph.capture_begin()
        for i in range(20):
            lib.lam_decode(ctx.handle, args[i % 4], gs.cuda_stream)
        graph.capture_end()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"   graph: {e0.elapsed_time(e1) * 1e3 / 200:.1f} us/launch", flush=True)
