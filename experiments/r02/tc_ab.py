"""A/B of the decode kernels on a C3-shaped layer (B=128, 64/8 heads, l=4096, paged, rotating
pools so the KV never sits in L2).  Prints us/layer and GB/s per configuration (env vars are
read per process, so each configuration runs in its own process)."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2405_01814_b200 import decode as dec  # noqa: E402

kern = sys.argv[1]
B, Hq, Hkv, D, L, P = [int(x) for x in (sys.argv[2:8] if len(sys.argv) > 2 else (128, 64, 8, 128, 4096, 64))]
npg = B * L // P
sets = max(2, -(-2 * 2**30 // (2 * npg * Hkv * P * D * 2)))
g = torch.Generator(device="cuda").manual_seed(0)
pools = [(torch.empty((npg, Hkv, P, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g),
          torch.empty((npg, Hkv, P, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g))
         for _ in range(sets)]
pt = torch.randperm(npg, generator=torch.Generator().manual_seed(1)).to(torch.int32).view(B, L // P).cuda()
q = torch.empty((B, Hq, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g)
lens = torch.full((B,), L, dtype=torch.int32, device="cuda")
split = int(os.environ.get("AB_SPLIT", 0))
for rep in range(2):
    for i in range(3):
        dec.decode(q, *pools[i % sets], lens, page_table=pt, max_len=L, kernel=kern, split_tokens=split)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 60
    e0.record()
    for i in range(n):
        dec.decode(q, *pools[i % sets], lens, page_table=pt, max_len=L, kernel=kern, split_tokens=split,
                   overlap_prev=i > 0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{kern} {os.environ.get('LAM_DECODE_FLAGS', '0')} st={os.environ.get('LAM_TC_STAGES', '3')} "
          f"B={B} Hq={Hq} Hkv={Hkv} L={L} split={split}: {ms*1e3:.1f} us, "
          f"{2 * B * L * Hkv * D * 2 / ms / 1e6:.0f} GB/s", flush=True)
