"""Small cases of every shipped decode path, for compute-sanitizer (memcheck / synccheck):
tcgen05, mma.sync and SIMT kernels, paged and dense, fused append, splits, ragged lengths,
request order, an overlap_prev chain (programmatic dependent launch) and a step launch."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2405_01814_b200 import decode as dec  # noqa: E402
from tests.helpers import make_dense, oracle_decode, page_table_for, to_paged  # noqa: E402

worst = 0.0
for kernel, G, dtype in (("gqa_tc", 8, torch.bfloat16), ("gqa_tc", 1, torch.bfloat16),
                         ("gqa_mma", 8, torch.bfloat16), ("simt", 1, torch.float32),
                         ("simt", 2, torch.float16)):
    B, Hkv, D = 3, 2, 128
    lens = [1, 77, 300]
    q, k, v = make_dense(B, Hkv * G, Hkv, D, 320, dtype, seed=G)
    pt, npg = page_table_for(lens, 64, seed=1)
    kp, vp = to_paged(k, lens, 64, pt, npg, fill=0.0), to_paged(v, lens, 64, pt, npg, fill=0.0)
    ptt = torch.tensor(pt, device="cuda")
    lt = torch.tensor(lens, dtype=torch.int32, device="cuda")
    kn = torch.randn((B, Hkv, D), device="cuda").to(dtype)
    for split in (0, 128):
        out = dec.decode(q, kp, vp, lt, page_table=ptt, max_len=max(lens), kernel=kernel,
                         split_tokens=split, k_new=kn, v_new=kn, out_dtype=torch.float32,
                         request_order=dec.longest_first(lt))
        out2 = dec.decode(q, k, v, lt, max_len=max(lens), kernel=kernel, split_tokens=split,
                          out_dtype=torch.float32)
    torch.cuda.synchronize()
    want = oracle_decode(q, k, v, lens, 1 / math.sqrt(D))
    worst = max(worst, float(np.abs(out2.cpu().numpy() - want).max()))
# overlap_prev chain
B, Hkv, G, D, P = 8, 2, 8, 128, 64
g = torch.Generator(device="cuda").manual_seed(3)
lens = torch.randint(1, 300, (B,), generator=g, device="cuda", dtype=torch.int32)
pools = [(torch.empty((B * 5, Hkv, P, D), device="cuda").uniform_(-1, 1, generator=g).to(torch.bfloat16),
          torch.empty((B * 5, Hkv, P, D), device="cuda").uniform_(-1, 1, generator=g).to(torch.bfloat16))
         for _ in range(3)]
pt = torch.randperm(B * 5, generator=g, device="cuda").to(torch.int32).view(B, 5)
x = torch.empty((B, Hkv * G, D), device="cuda").uniform_(-1, 1, generator=g).to(torch.bfloat16)
for layer in range(3):
    x = dec.decode(x, pools[layer][0], pools[layer][1], lens, page_table=pt, max_len=300,
                   k_new=x[:, :Hkv], v_new=x[:, :Hkv], overlap_prev=layer > 0)
# step launch (local, two micro-batches, fused append, splits)
from paper_2405_01814_b200.kvcache import PagedKVCache  # noqa: E402

L, B = 3, 6
cache = PagedKVCache(L, Hkv, D, P, 40, B, 6, dtype=torch.bfloat16, device=torch.device("cuda"),
                     shuffle_seed=2)
cache.set_lengths([1, 100, 300, 64, 129, 7])
cache.sync()
cache.fill_random(g)
xs = torch.empty((L, B, Hkv * G + 2 * Hkv, D), device="cuda").uniform_(-1, 1, generator=g).to(torch.bfloat16)
for split in (0, 128):
    dec.decode_step(xs[:, :, :Hkv * G], cache.k, cache.v, cache.seq_lens, n_mb=2,
                    page_table=cache.page_table, max_len=300, k_new=xs[:, :, Hkv * G:Hkv * G + Hkv],
                    v_new=xs[:, :, Hkv * G + Hkv:], split_tokens=split)
torch.cuda.synchronize()
print("sanitize cases done, worst max-abs vs oracle", worst)
