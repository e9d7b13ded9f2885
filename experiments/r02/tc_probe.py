"""Probe of the tcgen05 GQA kernel: small parity cases vs the oracle, then a same-process
timing A/B against the mma.sync kernel on a C3-shaped layer (B=128, 64/8 heads, l=4096)."""
import math
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2405_01814_b200 import decode as dec  # noqa: E402
from tests.helpers import make_dense, oracle_decode, page_table_for, to_paged  # noqa: E402


def case(G, lens, paged, dtype=torch.bfloat16, split=0, fused=False):
    B, Hkv, D = len(lens), 2, 128
    lmax = max(64, -(-max(lens) // 64) * 64)
    q, k, v = make_dense(B, Hkv * G, Hkv, D, lmax, dtype, seed=G + len(lens))
    for b, l in enumerate(lens):
        k[b, :, l:] = float("nan")
        v[b, :, l:] = float("nan")
    scale = 1 / math.sqrt(D)
    kw = {}
    if fused:
        kn = torch.randn((B, Hkv, D), device="cuda").to(dtype)
        vn = torch.randn((B, Hkv, D), device="cuda").to(dtype)
        for b, l in enumerate(lens):
            k[b, :, l - 1] = kn[b]
            v[b, :, l - 1] = vn[b]
        kw = dict(k_new=kn, v_new=vn)
    want = oracle_decode(q, k, v, lens, scale)
    if paged:
        pt, npg = page_table_for(lens, 64, seed=G)
        kp, vp = to_paged(k, lens, 64, pt, npg), to_paged(v, lens, 64, pt, npg)
        if fused:  # stale rows where the new token goes
            for b, l in enumerate(lens):
                kp[int(pt[b, (l - 1) // 64]), :, (l - 1) % 64] = float("nan")
        ptt = torch.tensor(pt, device="cuda")
    else:
        kp, vp, ptt = k.clone(), v.clone(), None
    out = dec.decode(q, kp, vp, torch.tensor(lens, dtype=torch.int32, device="cuda"), page_table=ptt,
                     max_len=max(lens), scale=scale, out_dtype=torch.float32, kernel="gqa_tc",
                     split_tokens=split, **kw)
    torch.cuda.synchronize()
    err = float(np.abs(out.cpu().numpy() - want).max())
    print(f"G={G} lens={lens[:4]}.. paged={paged} split={split} fused={fused}: max-abs {err:.2e}",
          "OK" if err <= 2e-3 else "FAIL", flush=True)
    return err <= 2e-3


ok = True
if len(sys.argv) > 1 and sys.argv[1] == "parity":
    for fn in (lambda: case(8, [1, 77, 300], True), lambda: case(8, [300], True), lambda: case(8, [128], True),
               lambda: case(8, [256], True), lambda: case(1, [64], False), lambda: case(8, [1], True)):
        fn()
    sys.exit(0)
ok &= case(8, [1, 77, 300], True)
ok &= case(8, [128, 129, 64, 500], True)
ok &= case(1, [1, 77, 300], False)
ok &= case(4, [1000, 33, 256], True, split=128)
ok &= case(8, [1, 64, 65, 300, 129], True, fused=True)
ok &= case(2, [0, 300, 17], True)
print("parity", "OK" if ok else "FAIL", flush=True)
if not ok:
    sys.exit(1)

# timing A/B: C3-shaped layer, paged, shuffled pages
B, Hq, Hkv, D, L, P = 128, 64, 8, 128, 4096, 64
npg = B * L // P
sets = 4
g = torch.Generator(device="cuda").manual_seed(0)
pools = [(torch.empty((npg, Hkv, P, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g),
          torch.empty((npg, Hkv, P, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g))
         for _ in range(sets)]
pt = torch.randperm(npg, generator=torch.Generator().manual_seed(1)).to(torch.int32).view(B, L // P).cuda()
q = torch.empty((B, Hq, D), dtype=torch.bfloat16, device="cuda").uniform_(-1, 1, generator=g)
lens = torch.full((B,), L, dtype=torch.int32, device="cuda")
outs = {}
for kern in ("gqa_mma", "gqa_tc", "gqa_mma", "gqa_tc"):
    for i in range(3):
        dec.decode(q, *pools[i % sets], lens, page_table=pt, max_len=L, kernel=kern)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 40
    e0.record()
    for i in range(n):
        o = dec.decode(q, *pools[i % sets], lens, page_table=pt, max_len=L, kernel=kern, overlap_prev=i > 0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    outs[kern] = dec.decode(q, *pools[0], lens, page_table=pt, max_len=L, kernel=kern, out_dtype=torch.float32)
    print(f"{kern}: {ms*1e3:.1f} us per layer, {2 * B * L * Hkv * D * 2 / ms / 1e6:.0f} GB/s", flush=True)
torch.cuda.synchronize()
print("tc vs mma max-abs", float((outs["gqa_tc"] - outs["gqa_mma"]).abs().max()))
