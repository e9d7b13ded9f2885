"""Tuning sweep for one decode layer: time lam_decode for several split sizes / variants.

    python scripts/exp_decode.py --cfg c3 --splits 0,512,1024,2048 [--iters 20]

Rotates over enough distinct KV buffers that no launch hits L2.  Prints one line per variant.
"""
import argparse
import math
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_01814_b200 import decode as dec  # noqa: E402

CFG = {
    "c1": dict(B=8, Hq=32, Hkv=32, L=1024, dtype=torch.float32, paged=False),
    "c2": dict(B=64, Hq=32, Hkv=32, L=4096, dtype=torch.bfloat16, paged=True),
    "c3": dict(B=128, Hq=64, Hkv=8, L=4096, dtype=torch.bfloat16, paged=True),
    "c3n8": dict(B=512, Hq=8, Hkv=1, L=4096, dtype=torch.bfloat16, paged=True),
    "c4": dict(B=32, Hq=64, Hkv=8, L=32768, dtype=torch.bfloat16, paged=True),
    "c4n8": dict(B=128, Hq=8, Hkv=1, L=32768, dtype=torch.bfloat16, paged=True),
    "c5": dict(B=256, Hq=64, Hkv=8, L=16384, dtype=torch.bfloat16, paged=True, mixed=True),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="c3")
    ap.add_argument("--splits", default="0")
    ap.add_argument("--kernels", default="auto")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warm", type=int, default=5)
    ap.add_argument("--P", type=int, default=64)
    ap.add_argument("--no-order", action="store_true")
    ap.add_argument("--fused", action="store_true", help="fused append (k_new / v_new)")
    ap.add_argument("--nbuf", type=int, default=0, help="KV buffer sets to rotate (0: >= 2 GiB)")
    a = ap.parse_args()
    c = CFG[a.cfg]
    B, Hq, Hkv, L, dt, D, P = c["B"], c["Hq"], c["Hkv"], c["L"], c["dtype"], 128, a.P
    esz = torch.tensor([], dtype=dt).element_size()
    import numpy as np

    if c.get("mixed"):
        r = np.random.default_rng(2024)
        lens_np = np.exp(r.uniform(np.log(128), np.log(L), B)).astype(np.int32)
    else:
        lens_np = np.full(B, L, np.int32)
    layer_bytes = 2 * int(lens_np.sum()) * Hkv * D * esz
    nbuf = a.nbuf or max(2, math.ceil(2 * 2**30 / layer_bytes))
    g = torch.Generator(device="cuda").manual_seed(0)
    bufs = []
    for _ in range(nbuf):
        if c["paged"]:
            npages = B * L // P
            kp = torch.empty((npages, Hkv, P, D), dtype=dt, device="cuda").uniform_(-1, 1, generator=g)
            vp = torch.empty_like(kp).uniform_(-1, 1, generator=g)
            pt = torch.randperm(npages, generator=torch.Generator().manual_seed(1)).to(torch.int32).view(B, L // P).cuda()
        else:
            kp = torch.empty((B, Hkv, L, D), dtype=dt, device="cuda").uniform_(-1, 1, generator=g)
            vp = torch.empty_like(kp).uniform_(-1, 1, generator=g)
            pt = None
        bufs.append((kp, vp, pt))
    q = torch.empty((B, Hq, D), dtype=dt, device="cuda").uniform_(-1, 1, generator=g)
    lens = torch.tensor(lens_np, dtype=torch.int32, device="cuda")
    order = None if (a.no_order or not c.get("mixed")) else dec.longest_first(lens)
    out = torch.empty_like(q)
    kn = vn = None
    if a.fused:
        kn = torch.empty((B, Hkv, D), dtype=dt, device="cuda").uniform_(-1, 1, generator=g)
        vn = torch.empty_like(kn).uniform_(-1, 1, generator=g)
    for kern in a.kernels.split(","):
        for st in [int(x) for x in a.splits.split(",")]:
            try:
                kname, S, chunk = dec.plan(q, bufs[0][0], bufs[0][1], lens, page_table=bufs[0][2],
                                           max_len=L, kernel=kern, split_tokens=st)
            except Exception as e:  # noqa: BLE001
                print(f"{a.cfg} kernel={kern} split={st}: {e}")
                continue
            def run(i):
                kp, vp, pt = bufs[i % nbuf]
                dec.decode(q, kp, vp, lens, page_table=pt, max_len=L, out=out, kernel=kern,
                           split_tokens=st, request_order=order, k_new=kn, v_new=vn)
            for i in range(a.warm):
                run(i)
            torch.cuda.synchronize()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(a.iters)]
            for i, (e0, e1) in enumerate(evs):
                e0.record()
                run(i)
                e1.record()
            torch.cuda.synchronize()
            ts = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
            med = ts[len(ts) // 2]
            print(f"{a.cfg} kernel={kname} S={S} chunk={chunk}: median {med*1e3:.1f} us "
                  f"min {ts[0]*1e3:.1f} -> {layer_bytes / (med / 1e3) / 1e9:.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
