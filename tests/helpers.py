"""Shared builders for the GPU parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np
import torch


def bf16_round_np(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def make_dense(B, Hq, Hkv, D, lmax, dtype, seed=0, device="cuda", lo=-1.0, hi=1.0):
    """Seeded uniform q [B,Hq,D], k/v [B,Hkv,lmax,D] on the device in `dtype`."""
    g = torch.Generator(device=device).manual_seed(seed)
    q = torch.empty((B, Hq, D), dtype=torch.float32, device=device).uniform_(lo, hi, generator=g)
    k = torch.empty((B, Hkv, lmax, D), dtype=torch.float32, device=device).uniform_(lo, hi, generator=g)
    v = torch.empty((B, Hkv, lmax, D), dtype=torch.float32, device=device).uniform_(lo, hi, generator=g)
    return q.to(dtype), k.to(dtype), v.to(dtype)


def page_table_for(lens, P, seed=0, spare=3):
    """Shuffled physical pages for each request: int32 [B, max_pages], num_pages."""
    lens = np.asarray(lens)
    pages = np.maximum(1, -(-lens // P))
    total = int(pages.sum()) + spare
    perm = np.random.default_rng(seed).permutation(total).astype(np.int32)
    pt = np.zeros((len(lens), int(pages.max())), np.int32)
    o = 0
    for b, n in enumerate(pages):
        pt[b, :n] = perm[o: o + n]
        o += n
    return pt, total


def to_paged(k_dense: torch.Tensor, lens, P, page_table: np.ndarray, num_pages: int,
             fill: float = float("nan")):
    """Scatter dense [B,Hkv,lmax,D] into a pool [num_pages,Hkv,P,D] (torch indexing, test
    infrastructure).  Unused rows are filled with `fill` (NaN by default) so that a kernel
    reading past a sequence end is caught."""
    B, Hkv, lmax, D = k_dense.shape
    pool = torch.full((num_pages, Hkv, P, D), fill, dtype=k_dense.dtype, device=k_dense.device)
    for b in range(B):
        l = int(lens[b])
        for i in range(-(-l // P)):
            t0, t1 = i * P, min(l, (i + 1) * P)
            pool[int(page_table[b, i]), :, : t1 - t0] = k_dense[b, :, t0:t1]
    return pool


def oracle_decode(q, k, v, lens, scale, pairs=None, want_lse=False, compute_f64=False):
    from oracle import oracle as O

    return O.decode_dense(q.float().cpu().numpy(), k.float().cpu().numpy(),
                          v.float().cpu().numpy(), np.asarray(lens, np.int32), scale,
                          compute_f64=compute_f64, pairs=pairs, want_lse=want_lse)
