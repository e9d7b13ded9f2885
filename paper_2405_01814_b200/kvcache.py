"""HBM-resident paged KV store (the B200 side of the reference's KvLedger byte accounting,
reference core/src/sim.cpp:14-45).

Pools are one allocation per K and V: [layers, num_pages, Hkv, page_size, D], so a layer's
pool is a contiguous [num_pages, Hkv, P, D] view, one (page, kv head) block is P*D
contiguous elements (one TMA bulk copy per decode tile) and every row is 16-byte aligned.
Pages are handed out from a host free list (optionally shuffled, to exercise arbitrary
physical placement); the page table is int32 [max_batch, max_pages_per_seq] on the device.
"""
from __future__ import annotations

import numpy as np
import torch

from . import decode as _decode


class PagedKVCache:
    def __init__(self, num_layers: int, num_kv_heads: int, head_dim: int, page_size: int,
                 num_pages: int, max_batch: int, max_pages_per_seq: int,
                 dtype: torch.dtype = torch.bfloat16, device: str | torch.device = "cuda",
                 shuffle_seed: int | None = None):
        self.num_layers, self.num_kv_heads, self.head_dim = num_layers, num_kv_heads, head_dim
        self.page_size, self.num_pages = page_size, num_pages
        self.dtype, self.device = dtype, torch.device(device)
        shape = (num_layers, num_pages, num_kv_heads, page_size, head_dim)
        self.k = torch.empty(shape, dtype=dtype, device=self.device)
        self.v = torch.empty(shape, dtype=dtype, device=self.device)
        order = np.arange(num_pages, dtype=np.int32)
        if shuffle_seed is not None:
            np.random.default_rng(shuffle_seed).shuffle(order)
        self._free = list(order[::-1])  # pop() hands out order[0], order[1], ...
        self.max_batch, self.max_pages_per_seq = max_batch, max_pages_per_seq
        self.page_table_host = np.full((max_batch, max_pages_per_seq), -1, dtype=np.int32)
        self.pages_of = [[] for _ in range(max_batch)]
        self.seq_lens_host = np.zeros(max_batch, dtype=np.int32)
        self.page_table = torch.zeros((max_batch, max_pages_per_seq), dtype=torch.int32,
                                      device=self.device)
        self.seq_lens = torch.zeros(max_batch, dtype=torch.int32, device=self.device)

    # ---- allocation (host bookkeeping) ----
    def free_pages(self) -> int:
        return len(self._free)

    def reserve(self, b: int, n_tokens: int) -> None:
        """Make request b able to hold n_tokens tokens (allocates whole pages)."""
        need = -(-n_tokens // self.page_size)
        if need > self.max_pages_per_seq:
            raise ValueError("request exceeds max_pages_per_seq")
        while len(self.pages_of[b]) < need:
            if not self._free:
                raise MemoryError("KV pool exhausted")
            p = self._free.pop()
            self.page_table_host[b, len(self.pages_of[b])] = p
            self.pages_of[b].append(p)

    def release(self, b: int) -> None:
        self._free.extend(reversed(self.pages_of[b]))
        self.pages_of[b] = []
        self.page_table_host[b, :] = -1
        self.seq_lens_host[b] = 0

    def set_lengths(self, lens) -> None:
        lens = np.asarray(lens, dtype=np.int32)
        for b, n in enumerate(lens):
            self.reserve(b, int(n))
        self.seq_lens_host[: len(lens)] = lens

    def sync(self) -> None:
        """Push the host page table and lengths to the device."""
        pt = np.where(self.page_table_host < 0, 0, self.page_table_host)
        self.page_table.copy_(torch.from_numpy(pt))
        self.seq_lens.copy_(torch.from_numpy(self.seq_lens_host))

    # ---- device views / ops ----
    def layer(self, layer: int):
        return self.k[layer], self.v[layer]

    def fill_random(self, generator: torch.Generator | None = None, lo=-1.0, hi=1.0) -> None:
        """Uniform(lo, hi) synthetic contents, layer by layer (bounded temporary memory)."""
        for layer in range(self.num_layers):
            for pool in (self.k[layer], self.v[layer]):
                pool.uniform_(lo, hi, generator=generator)

    def append(self, layer: int, k_new: torch.Tensor, v_new: torch.Tensor,
               positions: torch.Tensor, stream=None) -> None:
        kp, vp = self.layer(layer)
        _decode.kv_append(k_new, v_new, kp, vp, positions, self.page_table[: k_new.shape[0]],
                          stream=stream)

    def decode(self, layer: int, q: torch.Tensor, max_len: int | None = None, **kw):
        kp, vp = self.layer(layer)
        B = q.shape[0]
        return _decode.decode(q, kp, vp, self.seq_lens[:B], page_table=self.page_table[:B],
                              max_len=max_len if max_len is not None else
                              int(self.seq_lens_host[:B].max(initial=0)), **kw)
