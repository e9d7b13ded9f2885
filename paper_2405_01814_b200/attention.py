"""Python mirror of the reference operator API (reference core/include/disagg/attention.hpp).

Same names, argument meaning and error behaviour as the C++ API, over numpy arrays
instead of nested std::vectors.  Every computation runs on the GPU through the C-ABI
host-buffer entry points (lam_*_host); host code here only validates and marshals, as
the C++ drop-in (dropin/attention.cpp) does.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import Error, ValidationError, check

__all__ = [
    "AttnInstance", "PartialAttention", "MultiHeadInstance", "HeadRange", "RequestAssignment",
    "exact_attention", "partial_attention", "merge", "finalize", "split_prev_new",
    "multi_head_attention", "head_partition", "request_partition", "exact_attention_batch",
    "Error", "ValidationError",
]


def _dt(dtype) -> int:
    dtype = np.dtype(dtype)
    if dtype == np.float64:
        return _lib.LAM_F64
    if dtype == np.float32:
        return _lib.LAM_F32
    raise ValidationError(f"unsupported dtype {dtype}; the reference instantiates float and double")


def _ptr(a: np.ndarray | None) -> int | None:
    return None if a is None else a.ctypes.data


@dataclass
class AttnInstance:
    """attention.hpp:20-30: query[d], keys[l][d], values[l][d], scale."""

    query: np.ndarray
    keys: np.ndarray
    values: np.ndarray
    scale: float = 1.0

    def __post_init__(self):
        self.query = np.asarray(self.query)
        dt = self.query.dtype if self.query.dtype in (np.float32, np.float64) else np.float64
        self.query = np.ascontiguousarray(self.query, dtype=dt)
        d = self.query.shape[0]
        self.keys = np.ascontiguousarray(np.asarray(self.keys, dtype=dt).reshape(-1, d))
        self.values = np.ascontiguousarray(np.asarray(self.values, dtype=dt).reshape(-1, d))

    @property
    def dtype(self):
        return self.query.dtype

    def length(self) -> int:
        return int(self.keys.shape[0])

    def head_dim(self) -> int:
        return int(self.query.shape[0])

    def validate(self) -> None:
        if self.query.size == 0:
            raise ValidationError("query must be non-empty")
        if self.keys.shape[0] != self.values.shape[0]:
            raise ValidationError("keys and values must have equal row counts")
        for name, arr in (("query", self.query), ("key", self.keys), ("value", self.values)):
            if not np.all(np.isfinite(arr)):
                raise ValidationError(f"{name} entries must be finite")


@dataclass
class PartialAttention:
    """attention.hpp:36-45 max-shifted partial: acc, log_denom, max_logit, token_count."""

    acc: np.ndarray
    log_denom: float = float("-inf")
    max_logit: float = float("-inf")
    token_count: int = 0

    @staticmethod
    def identity(head_dim: int, dtype=np.float64) -> "PartialAttention":
        return PartialAttention(np.zeros(head_dim, dtype=dtype))

    def empty(self) -> bool:
        return self.token_count == 0


def exact_attention_batch(q: np.ndarray, k_rows: np.ndarray, v_rows: np.ndarray,
                          kv_row0: np.ndarray, kv_len: np.ndarray,
                          scale: np.ndarray) -> np.ndarray:
    """exact_attention over n instances sharing row pools (lam_exact_attention_host)."""
    q = np.ascontiguousarray(q)
    dt = q.dtype
    n, d = q.shape
    k_rows = np.ascontiguousarray(k_rows, dtype=dt).reshape(-1, d)
    v_rows = np.ascontiguousarray(v_rows, dtype=dt).reshape(-1, d)
    row0 = np.ascontiguousarray(kv_row0, dtype=np.int64)
    ln = np.ascontiguousarray(kv_len, dtype=np.int64)
    sc = np.ascontiguousarray(np.broadcast_to(np.asarray(scale, dtype=dt), (n,)))
    out = np.empty((n, d), dtype=dt)
    check(_lib.load().lam_exact_attention_host(
        _dt(dt), n, d, _ptr(q), k_rows.shape[0], _ptr(k_rows), _ptr(v_rows), _ptr(row0),
        _ptr(ln), _ptr(sc), _ptr(out)))
    return out


def exact_attention(inst: AttnInstance) -> np.ndarray:
    """softmax(q K^T scale) V (attention.cpp:48-70).  Error on an empty key set."""
    if inst.length() == 0:
        raise Error("exact_attention requires a non-empty key set")
    return exact_attention_batch(inst.query[None, :], inst.keys, inst.values, np.zeros(1),
                                 np.array([inst.length()]), inst.scale)[0]


def _partials(inst: AttnInstance, sets: Sequence[Sequence[int]]) -> list[PartialAttention]:
    dt = inst.dtype
    d = inst.head_dim()
    n = len(sets)
    q = np.ascontiguousarray(np.broadcast_to(inst.query, (n, d)))
    idx = np.ascontiguousarray(np.concatenate([np.asarray(s, dtype=np.int64).ravel() for s in sets])
                               if n else np.zeros(0, np.int64), dtype=np.int64)
    off = np.zeros(n + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(s) for s in sets])
    row0 = np.zeros(n, dtype=np.int64)
    ln = np.full(n, inst.length(), dtype=np.int64)
    sc = np.full(n, inst.scale, dtype=dt)
    acc = np.empty((n, d), dtype=dt)
    mx = np.empty(n, dtype=dt)
    ld = np.empty(n, dtype=dt)
    cnt = np.empty(n, dtype=np.int64)
    check(_lib.load().lam_partial_attention_host(
        _dt(dt), n, d, _ptr(q), inst.length(), _ptr(inst.keys), _ptr(inst.values), _ptr(row0),
        _ptr(ln), _ptr(idx if idx.size else np.zeros(1, np.int64)), _ptr(off), _ptr(sc), _ptr(acc),
        _ptr(mx), _ptr(ld), _ptr(cnt)))
    return [PartialAttention(acc[i].copy(), dt.type(ld[i]), dt.type(mx[i]), int(cnt[i]))
            for i in range(n)]


def partial_attention(inst: AttnInstance, indices: Sequence[int]) -> PartialAttention:
    """Partial over an index subset (attention.cpp:72-98); empty subset -> identity."""
    return _partials(inst, [indices])[0]


def merge(a: PartialAttention, b: PartialAttention) -> PartialAttention:
    """Associative merge (attention.cpp:100-118); identity early-outs are bitwise."""
    if not a.empty() and not b.empty() and a.acc.shape != b.acc.shape:
        raise ValidationError("partials must share a head dim")
    dt = a.acc.dtype if not a.empty() else b.acc.dtype
    d = a.acc.shape[0] if not a.empty() else b.acc.shape[0]

    def side(p):
        acc = np.zeros(d, dtype=dt)
        acc[: min(d, p.acc.shape[0])] = p.acc[:d]
        return (acc, np.array([p.max_logit], dt), np.array([p.log_denom], dt),
                np.array([p.token_count], np.int64))

    aa, am, al, ac = side(a)
    ba, bm, bl, bc = side(b)
    oa = np.empty(d, dt)
    om, ol = np.empty(1, dt), np.empty(1, dt)
    oc = np.empty(1, np.int64)
    check(_lib.load().lam_merge_host(_dt(dt), 1, d, _ptr(aa), _ptr(am), _ptr(al), _ptr(ac),
                                     _ptr(ba), _ptr(bm), _ptr(bl), _ptr(bc), _ptr(oa), _ptr(om),
                                     _ptr(ol), _ptr(oc)))
    return PartialAttention(oa, dt.type(ol[0]), dt.type(om[0]), int(oc[0]))


def finalize(p: PartialAttention) -> np.ndarray:
    """acc / exp(log_denom) (attention.cpp:120-127); Error on the empty partial."""
    if p.empty():
        raise Error("cannot finalize an empty partial")
    dt = p.acc.dtype
    out = np.empty_like(p.acc)
    ld = np.array([p.log_denom], dt)
    cnt = np.array([p.token_count], np.int64)
    check(_lib.load().lam_finalize_host(_dt(dt), 1, p.acc.shape[0], _ptr(np.ascontiguousarray(p.acc)),
                                        _ptr(ld), _ptr(cnt), _ptr(out)))
    return out


def split_prev_new(inst: AttnInstance, boundary: int):
    """Partials over [0, boundary) and [boundary, l) (attention.cpp:129-139)."""
    if boundary < 0 or boundary > inst.length():
        raise Error("split boundary out of range")
    prev = np.arange(boundary, dtype=np.int64)
    fresh = np.arange(boundary, inst.length(), dtype=np.int64)
    a, b = _partials(inst, [prev, fresh])
    return a, b


@dataclass
class MultiHeadInstance:
    """attention.hpp:77-87: queries[Hq][d], kv_keys/kv_values[Hkv][l][d], scale."""

    queries: np.ndarray
    kv_keys: np.ndarray
    kv_values: np.ndarray
    scale: float = 1.0

    def num_query_heads(self) -> int:
        return int(np.asarray(self.queries).shape[0])

    def num_kv_heads(self) -> int:
        return int(np.asarray(self.kv_keys).shape[0])

    def head_instance(self, query_head: int) -> AttnInstance:
        group = self.num_query_heads() // self.num_kv_heads()
        return AttnInstance(np.array(self.queries[query_head]),
                            np.array(self.kv_keys[query_head // group]),
                            np.array(self.kv_values[query_head // group]), self.scale)


def multi_head_attention(inst: MultiHeadInstance) -> np.ndarray:
    """Per-head outputs, head-major (attention.cpp:152-162); GQA without KV copies."""
    if inst.num_kv_heads() <= 0:
        raise ValidationError("need at least one KV head")
    if inst.num_query_heads() % inst.num_kv_heads() != 0:
        raise ValidationError("query heads must be a multiple of KV heads")
    q = np.ascontiguousarray(inst.queries)
    dt = q.dtype if q.dtype in (np.float32, np.float64) else np.float64
    q = q.astype(dt, copy=False)
    hq, d = q.shape
    k = np.ascontiguousarray(inst.kv_keys, dtype=dt)
    v = np.ascontiguousarray(inst.kv_values, dtype=dt)
    hkv, l = k.shape[0], k.shape[1]
    if l == 0:
        raise Error("exact_attention requires a non-empty key set")
    group = hq // hkv
    heads = np.arange(hq)
    row0 = (heads // group) * l
    return exact_attention_batch(q, k.reshape(-1, d), v.reshape(-1, d), row0,
                                 np.full(hq, l), np.full(hq, inst.scale, dtype=dt))


@dataclass
class HeadRange:
    begin: int = 0
    end: int = 0


@dataclass
class RequestAssignment:
    device_of: list = field(default_factory=list)
    device_load: list = field(default_factory=list)
    imbalance: float = 1.0


def head_partition(num_kv_heads: int, num_devices: int) -> list[HeadRange]:
    """Contiguous equal KV-head ranges (attention.cpp:164-177)."""
    r = np.zeros(2 * max(num_devices, 0), dtype=np.int64)
    check(_lib.load().lam_head_partition(num_kv_heads, num_devices,
                                         _ptr(r) if r.size else None))
    return [HeadRange(int(r[2 * i]), int(r[2 * i + 1])) for i in range(num_devices)]


def request_partition(kv_sizes: Sequence[float], num_devices: int) -> RequestAssignment:
    """Greedy longest-first bin packing (attention.cpp:179-203)."""
    s = np.ascontiguousarray(kv_sizes, dtype=np.float64)
    dev = np.zeros(max(s.size, 1), dtype=np.int64)
    load = np.zeros(max(num_devices, 1), dtype=np.float64)
    imb = C.c_double(1.0)
    check(_lib.load().lam_request_partition(_ptr(s) if s.size else None, s.size, num_devices,
                                            _ptr(dev), _ptr(load), C.byref(imb)))
    return RequestAssignment([int(x) for x in dev[: s.size]], [float(x) for x in load[:num_devices]],
                             float(imb.value))
