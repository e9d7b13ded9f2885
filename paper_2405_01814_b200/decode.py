"""Device-tensor API of the production decode path (torch tensors in, torch tensors out).

torch provides device memory and streams only; every kernel is ours (liblamina_attn.so):

  decode(q, k_pool, v_pool, seq_lens, ...)  split-K decode attention (SIMT or GQA tensor-core)
  kv_append(...)                            bit-exact new-token write into the paged pools
  kv_gather(...)                            paged -> dense copy (inverse of the paging)

KV pools are [num_pages, Hkv, page_size, D] with a page table [B, pt_stride] (paged), or
[B, Hkv, l_max, D] with page_table=None (dense, the reference's per-request layout).
"""
from __future__ import annotations

import math

import torch

from . import _lib
from ._lib import DecodeArgs, StepLayout, check

_DT = {torch.float32: _lib.LAM_F32, torch.bfloat16: _lib.LAM_BF16, torch.float16: _lib.LAM_F16}
_KERNELS = {"auto": _lib.LAM_KERNEL_AUTO, "simt": _lib.LAM_KERNEL_SIMT,
            "gqa_mma": _lib.LAM_KERNEL_GQA_MMA, "gqa_tc": _lib.LAM_KERNEL_GQA_TC}


def _stream_ptr(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise _lib.ValidationError("decode path tensors must live on a CUDA device")


def make_args(q: torch.Tensor, k_pool: torch.Tensor, v_pool: torch.Tensor,
              seq_lens: torch.Tensor, *, page_table: torch.Tensor | None = None,
              max_len: int | None = None, scale: float | None = None,
              out: torch.Tensor | None = None, out_dtype: torch.dtype | None = None,
              lse: torch.Tensor | None = None, kernel: str = "auto",
              split_tokens: int = 0, k_new: torch.Tensor | None = None,
              v_new: torch.Tensor | None = None,
              request_order: torch.Tensor | None = None,
              overlap_prev: bool = False) -> tuple[DecodeArgs, torch.Tensor]:
    """Fill lam_decode_args from tensors; returns (args, out).  With k_new/v_new ([B, Hkv, D],
    a shared batch stride allowed) the launch also appends each request's new token at
    position seq_lens[b] - 1 (fused lam_kv_append)."""
    _require_cuda(q, k_pool, v_pool, seq_lens, page_table)
    if q.dim() != 3:
        raise _lib.ValidationError("q must be [B, Hq, D]")
    B, Hq, D = q.shape
    if k_pool.dim() != 4 or k_pool.shape != v_pool.shape:
        raise _lib.ValidationError("k_pool/v_pool must be equal-shaped 4-D pools")
    Hkv, P = k_pool.shape[1], k_pool.shape[2]
    if k_pool.shape[3] != D:
        raise _lib.ValidationError("pool head_dim differs from q")
    if k_pool.dtype != q.dtype or v_pool.dtype != q.dtype:
        raise _lib.ValidationError("q and the KV pools must share a dtype")
    for t in (k_pool, v_pool):
        if not t.is_contiguous():
            raise _lib.ValidationError("KV pools must be contiguous")
    if q.stride(2) != 1 or q.stride(1) != D:
        raise _lib.ValidationError("q rows must be contiguous [B, Hq, D] (a batch stride is allowed)")
    if seq_lens.dtype != torch.int32:
        raise _lib.ValidationError("seq_lens must be int32")
    if page_table is not None and page_table.dtype != torch.int32:
        raise _lib.ValidationError("page_table must be int32")
    if seq_lens.shape != (B,):
        raise _lib.ValidationError(f"seq_lens must be [B] = [{B}]")
    if page_table is not None:
        if page_table.dim() != 2 or page_table.shape[0] < B or not page_table[:B].is_contiguous():
            raise _lib.ValidationError("page_table must be [>= B, pages] with contiguous rows")
    elif k_pool.shape[0] < B:
        raise _lib.ValidationError("dense KV pools need one [Hkv, l_max, D] block per request")
    odt = out_dtype or (out.dtype if out is not None else q.dtype)
    if odt not in (q.dtype, torch.float32):
        raise _lib.ValidationError("out dtype must be the KV dtype or float32")
    if out is None:
        out = torch.empty((B, Hq, D), dtype=odt, device=q.device)
    elif out.shape != (B, Hq, D) or out.dtype != odt or not out.is_contiguous() or not out.is_cuda:
        raise _lib.ValidationError(f"out must be a contiguous CUDA [{B}, {Hq}, {D}] {odt} tensor")
    a = DecodeArgs()
    a.kv_dtype = _DT[q.dtype]
    a.out_dtype = _DT[odt]
    a.batch, a.num_q_heads, a.num_kv_heads, a.head_dim = B, Hq, Hkv, D
    a.scale = float(scale if scale is not None else 1.0 / math.sqrt(D))
    a.page_size = P
    a.pt_stride = page_table.shape[1] if page_table is not None else 0
    a.max_len = int(max_len if max_len is not None else
                    (page_table.shape[1] * P if page_table is not None else P))
    a.split_tokens = int(split_tokens)
    a.kernel = _KERNELS[kernel]
    a.num_pages = k_pool.shape[0] if page_table is not None else 0
    a.q, a.k_pool, a.v_pool = q.data_ptr(), k_pool.data_ptr(), v_pool.data_ptr()
    a.page_table = page_table.data_ptr() if page_table is not None else None
    a.seq_lens = seq_lens.data_ptr()
    a.out = out.data_ptr()
    a.lse = lse.data_ptr() if lse is not None else None
    a.q_batch_stride = q.stride(0) if B > 1 and q.stride(0) != Hq * D else 0
    if (k_new is None) != (v_new is None):
        raise _lib.ValidationError("fused append needs both k_new and v_new")
    if k_new is not None:
        _require_cuda(k_new, v_new)
        if (k_new.shape != (B, Hkv, D) or k_new.dtype != q.dtype or k_new.stride(2) != 1
                or k_new.stride(1) != D or v_new.stride() != k_new.stride()
                or v_new.shape != k_new.shape):
            raise _lib.ValidationError("k_new/v_new must be [B, Hkv, D] rows sharing a batch stride")
        a.k_new, a.v_new = k_new.data_ptr(), v_new.data_ptr()
        a.new_batch_stride = k_new.stride(0) if B > 1 else 0
    if request_order is not None:
        _require_cuda(request_order)
        if request_order.dtype != torch.int32 or request_order.shape != (B,):
            raise _lib.ValidationError("request_order must be int32 [B]")
        a.request_order = request_order.data_ptr()
    a.overlap_prev = 1 if overlap_prev else 0
    return a, out


def decode(q, k_pool, v_pool, seq_lens, *, page_table=None, max_len=None, scale=None, out=None,
           out_dtype=None, return_lse=False, kernel="auto", split_tokens=0, ctx=None,
           stream=None, k_new=None, v_new=None, request_order=None, overlap_prev=False):
    """softmax(q K^T scale) V per (request, q head) over the request's first seq_lens[b]
    tokens; q head h reads KV head h // (Hq // Hkv).  With k_new / v_new the request's new
    token (position seq_lens[b] - 1) is taken from them and appended to the pools in the same
    launch.  overlap_prev: see lam_decode_args.overlap_prev (the launch may start streaming KV
    while the stream's preceding kernel drains; q / k_new / v_new are read after it completes)."""
    lse = None
    if return_lse:
        lse = torch.empty(q.shape[:2], dtype=torch.float32, device=q.device)
    a, out = make_args(q, k_pool, v_pool, seq_lens, page_table=page_table, max_len=max_len,
                       scale=scale, out=out, out_dtype=out_dtype, lse=lse, kernel=kernel,
                       split_tokens=split_tokens, k_new=k_new, v_new=v_new,
                       request_order=request_order, overlap_prev=overlap_prev)
    ctx = ctx or _lib.context(q.device.index or 0)
    check(_lib.load().lam_decode(ctx.handle, a, _stream_ptr(stream)))
    return (out, lse) if return_lse else out


def step_layout(n_layers: int, n_mb: int, rows_per_mb: int, *, pool_layers: int | None = None,
                layer0: int = 0, pool_layer_rows: int = 0, lm_q_stride: int = 0,
                lm_new_stride: int = 0, lm_out_stride: int = 0, flag_mb_stride: int = 0,
                epoch: int = 0) -> StepLayout:
    """lam_step_layout: launch lm = layer * n_mb + mb of a step launch (see lamina_attn.h)."""
    st = StepLayout()
    st.n_layers, st.n_mb, st.rows_per_mb = n_layers, n_mb, rows_per_mb
    st.pool_layers = pool_layers if pool_layers is not None else n_layers
    st.layer0, st.pool_layer_rows = layer0, pool_layer_rows
    st.lm_q_stride, st.lm_new_stride, st.lm_out_stride = lm_q_stride, lm_new_stride, lm_out_stride
    st.flag_mb_stride, st.epoch = flag_mb_stride, epoch & 0xFFFFFFFF
    return st


def decode_step(q, k_pools, v_pools, seq_lens, *, n_mb=1, page_table=None, max_len=None,
                scale=None, out=None, k_new=None, v_new=None, request_order=None, kernel="auto",
                layer0=0, ctx=None, stream=None, overlap_prev=False, split_tokens=0):
    """Every layer (and micro-batch) of a decode step in one persistent launch (lam_decode_step).

    q [L, n_mb * rows, Hq, D] (row stride within a layer allowed), k_pools / v_pools
    [pool_layers, pages, Hkv, P, D] (layer l uses pool layer (layer0 + l) % pool_layers),
    k_new / v_new [L, n_mb * rows, Hkv, D] (optional fused append), out [L, n_mb * rows, Hq, D].
    request_order [n_mb * rows] holds each micro-batch's permutation (indices local to it)."""
    L, B = q.shape[0], q.shape[1]
    if B % n_mb:
        raise _lib.ValidationError("rows must split evenly into micro-batches")
    if out is None:
        out = torch.empty((L,) + tuple(q.shape[1:]), dtype=q.dtype, device=q.device)
    a, _ = make_args(q[0], k_pools[0], v_pools[0], seq_lens, page_table=page_table, max_len=max_len,
                     scale=scale, out=out[0], kernel=kernel, split_tokens=split_tokens,
                     k_new=k_new[0] if k_new is not None else None,
                     v_new=v_new[0] if v_new is not None else None, request_order=None,
                     overlap_prev=overlap_prev)
    if request_order is not None:
        _require_cuda(request_order)
        if request_order.dtype != torch.int32 or request_order.shape != (B,):
            raise _lib.ValidationError("request_order must be int32 [B]")
        a.request_order = request_order.data_ptr()
    st = step_layout(L, n_mb, B // n_mb, pool_layers=k_pools.shape[0], layer0=layer0,
                     pool_layer_rows=k_pools[0].numel() // k_pools.shape[-1])
    # launch lm = layer * n_mb + mb starts rows * stride(1) elements after launch lm - 1, which
    # needs each layer's rows stored back to back (stride(0) = n_mb * rows * stride(1))
    rows = B // n_mb
    for t, name in ((q, "lm_q_stride"), (out, "lm_out_stride")) + (
            ((k_new, "lm_new_stride"),) if k_new is not None else ()):
        if n_mb > 1 and t.stride(0) != n_mb * rows * t.stride(1):
            raise _lib.ValidationError(f"{name}: a layer's rows must be stored back to back")
        setattr(st, name, t.stride(0) if n_mb == 1 else rows * t.stride(1))
    ctx = ctx or _lib.context(q.device.index or 0)
    check(_lib.load().lam_decode_step(ctx.handle, a, st, None, _stream_ptr(stream)))
    return out


def longest_first(seq_lens: torch.Tensor) -> torch.Tensor:
    """Request permutation for `request_order`: longest sequence first (LPT)."""
    return torch.argsort(seq_lens, descending=True, stable=True).to(torch.int32)


def plan(q, k_pool, v_pool, seq_lens, **kw):
    """(kernel family, splits, tokens per split) lam_decode would use."""
    ctx = kw.pop("ctx", None) or _lib.context(q.device.index or 0)
    a, _ = make_args(q, k_pool, v_pool, seq_lens, **kw)
    import ctypes as C

    k, s, t = C.c_int32(), C.c_int32(), C.c_int32()
    check(_lib.load().lam_decode_plan(ctx.handle, a, C.byref(k), C.byref(s), C.byref(t)))
    names = {_lib.LAM_KERNEL_SIMT: "simt", _lib.LAM_KERNEL_GQA_MMA: "gqa_mma",
             _lib.LAM_KERNEL_GQA_TC: "gqa_tc"}
    return names[k.value], s.value, t.value


def plan_grid(q, k_pool, v_pool, seq_lens, **kw) -> int:
    """Persistent grid size (CTAs) lam_decode would launch."""
    ctx = kw.pop("ctx", None) or _lib.context(q.device.index or 0)
    a, _ = make_args(q, k_pool, v_pool, seq_lens, **kw)
    import ctypes as C

    n = C.c_int32()
    check(_lib.load().lam_decode_plan_grid(ctx.handle, a, C.byref(n)))
    return n.value


def kv_append(k_new, v_new, k_pool, v_pool, positions, page_table=None, stream=None):
    """k_pool[page(b, pos)][h][pos % P] = k_new[b][h] (and V), pos = positions[b].
    k_new / v_new are [B, Hkv, D] with contiguous heads; a batch stride (e.g. slices of a packed
    QKV projection output [B, Hq + 2 Hkv, D]) is allowed if both share it."""
    _require_cuda(k_new, v_new, k_pool, v_pool, positions, page_table)
    B, Hkv, D = k_new.shape
    if (k_new.stride(2) != 1 or k_new.stride(1) != D or v_new.stride() != k_new.stride()):
        raise _lib.ValidationError("k_new/v_new must be [B, Hkv, D] rows with one shared batch stride")
    P = k_pool.shape[2]
    pts = page_table.shape[1] if page_table is not None else 0
    check(_lib.load().lam_kv_append(
        _DT[k_new.dtype], B, Hkv, D, P, pts,
        page_table.data_ptr() if page_table is not None else None, positions.data_ptr(),
        k_new.data_ptr(), v_new.data_ptr(), k_new.stride(0) if B > 1 else 0, k_pool.data_ptr(),
        v_pool.data_ptr(), _stream_ptr(stream)))


def kv_gather(pool, page_table, seq_lens, l_max, stream=None):
    """Dense [B, Hkv, l_max, D] copy of the first seq_lens[b] tokens of each request."""
    _require_cuda(pool, page_table, seq_lens)
    B = seq_lens.shape[0]
    _, Hkv, P, D = pool.shape
    dense = torch.zeros((B, Hkv, l_max, D), dtype=pool.dtype, device=pool.device)
    check(_lib.load().lam_kv_gather(_DT[pool.dtype], B, Hkv, D, P, page_table.shape[1],
                                    page_table.data_ptr(), seq_lens.data_ptr(), l_max,
                                    pool.data_ptr(), dense.data_ptr(), _stream_ptr(stream)))
    return dense
