"""B200-native (sm_100a) implementation of Lamina's offloaded decode-attention operator
(arXiv 2405.01814), behind the reference's operator API (proj/core attention.hpp).

Layout:
  csrc/      CUDA kernels (TMA-fed split-K decode, GQA tensor-core decode, KV append/gather,
             reference-API instance kernels) and the extern "C" boundary (capi.cu)
  dropin/    the C++ drop-in for the reference's disagg::* attention API
  _lib.py    ctypes binding of include/lamina_attn.h
  attention  Python mirror of the reference API (numpy in, GPU compute)
  decode     torch-tensor API of the production path
  kvcache    paged HBM KV store
  dist       KV-head-sharded attention worker pool over torch.distributed / NCCL
  perf       the reference's attn_cost / kv_bytes_per_token / mbu contract
"""
from ._lib import Error, ValidationError, CudaError  # noqa: F401

__version__ = "0.1.0"
