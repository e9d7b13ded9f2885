"""ctypes binding of the C-ABI in include/lamina_attn.h (lib/liblamina_attn.so).

The library is loaded from the package's in-tree lib/ directory.  There is no fallback:
if the .so is missing or cannot be loaded, importing an op raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"
CORE_PATH = LIB_DIR / "liblamina_attn.so"
DROPIN_PATH = LIB_DIR / "libdisagg_attention.so"

LAM_OK, LAM_ERR_ERROR, LAM_ERR_VALIDATION, LAM_ERR_CUDA = 0, 1, 2, 3
LAM_F32, LAM_F64, LAM_BF16, LAM_F16 = 0, 1, 2, 3
LAM_KERNEL_AUTO, LAM_KERNEL_SIMT, LAM_KERNEL_GQA_MMA, LAM_KERNEL_GQA_TC = 0, 1, 2, 3
LAM_STATUS_OK, LAM_STATUS_INPUT_TIMEOUT, LAM_STATUS_SLOT_TIMEOUT = 0, 1, 2


class Error(RuntimeError):
    """disagg::Error (reference model.hpp:25-28)."""


class ValidationError(Error):
    """disagg::ValidationError (reference model.hpp:31-34)."""


class CudaError(Error):
    """A CUDA runtime/driver failure surfaced through the C-ABI."""


class DecodeArgs(C.Structure):
    """lam_decode_args (include/lamina_attn.h)."""

    _fields_ = [
        ("kv_dtype", C.c_int32),
        ("out_dtype", C.c_int32),
        ("batch", C.c_int32),
        ("num_q_heads", C.c_int32),
        ("num_kv_heads", C.c_int32),
        ("head_dim", C.c_int32),
        ("scale", C.c_float),
        ("page_size", C.c_int32),
        ("pt_stride", C.c_int32),
        ("max_len", C.c_int32),
        ("split_tokens", C.c_int32),
        ("kernel", C.c_int32),
        ("num_pages", C.c_int64),
        ("q", C.c_void_p),
        ("k_pool", C.c_void_p),
        ("v_pool", C.c_void_p),
        ("page_table", C.c_void_p),
        ("seq_lens", C.c_void_p),
        ("out", C.c_void_p),
        ("lse", C.c_void_p),
        ("q_batch_stride", C.c_int64),
        ("k_new", C.c_void_p),
        ("v_new", C.c_void_p),
        ("new_batch_stride", C.c_int64),
        ("request_order", C.c_void_p),
        ("overlap_prev", C.c_int32),
    ]


LAM_MAX_PEERS = 8
LAM_IPC_HANDLE_BYTES = 64


class PeerIO(C.Structure):
    """lam_peer_io (include/lamina_attn.h)."""

    _fields_ = [
        ("n_src", C.c_int32),
        ("rows_per_src", C.c_int32),
        ("q_src", C.c_void_p * LAM_MAX_PEERS),
        ("out_dst", C.c_void_p * LAM_MAX_PEERS),
        ("k_new_offset", C.c_int64),
        ("v_new_offset", C.c_int64),
        ("n_wait", C.c_int32),
        ("n_done", C.c_int32),
        ("wait_value", C.c_uint32),
        ("done_value", C.c_uint32),
        ("wait_flags", C.c_void_p * LAM_MAX_PEERS),
        ("done_flags", C.c_void_p * LAM_MAX_PEERS),
        ("n_wait_kv", C.c_int32),
        ("kv_wait_value", C.c_uint32),
        ("kv_wait_flags", C.c_void_p * LAM_MAX_PEERS),
        ("n_relay", C.c_int32),
        ("relay_flag", C.c_void_p),
        ("relay_wait_flags", C.c_void_p * LAM_MAX_PEERS),
        ("row_src", C.c_void_p),
    ]


class StepLayout(C.Structure):
    """lam_step_layout (include/lamina_attn.h)."""

    _fields_ = [
        ("n_layers", C.c_int32),
        ("n_mb", C.c_int32),
        ("rows_per_mb", C.c_int32),
        ("pool_layers", C.c_int32),
        ("layer0", C.c_int32),
        ("flag_mb_stride", C.c_int32),
        ("pool_layer_rows", C.c_int64),
        ("lm_q_stride", C.c_int64),
        ("lm_new_stride", C.c_int64),
        ("lm_out_stride", C.c_int64),
        ("epoch", C.c_uint32),
        ("trace", C.c_void_p),
    ]


_P, _I32, _I64, _F64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double

# name -> (restype, argtypes)
SIGNATURES = {
    "lam_version": (C.c_int, []),
    "lam_last_error": (C.c_char_p, []),
    "lam_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "lam_ctx_destroy": (C.c_int, [_P]),
    "lam_ctx_reserve": (C.c_int, [_P, _I64, _I32, _I64]),
    "lam_ctx_num_sms": (C.c_int, [_P]),
    "lam_ctx_set_spin_timeout": (C.c_int, [_P, _I64]),
    "lam_ctx_status": (C.c_int, [_P, _P, _I32]),
    "lam_exact_attention": (C.c_int, [_P, C.c_int, _I64, _I32, _P, _P, _P, _P, _P, _P, _P, _P]),
    "lam_partial_attention": (C.c_int, [_P, C.c_int, _I64, _I32, _P, _P, _P, _P, _P, _P, _P, _P,
                                        _P, _P, _P, _P, _P]),
    "lam_merge": (C.c_int, [_P, C.c_int, _I64, _I32] + [_P] * 13),
    "lam_finalize": (C.c_int, [_P, C.c_int, _I64, _I32, _P, _P, _P, _P, _P]),
    "lam_exact_attention_host": (C.c_int, [C.c_int, _I64, _I32, _P, _I64, _P, _P, _P, _P, _P, _P]),
    "lam_partial_attention_host": (C.c_int, [C.c_int, _I64, _I32, _P, _I64, _P, _P, _P, _P, _P, _P,
                                             _P, _P, _P, _P, _P]),
    "lam_merge_host": (C.c_int, [C.c_int, _I64, _I32] + [_P] * 12),
    "lam_finalize_host": (C.c_int, [C.c_int, _I64, _I32, _P, _P, _P, _P]),
    "lam_head_partition": (C.c_int, [_I64, _I64, _P]),
    "lam_host_buffer": (C.c_void_p, [_I32, _I64]),
    "lam_request_partition": (C.c_int, [_P, _I64, _I64, _P, _P, _P]),
    "lam_decode": (C.c_int, [_P, C.POINTER(DecodeArgs), _P]),
    "lam_decode_plan": (C.c_int, [_P, C.POINTER(DecodeArgs), _P, _P, _P]),
    "lam_decode_plan_grid": (C.c_int, [_P, C.POINTER(DecodeArgs), _P]),
    "lam_kv_append": (C.c_int, [_I32, _I32, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _I64, _P, _P,
                                _P]),
    "lam_kv_gather": (C.c_int, [_I32, _I32, _I32, _I32, _I32, _I32, _P, _P, _I32, _P, _P, _P]),
    "lam_decode_step_host": (C.c_int, [_P, C.POINTER(DecodeArgs), _P, _P, _P, _P, _P, _P, _P,
                                       _P]),
    "lam_decode_layers_host": (C.c_int, [_P, C.POINTER(DecodeArgs), _I32, _P, _P, _P, _P, _P, _P,
                                         _P, _P]),
    "lam_decode_layers_host_stage_bytes": (C.c_int64, [C.POINTER(DecodeArgs)]),
    "lam_peer_alloc": (C.c_int, [_P, _I64, C.POINTER(C.c_void_p), _P]),
    "lam_peer_free": (C.c_int, [_P, _P]),
    "lam_peer_open": (C.c_int, [_P, _P, C.POINTER(C.c_void_p)]),
    "lam_peer_close": (C.c_int, [_P, _P]),
    "lam_stream_signal": (C.c_int, [_P, _P, _I32, C.c_uint32, _P]),
    "lam_stream_wait": (C.c_int, [_P, _P, _I32, C.c_uint32, _P]),
    "lam_decode_peer": (C.c_int, [_P, C.POINTER(DecodeArgs), C.POINTER(PeerIO), _P]),
    "lam_decode_step": (C.c_int, [_P, C.POINTER(DecodeArgs), C.POINTER(StepLayout),
                                  C.POINTER(PeerIO), _P]),
    "lam_decode_step_from_host": (C.c_int, [_P, C.POINTER(DecodeArgs), C.POINTER(StepLayout), _P,
                                            _P, _P, _P, _P, _P, _P]),
    "lam_decode_step_from_host_stage_bytes": (C.c_int64, [C.POINTER(DecodeArgs), _I32]),
}

_lib = None


def load() -> C.CDLL:
    """Load liblamina_attn.so (in-tree).  Raises if it is missing — there is no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not CORE_PATH.exists():
        raise ImportError(
            f"{CORE_PATH} is missing: build it with `python -m paper_2405_01814_b200.build` "
            "(or __graft_entry__.build()); the decode path has no CPU fallback")
    lib = C.CDLL(str(CORE_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    """Raise the reference exception type matching a C-ABI status."""
    if status == LAM_OK:
        return
    msg = (load().lam_last_error() or b"").decode()
    if status == LAM_ERR_VALIDATION:
        raise ValidationError(msg)
    if status == LAM_ERR_ERROR:
        raise Error(msg)
    raise CudaError(msg)


class Context:
    """Owns one lam_ctx (device binding + split-K workspace)."""

    def __init__(self, device: int = 0):
        self._lib = load()
        h = C.c_void_p()
        check(self._lib.lam_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    @property
    def num_sms(self) -> int:
        return self._lib.lam_ctx_num_sms(self.handle)

    def set_spin_timeout(self, ns: int) -> None:
        check(self._lib.lam_ctx_set_spin_timeout(self.handle, int(ns)))

    def status(self, clear: bool = True) -> int:
        """LAM_STATUS_* word of the context (synchronises the device)."""
        st = C.c_int32()
        check(self._lib.lam_ctx_status(self.handle, C.byref(st), int(clear)))
        return st.value

    def reserve(self, partial_rows: int, head_dim: int, counters: int) -> None:
        check(self._lib.lam_ctx_reserve(self.handle, partial_rows, head_dim, counters))

    def close(self) -> None:
        if self.handle:
            self._lib.lam_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass


_contexts: dict[int, Context] = {}


def context(device: int = 0) -> Context:
    """Process-wide context per device (one process per GPU is the deployment model)."""
    ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        _contexts[device] = ctx
    return ctx


def declared_functions(header: Path | None = None) -> list[str]:
    """Every function name declared in include/lamina_attn.h."""
    import re

    header = header or Path(__file__).resolve().parent.parent / "include" / "lamina_attn.h"
    text = header.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(lam_\w+)\s*\(", text, re.M)))
