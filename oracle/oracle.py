"""ctypes loaders for the CPU checkers.  TEST INFRASTRUCTURE ONLY.

  port()  oracle/_build/liboracle.so   our C restatement (attn_oracle.c)
  ref()   oracle/_ref/libref_attn.so   the reference's own attention.cpp (+ ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
import this module.  The product path never does.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_PATH = HERE / "_build" / "liboracle.so"
REF_PATH = HERE / "_ref" / "libref_attn.so"
REF_TEST_DROPIN = HERE / "_ref" / "test_attention_dropin"
REF_TEST_REF = HERE / "_ref" / "test_attention_ref"

_P, _I32, _I64, _F32, _F64 = C.c_void_p, C.c_int32, C.c_int64, C.c_float, C.c_double

_PORT_SIGS = {
    "orc_exact_f64": (C.c_int, [_I64, _I64, _P, _P, _P, _F64, _P]),
    "orc_exact_f32": (C.c_int, [_I64, _I64, _P, _P, _P, _F32, _P]),
    "orc_partial_f64": (C.c_int, [_I64, _I64, _P, _P, _P, _F64, _P, _I64, _P, _P, _P, _P]),
    "orc_partial_f32": (C.c_int, [_I64, _I64, _P, _P, _P, _F32, _P, _I64, _P, _P, _P, _P]),
    "orc_merge_f64": (None, [_I64, _P, _F64, _F64, _I64, _P, _F64, _F64, _I64, _P, _P, _P, _P]),
    "orc_merge_f32": (None, [_I64, _P, _F32, _F32, _I64, _P, _F32, _F32, _I64, _P, _P, _P, _P]),
    "orc_finalize_f64": (C.c_int, [_I64, _P, _F64, _I64, _P]),
    "orc_finalize_f32": (C.c_int, [_I64, _P, _F32, _I64, _P]),
    "orc_naive_ld": (None, [_I64, _I64, _P, _P, _P, _F64, _P]),
    "orc_head_partition": (C.c_int, [_I64, _I64, _P]),
    "orc_request_partition": (C.c_int, [_P, _I64, _I64, _P, _P, _P]),
    "orc_decode": (None, [C.c_int, _I32, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _F32, _I64, _P,
                          _P, _P, _P]),
    "orc_page_scatter": (None, [_I32, _I32, _I32, _I32, _I32, _P, _P, _I32, _P, _P]),
    "orc_page_gather": (None, [_I32, _I32, _I32, _I32, _I32, _P, _P, _I32, _P, _P]),
}

_REF_SIGS = {
    "ref_exact_f64": (C.c_int, [_I64, _I64, _P, _P, _P, _F64, _P]),
    "ref_exact_f32": (C.c_int, [_I64, _I64, _P, _P, _P, _F32, _P]),
    "ref_partial_f64": (C.c_int, [_I64, _I64, _P, _P, _P, _F64, _P, _I64, _P, _P, _P, _P]),
    "ref_partial_f32": (C.c_int, [_I64, _I64, _P, _P, _P, _F32, _P, _I64, _P, _P, _P, _P]),
    "ref_merge_f64": (None, [_I64, _P, _F64, _F64, _I64, _P, _F64, _F64, _I64, _P, _P, _P, _P]),
    "ref_merge_f32": (None, [_I64, _P, _F32, _F32, _I64, _P, _F32, _F32, _I64, _P, _P, _P, _P]),
    "ref_finalize_f64": (C.c_int, [_I64, _P, _F64, _I64, _P]),
    "ref_multi_head_f64": (C.c_int, [_I64, _I64, _I64, _I64, _P, _P, _P, _F64, _P]),
    "ref_multi_head_f32": (C.c_int, [_I64, _I64, _I64, _I64, _P, _P, _P, _F32, _P]),
    "ref_head_partition": (C.c_int, [_I64, _I64, _P, C.c_char_p, _I64]),
    "ref_request_partition": (C.c_int, [_P, _I64, _I64, _P, _P, _P]),
    "ref_rng_create": (_P, [C.c_uint64]),
    "ref_rng_destroy": (None, [_P]),
    "ref_rng_next": (C.c_uint64, [_P]),
    "ref_random_instance": (None, [_P, _I64, _I64, _F64, _P, _P, _P, _P]),
    "ref_random_partition": (None, [_P, _I64, _I64, _P]),
    "ref_bench_create": (_P, [_I32, _I32, _I32, _I32, _I32, _P, _P, _P, _P, _F32, _I64]),
    "ref_bench_run": (_F64, [_P, _I32, _P]),
    "ref_bench_destroy": (None, [_P]),
    "ref_hardware_threads": (C.c_int, []),
}

_port = None
_ref = None


def _bind(lib, sigs):
    for name, (res, args) in sigs.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


def port() -> C.CDLL:
    """Our C restatement; built on demand with make (gcc only)."""
    global _port
    if _port is None:
        if not PORT_PATH.exists():
            subprocess.run(["make", "-C", str(HERE), "port"], check=True, capture_output=True)
        _port = _bind(C.CDLL(str(PORT_PATH)), _PORT_SIGS)
    return _port


def ref_available() -> bool:
    return REF_PATH.exists()


def ref() -> C.CDLL:
    """The reference's own attention.cpp (prebuilt in oracle/_ref by oracle/Makefile)."""
    global _ref
    if _ref is None:
        if not REF_PATH.exists():
            raise FileNotFoundError(f"{REF_PATH} not built (needs /root/reference at build time)")
        _ref = _bind(C.CDLL(str(REF_PATH)), _REF_SIGS)
    return _ref


def ptr(a):
    return None if a is None else a.ctypes.data


# ---------------- numpy conveniences over the port ----------------

def exact(q, k, v, scale, lib="port"):
    """exact_attention on one instance (float32 or float64 arrays)."""
    q = np.ascontiguousarray(q)
    dt = q.dtype
    k = np.ascontiguousarray(k, dtype=dt).reshape(-1, q.size)
    v = np.ascontiguousarray(v, dtype=dt).reshape(-1, q.size)
    out = np.empty_like(q)
    L = port() if lib == "port" else ref()
    pre = "orc" if lib == "port" else "ref"
    sfx = "f64" if dt == np.float64 else "f32"
    rc = getattr(L, f"{pre}_exact_{sfx}")(q.size, k.shape[0], ptr(q), ptr(k), ptr(v), scale, ptr(out))
    if rc:
        raise RuntimeError("exact_attention requires a non-empty key set")
    return out


def partial(q, k, v, scale, idx, lib="port"):
    q = np.ascontiguousarray(q)
    dt = q.dtype
    d = q.size
    k = np.ascontiguousarray(k, dtype=dt).reshape(-1, d)
    v = np.ascontiguousarray(v, dtype=dt).reshape(-1, d)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    acc = np.empty(d, dt)
    mx, ld = np.empty(1, dt), np.empty(1, dt)
    cnt = np.empty(1, np.int64)
    L = port() if lib == "port" else ref()
    pre = "orc" if lib == "port" else "ref"
    sfx = "f64" if dt == np.float64 else "f32"
    rc = getattr(L, f"{pre}_partial_{sfx}")(d, k.shape[0], ptr(q), ptr(k), ptr(v), scale,
                                            ptr(idx) if idx.size else None, idx.size, ptr(acc),
                                            ptr(mx), ptr(ld), ptr(cnt))
    if rc:
        raise IndexError("token index out of range")
    return acc, dt.type(mx[0]), dt.type(ld[0]), int(cnt[0])


def merge(a, b, lib="port"):
    """a, b = (acc, max, log_denom, count) tuples."""
    acc_a = np.ascontiguousarray(a[0])
    dt = acc_a.dtype
    d = acc_a.size
    o = np.empty(d, dt)
    om, ol = np.empty(1, dt), np.empty(1, dt)
    oc = np.empty(1, np.int64)
    L = port() if lib == "port" else ref()
    pre = "orc" if lib == "port" else "ref"
    sfx = "f64" if dt == np.float64 else "f32"
    getattr(L, f"{pre}_merge_{sfx}")(d, ptr(acc_a), a[1], a[2], a[3],
                                     ptr(np.ascontiguousarray(b[0], dtype=dt)), b[1], b[2], b[3],
                                     ptr(o), ptr(om), ptr(ol), ptr(oc))
    return o, dt.type(om[0]), dt.type(ol[0]), int(oc[0])


def finalize(p):
    acc = np.ascontiguousarray(p[0])
    out = np.empty_like(acc)
    sfx = "f64" if acc.dtype == np.float64 else "f32"
    if getattr(port(), f"orc_finalize_{sfx}")(acc.size, ptr(acc), p[2], p[3], ptr(out)):
        raise RuntimeError("cannot finalize an empty partial")
    return out


def naive(q, k, v, scale):
    q = np.ascontiguousarray(q, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.float64).reshape(-1, q.size)
    v = np.ascontiguousarray(v, dtype=np.float64).reshape(-1, q.size)
    out = np.empty_like(q)
    port().orc_naive_ld(q.size, k.shape[0], ptr(q), ptr(k), ptr(v), scale, ptr(out))
    return out


def decode_dense(q, k, v, lens, scale, compute_f64=False, pairs=None, want_lse=False):
    """Batched decode over dense fp32 arrays q [B,Hq,D], k/v [B,Hkv,lmax,D]."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    k = np.ascontiguousarray(k, dtype=np.float32)
    v = np.ascontiguousarray(v, dtype=np.float32)
    lens = np.ascontiguousarray(lens, dtype=np.int32)
    B, Hq, D = q.shape
    Hkv, lmax = k.shape[1], k.shape[2]
    out = np.zeros_like(q)
    lse = np.zeros((B, Hq), np.float32) if want_lse else None
    pb = ph = None
    n = 0
    if pairs is not None:
        pairs = np.asarray(pairs, dtype=np.int32).reshape(-1, 2)
        pb = np.ascontiguousarray(pairs[:, 0])
        ph = np.ascontiguousarray(pairs[:, 1])
        n = pairs.shape[0]
    port().orc_decode(1 if compute_f64 else 0, B, Hq, Hkv, D, lmax, ptr(lens), ptr(q), ptr(k),
                      ptr(v), scale, n, ptr(pb), ptr(ph), ptr(out), ptr(lse))
    return (out, lse) if want_lse else out


def page_gather(pool, page_table, lens, lmax):
    """pool uint8 [pages, Hkv, P, row_bytes] -> dense [B, Hkv, lmax, row_bytes]."""
    pool = np.ascontiguousarray(pool)
    pt = np.ascontiguousarray(page_table, dtype=np.int32)
    lens = np.ascontiguousarray(lens, dtype=np.int32)
    _, Hkv, P, rb = pool.shape
    B = lens.size
    dense = np.zeros((B, Hkv, lmax, rb), np.uint8)
    port().orc_page_gather(rb, B, Hkv, P, pt.shape[1], ptr(pt), ptr(lens), lmax, ptr(pool),
                           ptr(dense))
    return dense


def page_scatter(dense, page_table, lens, num_pages, P):
    dense = np.ascontiguousarray(dense)
    pt = np.ascontiguousarray(page_table, dtype=np.int32)
    lens = np.ascontiguousarray(lens, dtype=np.int32)
    B, Hkv, lmax, rb = dense.shape
    pool = np.zeros((num_pages, Hkv, P, rb), np.uint8)
    port().orc_page_scatter(rb, B, Hkv, P, pt.shape[1], ptr(pt), ptr(lens), lmax, ptr(dense),
                            ptr(pool))
    return pool


class RefRng:
    """The reference tests' std::mt19937_64 + gen::random_instance / random_partition."""

    def __init__(self, seed: int):
        self.lib = ref()
        self.h = self.lib.ref_rng_create(seed)

    def __del__(self):
        try:
            self.lib.ref_rng_destroy(self.h)
        except Exception:
            pass

    def next(self) -> int:
        return int(self.lib.ref_rng_next(self.h))

    def random_instance(self, d, l, limit):
        q = np.empty(d, np.float64)
        k = np.empty((l, d), np.float64)
        v = np.empty((l, d), np.float64)
        s = C.c_double()
        self.lib.ref_random_instance(self.h, d, l, limit, ptr(q), ptr(k), ptr(v), C.byref(s))
        return q, k, v, s.value

    def random_partition(self, l, parts):
        part_of = np.empty(l, np.int64)
        self.lib.ref_random_partition(self.h, l, parts, ptr(part_of))
        return [np.nonzero(part_of == i)[0].astype(np.int64) for i in range(parts)]
