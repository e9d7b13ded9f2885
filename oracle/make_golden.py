"""Generate tests/golden/*.npz from the REFERENCE implementation itself.

Runs only where /root/reference exists (this build container): it loads
oracle/_ref/libref_attn.so (the reference's attention.cpp compiled by oracle/Makefile) and
its own test generators (tests/generators.hpp, std::mt19937_64), and records inputs and the
reference's outputs as small fixtures.  The GPU box never regenerates them; tests read the
committed .npz files.  TEST INFRASTRUCTURE ONLY.

    python -m oracle.make_golden
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from oracle import oracle as O

GOLDEN = Path(__file__).resolve().parent.parent / "tests" / "golden"


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 to the nearest bf16 value (ties to even), returned as fp32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def instances(seed: int, trials: int, d: int, l: int, limit: float):
    """random_instance cases exactly as test_attention.cpp draws them, with the reference's
    exact_attention<double>, partial over all tokens, and the long-double oracle."""
    rng = O.RefRng(seed)
    qs, ks, vs, sc, ex, acc, mx, ld = [], [], [], [], [], [], [], []
    for _ in range(trials):
        q, k, v, s = rng.random_instance(d, l, limit)
        qs.append(q); ks.append(k); vs.append(v); sc.append(s)
        ex.append(O.exact(q, k, v, s, lib="ref"))
        a, m, g, _ = O.partial(q, k, v, s, np.arange(l), lib="ref")
        acc.append(a); mx.append(m); ld.append(g)
    return dict(q=np.array(qs), k=np.array(ks), v=np.array(vs), scale=np.array(sc),
                exact=np.array(ex), acc=np.array(acc), max_logit=np.array(mx),
                log_denom=np.array(ld))


def merge_trees(seed: int, trials: int):
    """test_attention.cpp:99-130 style random partitions: reference partials per part and
    the left-fold merge, finalized."""
    rng = O.RefRng(seed)
    rec = []
    for _ in range(trials):
        d = 1 + rng.next() % 64
        l = 2 + rng.next() % 255
        parts = 2 + rng.next() % 7
        q, k, v, s = rng.random_instance(d, l, 80)
        part = rng.random_partition(l, parts)
        acc = (np.zeros(d), -np.inf, -np.inf, 0)
        for p in part:
            acc = O.merge(acc, O.partial(q, k, v, s, p, lib="ref"), lib="ref")
        out = np.empty(d)
        O.ref().ref_finalize_f64(d, O.ptr(acc[0]), acc[2], acc[3], O.ptr(out))
        part_of = np.zeros(l, np.int64)
        for i, p in enumerate(part):
            part_of[p] = i
        rec.append((q, k, v, s, part_of, out, O.exact(q, k, v, s, lib="ref")))
    return rec


def decode_case(rng: np.random.Generator, B, Hq, Hkv, D, lens, bf16: bool):
    lmax = int(max(lens))
    q = rng.uniform(-1, 1, (B, Hq, D)).astype(np.float32)
    k = rng.uniform(-1, 1, (B, Hkv, lmax, D)).astype(np.float32)
    v = rng.uniform(-1, 1, (B, Hkv, lmax, D)).astype(np.float32)
    if bf16:
        q, k, v = bf16_round(q), bf16_round(k), bf16_round(v)
    scale = np.float32(1.0 / np.sqrt(D))
    out32 = np.zeros_like(q)
    out64 = np.zeros((B, Hq, D), np.float64)
    G = Hq // Hkv
    for b in range(B):
        for h in range(Hq):
            l = int(lens[b])
            kb, vb = k[b, h // G, :l], v[b, h // G, :l]
            out32[b, h] = O.exact(q[b, h], kb, vb, float(scale), lib="ref")
            out64[b, h] = O.exact(q[b, h].astype(np.float64), kb.astype(np.float64),
                                  vb.astype(np.float64), float(scale), lib="ref")
    return dict(q=q, k=k, v=v, lens=np.asarray(lens, np.int32), scale=np.float32(scale),
                out_f32=out32, out_f64=out64)


def main():
    GOLDEN.mkdir(parents=True, exist_ok=True)
    # test_attention.cpp:48-55 (seed 42, d=8, l=16, logits +-10) and :132-143 (seed 7, +-80)
    np.savez_compressed(GOLDEN / "instances_seed42.npz", **instances(42, 50, 8, 16, 10.0))
    np.savez_compressed(GOLDEN / "instances_seed7.npz", **instances(7, 50, 8, 64, 80.0))
    np.savez_compressed(GOLDEN / "instances_seed3.npz", **instances(3, 20, 16, 64, 40.0))
    rec = merge_trees(6, 12)
    np.savez_compressed(
        GOLDEN / "merge_trees_seed6.npz",
        **{f"{name}_{i}": val for i, r in enumerate(rec)
           for name, val in zip(("q", "k", "v", "scale", "part_of", "tree", "exact"), r)},
        n=np.array(len(rec)))
    rng = np.random.default_rng(20240809)
    np.savez_compressed(GOLDEN / "decode_mha_f32.npz",
                        **decode_case(rng, 2, 4, 4, 128, [37, 64], bf16=False))
    np.savez_compressed(GOLDEN / "decode_gqa_bf16.npz",
                        **decode_case(rng, 2, 16, 2, 128, [100, 129], bf16=True))
    # partitioning known answers
    hp = {}
    for nkv, ndev in [(8, 1), (8, 2), (8, 4), (8, 8), (32, 4), (8, 3)]:
        r = np.zeros(2 * ndev, np.int64)
        msg = C.create_string_buffer(256)
        rc = O.ref().ref_head_partition(nkv, ndev, O.ptr(r), msg, 256)
        hp[f"hp_{nkv}_{ndev}"] = r if rc == 0 else np.array([-1])
        if rc:
            hp[f"hp_{nkv}_{ndev}_msg"] = np.array(msg.value.decode())
    sizes = np.random.default_rng(5).lognormal(7, 1, 37)
    for ndev in (1, 2, 3, 8):
        dev = np.zeros(sizes.size, np.int64)
        load = np.zeros(ndev)
        imb = C.c_double()
        O.ref().ref_request_partition(O.ptr(sizes), sizes.size, ndev, O.ptr(dev), O.ptr(load),
                                      C.byref(imb))
        hp[f"rp_{ndev}_device_of"] = dev
        hp[f"rp_{ndev}_load"] = load
        hp[f"rp_{ndev}_imbalance"] = np.array(imb.value)
    hp["rp_sizes"] = sizes
    np.savez_compressed(GOLDEN / "partition.npz", **hp)
    for f in sorted(GOLDEN.glob("*.npz")):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
