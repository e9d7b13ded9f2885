"""Pin the CPU oracle before trusting it: our C restatement (oracle/attn_oracle.c) must equal
the reference's own attention.cpp bit for bit — on the committed golden fixtures (generated
from the reference, oracle/make_golden.py) and, where oracle/_ref was built, on fresh draws
of the reference's own test generators."""
import numpy as np
import pytest

from oracle import oracle as O


@pytest.mark.parametrize("name", ["instances_seed42.npz", "instances_seed7.npz",
                                  "instances_seed3.npz"])
def test_port_matches_reference_fixtures_bitwise(golden, name):
    g = golden(name)
    for i in range(g["q"].shape[0]):
        q, k, v, s = g["q"][i], g["k"][i], g["v"][i], float(g["scale"][i])
        out = O.exact(q, k, v, s)
        assert np.array_equal(out, g["exact"][i])
        acc, mx, ld, cnt = O.partial(q, k, v, s, np.arange(k.shape[0]))
        assert np.array_equal(acc, g["acc"][i])
        assert mx == g["max_logit"][i] and ld == g["log_denom"][i] and cnt == k.shape[0]
        # the long-double oracle (tests/oracles.hpp:15-38) agrees within the reference's 1e-6
        naive = O.naive(q, k, v, s)
        rel = np.max(np.abs(out - naive) / np.maximum(np.abs(naive), 1e-12))
        assert rel <= 1e-6


def test_port_merge_trees_match_reference(golden):
    g = golden("merge_trees_seed6.npz")
    for i in range(int(g["n"])):
        q, k, v, s = g[f"q_{i}"], g[f"k_{i}"], g[f"v_{i}"], float(g[f"scale_{i}"])
        part_of = g[f"part_of_{i}"]
        acc = (np.zeros(q.size), -np.inf, -np.inf, 0)
        for p in range(int(part_of.max()) + 1):
            acc = O.merge(acc, O.partial(q, k, v, s, np.nonzero(part_of == p)[0]))
        tree = O.finalize(acc)
        assert np.array_equal(tree, g[f"tree_{i}"])
        assert np.array_equal(O.exact(q, k, v, s), g[f"exact_{i}"])


@pytest.mark.parametrize("name", ["decode_mha_f32.npz", "decode_gqa_bf16.npz"])
def test_port_decode_matches_reference_fixtures(golden, name):
    g = golden(name)
    out32 = O.decode_dense(g["q"], g["k"], g["v"], g["lens"], float(g["scale"]))
    assert np.array_equal(out32, g["out_f32"])
    out64 = O.decode_dense(g["q"], g["k"], g["v"], g["lens"], float(g["scale"]), compute_f64=True)
    assert np.allclose(out64, g["out_f64"], rtol=0, atol=1e-7)


def test_identity_and_empty_semantics():
    q = np.array([0.5, -0.25]); k = np.array([[1.0, 2.0]]); v = np.array([[3.0, -4.0]])
    # l = 1 returns the value row exactly (test_attention.cpp:24-29)
    assert np.array_equal(O.exact(q, k, v, 0.7), v[0])
    empty = O.partial(q, k, v, 0.7, np.zeros(0, np.int64))
    assert empty[3] == 0 and empty[1] == -np.inf and empty[2] == -np.inf
    p = O.partial(q, k, v, 0.7, np.array([0]))
    m = O.merge(p, empty)
    assert np.array_equal(m[0], p[0]) and m[1:] == p[1:]
    with pytest.raises(IndexError):
        O.partial(q, k, v, 0.7, np.array([1]))
    with pytest.raises(RuntimeError):
        O.finalize(empty)


def test_page_scatter_gather_roundtrip():
    rng = np.random.default_rng(0)
    B, Hkv, P, rb, lmax = 3, 2, 16, 32, 70
    lens = np.array([70, 1, 33], np.int32)
    pages = -(-lens // P)
    perm = rng.permutation(int(pages.sum()) + 4).astype(np.int32)
    pt = np.zeros((B, int(pages.max())), np.int32)
    o = 0
    for b in range(B):
        pt[b, : pages[b]] = perm[o: o + pages[b]]
        o += pages[b]
    dense = rng.integers(0, 256, (B, Hkv, lmax, rb), dtype=np.uint8)
    for b in range(B):
        dense[b, :, lens[b]:] = 0
    pool = O.page_scatter(dense, pt, lens, perm.size, P)
    assert np.array_equal(O.page_gather(pool, pt, lens, lmax), dense)


ref_only = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@ref_only
def test_port_equals_reference_on_fresh_generator_draws():
    rng = O.RefRng(20240809)
    for _ in range(200):
        d = 1 + rng.next() % 64
        l = 1 + rng.next() % 255
        q, k, v, s = rng.random_instance(d, l, 80.0)
        assert np.array_equal(O.exact(q, k, v, s), O.exact(q, k, v, s, lib="ref"))
        for dt in (np.float32,):
            a = O.exact(q.astype(dt), k.astype(dt), v.astype(dt), s)
            b = O.exact(q.astype(dt), k.astype(dt), v.astype(dt), s, lib="ref")
            assert np.array_equal(a, b)
        idx = np.nonzero(np.arange(l) % 3 == rng.next() % 3)[0]
        pa, pb = O.partial(q, k, v, s, idx), O.partial(q, k, v, s, idx, lib="ref")
        assert np.array_equal(pa[0], pb[0]) and pa[1:] == pb[1:]


@ref_only
def test_reference_suite_passes_against_reference_itself():
    import subprocess

    r = subprocess.run([str(O.REF_TEST_REF)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "15 passed | 0 failed" in r.stdout
