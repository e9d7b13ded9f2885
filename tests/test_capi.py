"""The drop-in boundary without a GPU: the C-ABI library loads, exports every symbol the
header declares, the C++ drop-in exports the reference's disagg:: API, and the host-side
partitioners match the reference (golden fixtures from the reference's own code)."""
import ctypes as C
import subprocess

import numpy as np
import pytest


def test_core_library_exports_every_declared_symbol(built):
    lib = built.load()
    names = built.declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(built.SIGNATURES), "ctypes table out of sync with lamina_attn.h"
    assert lib.lam_version() >= 1


def test_dropin_library_exports_reference_api(built):
    out = subprocess.run(["nm", "-DC", "--defined-only", str(built.DROPIN_PATH)],
                         capture_output=True, text=True, check=True).stdout
    for sym in [
        "disagg::exact_attention<float>", "disagg::exact_attention<double>",
        "disagg::partial_attention<double>", "disagg::partial_attention<float>",
        "disagg::merge<double>", "disagg::finalize<double>", "disagg::split_prev_new<double>",
        "disagg::multi_head_attention<double>", "disagg::multi_head_attention<float>",
        "disagg::head_partition(long, long)", "disagg::request_partition(",
        "disagg::PartialAttention<double>::identity(long)",
        "disagg::MultiHeadInstance<double>::head_instance(long) const",
        "disagg::AttnInstance<double>::validate() const",
    ]:
        assert sym in out, sym
    deps = subprocess.run(["ldd", str(built.DROPIN_PATH)], capture_output=True, text=True).stdout
    assert "liblamina_attn.so" in deps


def test_head_partition_matches_reference(built, golden):
    from paper_2405_01814_b200 import attention as A

    g = golden("partition.npz")
    for nkv, ndev in [(8, 1), (8, 2), (8, 4), (8, 8), (32, 4)]:
        r = A.head_partition(nkv, ndev)
        assert [x for hr in r for x in (hr.begin, hr.end)] == list(g[f"hp_{nkv}_{ndev}"])
    with pytest.raises(A.ValidationError) as e:
        A.head_partition(8, 3)
    assert "divisible" in str(e.value)
    assert str(e.value) == str(g["hp_8_3_msg"])
    with pytest.raises(A.ValidationError):
        A.head_partition(0, 1)
    with pytest.raises(A.ValidationError):
        A.head_partition(8, 0)


def test_request_partition_matches_reference(built, golden):
    from paper_2405_01814_b200 import attention as A

    g = golden("partition.npz")
    sizes = g["rp_sizes"]
    for ndev in (1, 2, 3, 8):
        a = A.request_partition(sizes, ndev)
        assert a.device_of == list(g[f"rp_{ndev}_device_of"])
        assert np.array_equal(np.array(a.device_load), g[f"rp_{ndev}_load"])
        assert a.imbalance == float(g[f"rp_{ndev}_imbalance"])
    # test_attention.cpp:271-282 known answers
    assert A.request_partition([100.0] * 8, 4).imbalance == pytest.approx(1.0)
    a = A.request_partition([8192, 128, 128, 128], 2)
    assert a.imbalance == pytest.approx(8192.0 / 4288.0, rel=1e-12)
    assert a.device_load[a.device_of[0]] == 8192.0
    assert A.request_partition([512.0], 6).imbalance == pytest.approx(6.0)
    with pytest.raises(A.ValidationError):
        A.request_partition([1.0], 0)


def test_no_gpu_fails_loudly(built):
    """Without a device the library must refuse, never compute on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = built.load()
    h = C.c_void_p()
    rc = lib.lam_ctx_create(0, C.byref(h))
    assert rc != 0
    from paper_2405_01814_b200 import attention as A

    with pytest.raises(A.Error):
        A.exact_attention(A.AttnInstance(np.ones(4), np.ones((3, 4)), np.ones((3, 4)), 0.5))
