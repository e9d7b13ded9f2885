"""Build the in-tree native libraries for sm_100a (B200).

    lib/liblamina_attn.so      CUDA kernels + the C-ABI of include/lamina_attn.h
    lib/libdisagg_attention.so the reference-API drop-in (include/disagg/attention.hpp)

nvcc cross-compiles here without a GPU; the .so files travel to the GPU box with the
repo snapshot.  Rebuilds only when a source or header is newer than its output.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"
OBJ = ROOT / "build" / "obj"
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-I", str(INCLUDE),
              "--expt-relaxed-constexpr"] + ARCH

CU_SOURCES = ["decode.cu", "instance.cu", "kv.cu", "capi.cu"]


def _newest(paths) -> float:
    return max((p.stat().st_mtime for p in paths if p.exists()), default=0.0)


def _headers():
    return list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.rglob("*.h*"))


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("command failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r


def _compile_cu(src: Path) -> Path:
    obj = OBJ / (src.stem + ".o")
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, _newest(_headers())):
        return obj
    _run([NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)])
    return obj


def build(verbose: bool = False) -> dict:
    LIB.mkdir(parents=True, exist_ok=True)
    OBJ.mkdir(parents=True, exist_ok=True)
    srcs = [CSRC / s for s in CU_SOURCES]
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(_compile_cu, srcs))
    core = LIB / "liblamina_attn.so"
    if not core.exists() or core.stat().st_mtime < _newest(objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(core), *map(str, objs), "-lcudart_static",
              "-lrt", "-ldl", "-lpthread"])
        if verbose:
            print("linked", core)
    dropin_src = PKG / "dropin" / "attention.cpp"
    dropin = LIB / "libdisagg_attention.so"
    if not dropin.exists() or dropin.stat().st_mtime < max(
            _newest([dropin_src, core]), _newest(list(INCLUDE.rglob("*.h*")))):
        _run([CXX, "-std=c++20", "-O2", "-fPIC", "-shared", "-I", str(INCLUDE), str(dropin_src),
              "-o", str(dropin), "-L", str(LIB), "-llamina_attn", "-Wl,-rpath,$ORIGIN"])
        if verbose:
            print("linked", dropin)
    bench_src = ROOT / "benchmarks" / "bench_attention_b200.cpp"
    bench_bin = ROOT / "benchmarks" / "bench_attention_b200"
    if bench_src.exists() and (not bench_bin.exists() or bench_bin.stat().st_mtime < max(
            _newest([bench_src, core, dropin]), _newest(list(INCLUDE.rglob("*.h*"))))):
        _run([NVCC, "-std=c++20", "-O2", *ARCH, "-I", str(INCLUDE), str(bench_src), "-o",
              str(bench_bin), "-L", str(LIB), "-ldisagg_attention", "-llamina_attn",
              "-Xlinker", "-rpath,$ORIGIN/../paper_2405_01814_b200/lib"])
        if verbose:
            print("linked", bench_bin)
    return {"core": str(core), "dropin": str(dropin), "bench": str(bench_bin)}


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
