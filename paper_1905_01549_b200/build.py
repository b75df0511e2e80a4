"""In-tree build of the native libraries (no JIT cache: the .so files travel to
the GPU box with the repo snapshot).

* ``libcgvk.so``     — the CUDA C-ABI library (include/cgvk.h), sm_100a only.
* ``libcgvkgen.so``  — host-only synthetic-input generators.
* ``cpp/cgv_shim_tests`` — the C++ ``cgv::`` shim's test driver (reference-style
  tests through the shim; run by tests/test_cpp_shim.py on a GPU box).
* ``oracle/``        — test infrastructure, built by ``oracle/Makefile``.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-std=c++17", "-O3", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC,-O2",
           "-Xptxas", "-warn-spills"]

CUDA_SOURCES = ["cgvk_api.cu"]
CUDA_DEPS = ["cgvk_api.cu", "cgvk_device.cuh", "cgvk_variants.cuh", "cgvk_generic.cuh",
             "cgvk_stream.cuh", "cgvk_dist.cuh", "cgvk_group.inc", "cgvk_band.cuh", "cgvk_run.inc"]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str], cwd: str | None = None) -> None:
    print("+", " ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=cwd)


def build_gen(force: bool = False) -> str:
    out = os.path.join(PKG, "libcgvkgen.so")
    deps = [os.path.join(CSRC, f) for f in ("cgvk_gen.c", "cgvk_gen.h")]
    if force or _stale(out, deps):
        _run(["gcc", "-std=gnu11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
              "-shared", "-o", out, os.path.join(CSRC, "cgvk_gen.c"), "-lm"])
    return out


def build_cuda(force: bool = False) -> str:
    out = os.path.join(PKG, "libcgvk.so")
    deps = [os.path.join(CSRC, f) for f in CUDA_DEPS] + [os.path.join(INCLUDE, "cgvk.h")]
    if force or _stale(out, deps):
        _run([NVCC, *ARCH, *NVFLAGS, "-I", INCLUDE, "-shared", "-o", out,
              *[os.path.join(CSRC, f) for f in CUDA_SOURCES], "-lcudart", "-lpthread"])
    return out


def build_cpp_shim(force: bool = False) -> str:
    cpp = os.path.join(PKG, "cpp")
    out = os.path.join(cpp, "cgv_shim_tests")
    src = os.path.join(cpp, "cgv_shim_tests.cpp")
    if not os.path.exists(src):
        return out
    deps = [src, os.path.join(INCLUDE, "cgvk.h")] + [
        os.path.join(cpp, "cgvariants", f) for f in os.listdir(os.path.join(cpp, "cgvariants"))]
    if force or _stale(out, deps):
        _run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I", cpp, "-I", INCLUDE, "-o", out,
              src, "-L", PKG, "-lcgvk", "-Wl,-rpath,$ORIGIN/.."])
    return out


def build_oracle(force: bool = False) -> None:
    oracle = os.path.join(ROOT, "oracle")
    flags = ["-B"] if force else []
    _run(["make", "-s", *flags, "-C", oracle, "restatement"])
    if os.path.isdir("/root/reference/proj/src"):
        _run(["make", "-s", *flags, "-C", oracle, "ref"])


def build_all(force: bool = False) -> None:
    build_gen(force)
    build_cuda(force)
    build_cpp_shim(force)
    build_oracle(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
