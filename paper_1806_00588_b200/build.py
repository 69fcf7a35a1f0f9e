"""Builds the in-tree libraries:

* paper_1806_00588_b200/liblshbeam_b200.so -- the CUDA kernels + C ABI
  (include/lshbeam_b200.h);
* paper_1806_00588_b200/liblshbeam.so -- the C++ drop-in API
  (include/lshbeam/*.hpp, namespace lshbeam) over that C ABI, so C++ callers
  of the reference library (its CLI, bench and test suites) link against the
  GPU build unchanged.


Explicit nvcc for sm_100a only (no PTX fallback, no other arch): every .cu
under csrc/ is compiled to an object with -lineinfo (ncu source view) and
linked into one shared library exporting the C ABI of include/lshbeam_b200.h.
The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import re
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "liblshbeam_b200.so")
CPP = os.path.join(PKG, "cpp")
CPPLIB = os.path.join(PKG, "liblshbeam.so")
CXX = os.environ.get("CXX_DROPIN", "/usr/bin/g++")
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-I" + os.path.join(ROOT, "include")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                "-I" + os.path.join(ROOT, "include"), "-I" + CSRC,
                "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps)


def _included_sources(src: str):
    """The .cu files a source #includes (k_step_fused.cu: the kernel bodies)."""
    with open(src) as f:
        names = re.findall(r'^#include "([^"]+\.cu)"', f.read(), re.M)
    return [os.path.join(os.path.dirname(src), n) for n in names]


def _compile(src: str, headers) -> str:
    obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
    if _newer(obj, [src, *headers, *_included_sources(src), __file__]):
        return obj
    cmd = [NVCC, *FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + sorted(
        glob.glob(os.path.join(CSRC, "*.h"))) + [
        os.path.join(ROOT, "include", "lshbeam_b200.h")]
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, headers), srcs))
    if not _newer(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static", "-lrt", "-ldl",
               "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    build_cpp()
    build_cli()
    if verbose:
        print(LIB)
        print(CPPLIB)
    return LIB


def build_cpp() -> str:
    """The C++ drop-in layer: g++ (C++20, like the reference) over cpp/*.cpp,
    linked against liblshbeam_b200.so with an $ORIGIN rpath."""
    srcs = sorted(glob.glob(os.path.join(CPP, "*.cpp")))
    deps = srcs + sorted(glob.glob(os.path.join(CPP, "*.hpp"))) + sorted(
        glob.glob(os.path.join(ROOT, "include", "lshbeam", "*.hpp"))) + [
        os.path.join(ROOT, "include", "lshbeam_b200.h"), LIB, __file__]
    if _newer(CPPLIB, deps):
        return CPPLIB
    cmd = [CXX, *CXXFLAGS, "-shared", "-o", CPPLIB, *srcs, "-L" + PKG, "-llshbeam_b200",
           "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"C++ drop-in build failed:\n{r.stderr}")
    return CPPLIB


CLI_SRC = os.path.join(PKG, "cli", "lshbeam_main.cpp")
CLI_BIN = os.path.join(PKG, "lshbeam")
JSON_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"


def build_cli() -> str | None:
    """The `lshbeam` CLI (build/decode/grid) over liblshbeam.so. Needs
    nlohmann/json (vendored by cudnn-frontend in this image); skipped if absent."""
    if not os.path.exists(os.path.join(JSON_INC, "json.hpp")):
        return None
    deps = [CLI_SRC, CPPLIB, __file__]
    if _newer(CLI_BIN, deps):
        return CLI_BIN
    cmd = [CXX, *CXXFLAGS, "-I" + JSON_INC, "-o", CLI_BIN, CLI_SRC, "-L" + PKG, "-llshbeam",
           "-llshbeam_b200", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"CLI build failed:\n{r.stderr}")
    return CLI_BIN


if __name__ == "__main__":
    build(verbose=True)
