"""Builds libdouble_b200.so in-tree for sm_100a with nvcc (no JIT cache, no torch extension).

    python -m paper_2601_05524_b200.build   (or __graft_entry__.build())
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libdouble_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
         "-Xptxas", "-warn-spills"]


def _hash_inputs(src: str) -> str:
    h = hashlib.sha256()
    for f in [src] + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + \
            [os.path.join(ROOT, "include", "double_b200.h")]:
        h.update(open(f, "rb").read())
    h.update(" ".join(FLAGS + ARCH).encode())
    return h.hexdigest()[:16]


def _compile(src: str, verbose: bool) -> str:
    name = os.path.splitext(os.path.basename(src))[0]
    obj = os.path.join(OBJ, f"{name}-{_hash_inputs(src)}.o")
    if os.path.exists(obj):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip() and verbose:
        print(r.stderr, file=sys.stderr)
    os.replace(obj + ".tmp", obj)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    cmd = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-Xcompiler", "-fPIC",
           "-lcuda" if False else "-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(LIB + ".tmp", LIB)
    return LIB


CPP_TEST = os.path.join(ROOT, "build", "test_cpp_api")


def build_cpp_test() -> str:
    """tests/cpp/test_cpp_api.cpp against include/double_b200.hpp, linked to the in-tree library."""
    src = os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp")
    os.makedirs(os.path.dirname(CPP_TEST), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), src, "-o", CPP_TEST,
           "-L", PKG, "-ldouble_b200", f"-Wl,-rpath,{PKG}", "-Wl,-rpath,$ORIGIN/../paper_2601_05524_b200"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"C++ API test build failed:\n{r.stderr}")
    return CPP_TEST


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
