"""In-tree build of the sm_100a library (no JIT cache: the .so travels with the repo).

``python paper_2206_07244_b200/build.py`` compiles ``csrc/capi.cu`` (which includes
every kernel) into ``paper_2206_07244_b200/lib/libspgemm_b200.so``.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libspgemm_b200.so")
SOURCES = [os.path.join(CSRC, "capi.cu")]
CXX_SOURCES = [os.path.join(CSRC, "cxx_api.cpp"), os.path.join(CSRC, "multi.cpp")]  # the reference's C++ API over the C ABI
HEADERS = [os.path.join(ROOT, "include", "spgemm_capi.h")] + [
    os.path.join(ROOT, "include", "spgemm", h) for h in sorted(os.listdir(os.path.join(ROOT, "include", "spgemm")))]
DEPS = SOURCES + CXX_SOURCES + HEADERS + [os.path.join(CSRC, h) for h in ("kernels.cuh", "kernels_heap.cuh", "kernels_coo.cuh")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-fmad=false",  # keep products and sums as separate roundings (value parity)
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    objs = []
    for src in CXX_SOURCES:
        obj = os.path.join(LIBDIR, os.path.basename(src) + ".o")
        cc = ["g++", "-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
              "-c", src, "-o", obj]
        r = subprocess.run(cc, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"g++ failed on {src}")
        objs.append(obj)
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", LIB, *SOURCES, *objs]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(LIBDIR, "ptxas.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed ({res.returncode}); see {log}")
    if verbose:
        sys.stdout.write(res.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
