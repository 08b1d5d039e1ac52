"""Build libtinyserve.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

Two artefacts from the same source: the release library libtinyserve.so (the product: fixed,
measured launch choices, no environment reads, no debug exports) and the dev library
libtinyserve_dev.so (-DTS_DEV_KNOBS: the A/B environment knobs of DESIGN.md §5, the
per-CTA timestamp hooks and the TS_DEBUG device error word).  Tests load the dev library
only in child processes that set TS_DEV_LIB=1 (tests/test_gpu_variants.py)."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libtinyserve.so")
DEV_LIB = os.path.join(HERE, "libtinyserve_dev.so")
SOURCES = [os.path.join(HERE, "csrc", "api.cu")]
DEPS = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu*")) +
              [os.path.join(ROOT, "include", "tinyserve.h")])
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    return "nvcc"


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, dev: bool = False) -> str:
    lib = DEV_LIB if dev else LIB
    if not force and not stale(lib):
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    extra = os.environ.get("TS_NVCC_EXTRA", "").split()  # development builds only
    cmd = [nvcc(), *NVCC_FLAGS, *(["-DTS_DEV_KNOBS"] if dev else []), *extra,
           *(["-Xptxas", "-v"] if verbose else []), *SOURCES, "-o", tmp]
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, dev="--dev" in sys.argv))
