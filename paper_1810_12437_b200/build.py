"""Builds libpcgs.so (the CUDA kernels + C ABI) in-tree with nvcc for sm_100a.

The library is plain nvcc output (no torch extension machinery): its ABI is
declared in include/pcgs.h and bound with ctypes in _lib.py.
"""
from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libpcgs.so"
SOURCES = [CSRC / "pcgs.cu", CSRC / "gibbs.cu", CSRC / "sliced.cu", CSRC / "sliced.cpp", CSRC / "sgibbs.cu", CSRC / "rowsplit.cu", CSRC / "store.cpp", CSRC / "mtx.cpp"]
HEADERS = [CSRC / "store.h", CSRC / "mtx.h", CSRC / "device.cuh", CSRC / "internal.cuh", CSRC / "sliced.h", CSRC / "sliced.cuh", CSRC / "pg.cuh", CSRC / "gibbs_math.cuh",
           ROOT / "include" / "pcgs.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + HEADERS)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
           "-shared", "-I", str(ROOT / "include"), "-I", str(CSRC),
           "-Xptxas", "-v" if verbose else "-O3",
           "-o", str(LIB) + ".tmp", *map(str, SOURCES), "-lz"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    if verbose:
        print(res.stdout + res.stderr)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    import sys
    build_library(force=True, verbose="-v" in sys.argv)
    print(LIB)
