"""Builds libsplidar.so in-tree (paper_2509_20500_b200/lib/) for sm_100a with nvcc.

    python -m paper_2509_20500_b200.build [--force] [--verbose]

The library is linked against the static CUDA runtime (nvcc's default), so it loads without a
GPU; kernels are compiled only for sm_100a (B200) with -lineinfo for Nsight Compute's source page.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libsplidar.so")
INCLUDE = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(INCLUDE, "splidar.h")]


def nvcc_version() -> str:
    out = subprocess.check_output([NVCC, "--version"], text=True)
    for tok in out.replace(",", " ").split():
        if tok.startswith("V") and tok[1:2].isdigit():
            return tok[1:]
    return "unknown"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
           "-Xptxas", "-warn-spills", f"-DSPL_NVCC_VERSION=\"{nvcc_version()}\"", f"-I{INCLUDE}",
           "-o", tmp, *_sources()]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(p)
