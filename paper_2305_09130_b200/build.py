"""Builds the in-tree CUDA library libmctune_b200.so for sm_100a with nvcc.

Usage: python -m paper_2305_09130_b200.build [--force]
The .so lands next to this file (git-ignored; travels to the GPU box with the
gpurun snapshot).  No JIT cache is used.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("MCTB_BUILD_OUT") or os.path.join(HERE, "libmctune_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O2",
         "-Xlinker", "--no-undefined",
         "-cudart", "static", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def sources() -> list[str]:
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def deps() -> list[str]:
    out = []
    for d in (CSRC, os.path.join(HERE, "..", "include")):
        for f in os.listdir(d):
            if f.endswith((".cu", ".cuh", ".h", ".hpp")):
                out.append(os.path.join(d, f))
    return out


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    extra = os.environ.get("MCTB_NVCC_EXTRA", "").split()  # experiments (e.g. -DMCTB_BFS_MINB=5)
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-o", LIB + ".tmp", *sources()]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libmctune_b200.so")
    if verbose:
        sys.stderr.write(r.stderr)
    with open(os.path.join(HERE, "ptxas.log"), "w") as f:
        f.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
