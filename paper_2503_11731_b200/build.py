"""Build libgsr.so (in-tree) with nvcc for sm_100a.

The shared library exports the C-ABI of include/gsr.h.  cudart is linked
statically; device memory and streams come from the caller (PyTorch).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "libgsr.so")
SOURCES = ["abi.cu", "project.cu", "sort.cu", "render.cu", "decode.cu", "route.cu", "backward.cu"]
HEADERS = ["gsr_internal.cuh", "scan.cuh", "binning.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-cudart", "static"]


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "gsr.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """(Re)build libgsr.so when forced or older than its sources.  Concurrent
    callers (e.g. the ranks of a torchrun job) serialise on a lock file, and
    the ones that wait find it fresh."""
    if not force and not _stale():
        return SO
    import fcntl
    with open(SO + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if not force and not _stale():
            return SO
        tmp = f"{SO}.{os.getpid()}.tmp"
        cmd = [NVCC] + FLAGS + (["-Xptxas", "-v"] if verbose else []) + ["-o", tmp] + \
            [os.path.join(CSRC, f) for f in SOURCES]
        r = subprocess.run(cmd, cwd=CSRC, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc failed building libgsr.so")
        if verbose:
            sys.stderr.write(r.stderr)
        os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
