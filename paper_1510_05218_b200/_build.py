"""Build helpers: compile libthiim_gpu.so for sm_100a in-tree with nvcc.

The library is built IN-TREE (next to this file) so it travels to the GPU box
with the repo snapshot.  Flags: -fmad=false (no contraction anywhere; the
kernels additionally use explicit _rn intrinsics), -lineinfo for ncu source
pages, host code with -ffp-contract=off (the host generator must reproduce
the device one bitwise).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libthiim_gpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xptxas", "-v",
    "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off,-O2",
    "-shared",
]


def _sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
            if f.endswith((".cu", ".cuh", ".h"))] + \
           [os.path.join(HERE, "..", "include", "thiim_gpu.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in _sources())


def build(verbose: bool = False, force: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    # THIIM_NVCC_EXTRA: extra flags for experiments (e.g. -DTHIIM_RING_FENCE=1)
    extra = os.environ.get("THIIM_NVCC_EXTRA", "").split()
    cmd = [NVCC, *NVCC_FLAGS, *extra, "-o", LIB + ".tmp", os.path.join(CSRC, "thiim_gpu.cu"), "-lgomp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libthiim_gpu.so (see %s)" % log)
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        sys.stderr.write(r.stderr)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
