"""Build libgts.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgts.so")
SOURCES = ["engine.cu", "builder.cpp"]
HEADERS = ["kernels.cuh", "tcgen05.cuh", "sharded.cuh", "devbuild.cuh", "updates.cuh", "common.h", os.path.join("..", "..", "include", "gts.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off,-O3",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = SOURCES + HEADERS
    return any(os.path.getmtime(os.path.join(CSRC, d)) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-shared", "-o", LIB, *[os.path.join(CSRC, s) for s in SOURCES], "-lgomp"]
    env = dict(os.environ)
    env["PATH"] = "/usr/bin:" + env.get("PATH", "")   # system gcc (has libgomp)
    proc = subprocess.run(cmd, cwd=CSRC, env=env, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("nvcc build of libgts.so failed")
    if verbose:
        sys.stderr.write(proc.stderr)
    with open(os.path.join(HERE, "ptxas.log"), "w") as fh:
        fh.write(proc.stderr)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="-v" in sys.argv)
    print(LIB)
