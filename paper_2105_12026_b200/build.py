"""Build libebc200.so in-tree with nvcc for sm_100a (no JIT cache, so the .so
travels with the repo snapshot to the GPU box)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libebc200.so")
SOURCES = ["ebc200.cu"]
HEADERS = ["kernels.cuh", "ptx.cuh", "screen_tc.cuh", "multiset.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "ebc200.h"))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build_native(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v", "-shared", "-Xcompiler", "-fPIC",
           "-o", LIB, *[os.path.join(CSRC, s) for s in SOURCES], "-ldl"]
    if os.path.exists(LIB):
        os.remove(LIB)  # a failed build must not leave a stale library behind
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + proc.stdout + proc.stderr)
    if verbose:
        sys.stdout.write(proc.stderr)
    return LIB


if __name__ == "__main__":
    print(build_native(force="--force" in sys.argv, verbose="-v" in sys.argv))
