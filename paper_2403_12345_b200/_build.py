"""Build libemc.so in-tree for sm_100a (nvcc; no GPU needed to compile).

    python -m paper_2403_12345_b200._build [--force]

Flags: -fmad=false is part of the bit-exactness contract (the reference's
numba code never contracts a*b+c); -lineinfo maps ncu source views.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "emc_engine.cu")
OUT = os.path.join(HERE, "libemc.so")
DEPS = [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))] + \
    [os.path.join(HERE, "..", "include", "emc.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
              "-diag-suppress", "550"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines=()) -> str:
    if not force and os.path.exists(out):
        t = os.path.getmtime(out)
        if all(os.path.getmtime(d) <= t for d in DEPS if os.path.exists(d)):
            return out
    tmp = out + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-o", tmp, SRC]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
