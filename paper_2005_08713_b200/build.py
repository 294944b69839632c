"""Build the sm_100a shared library in-tree (nvcc, -gencode arch=compute_100a,code=sm_100a)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = [os.path.join(HERE, "csrc", f) for f in ("dwt.cu", "encode.cu", "decode.cu", "truncate.cu", "archive.cu", "capi.cu")]
HDRS = [os.path.join(HERE, "csrc", f) for f in ("common.cuh", "coder.cuh")] + [
    os.path.join(os.path.dirname(HERE), "include", "wbpc_b200.h")]
OUT = os.path.join(HERE, "libwbpc_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-shared", "--use_fast_math"]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(p) <= t for p in SRC + HDRS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    extra = os.environ.get("WBPC_NVCC_EXTRA", "").split()
    cmd = [NVCC] + FLAGS + extra + (["-Xptxas", "-v"] if verbose else []) + ["-o", OUT] + SRC
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
