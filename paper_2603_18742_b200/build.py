"""Build libdmpq.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2603_18742_b200.build

The product library links the CUDA runtime statically, so it loads on a CPU-only
machine (for the ABI-export tests) and on the B200 box without extra paths.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdmpq.so")
SOURCES = ["host.cu", "quant.cu", "quant_tma.cu", "quant_had.cu", "pack.cu", "cast.cu", "tdc.cu", "gemm.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",                   # parity: every float op rounds as written
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden",
    "-cudart", "static",
    "-DDMPQ_BUILD",
]


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "dmpq.h"))
    if not force and os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(d) for d in deps):
        return LIB
    extra = os.environ.get("DMPQ_NVCC_EXTRA", "").split()   # development experiments (e.g. -DQUANT_CH32_REGS=96)
    cmd = [NVCC, *FLAGS, *extra, "-shared", "-o", LIB, *srcs, "-ldl"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
