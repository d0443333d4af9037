"""Build the native library in-tree: paper_2605_13343_b200/libhfpg.so (sm_100a only).

nvcc compiles the CUDA kernels for `-gencode arch=compute_100a,code=sm_100a` and the host C++
(C ABI, generators, HFTC I/O) with the same FMA-contraction settings as the reference's
`-O3 -march=native` gnu++20 build, so the host generators stay bit-identical to it.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libhfpg.so")
SRCS = ["csrc/hfpg_device.cu", "csrc/toynet.cu", "csrc/train_loop.cu", "csrc/host_structure.cpp",
        "csrc/partition_host.cpp", "csrc/ic0_host.cpp"]
DEPS = SRCS + ["csrc/kernels.cuh", "csrc/device_common.cuh", "csrc/internal.hpp", "csrc/pcg_exact.cuh",
               "csrc/gemm_tcgen05.cuh", "csrc/gemm_persistent.cuh", "csrc/attention_tcgen05.cuh", "csrc/leaf_coarse.cuh", "csrc/solve_persistent.cuh", "csrc/comm.cuh", "csrc/partition_host.hpp", "csrc/framegen.cuh", "csrc/crmath.cuh", "csrc/toynet_kernels.cuh", "csrc/ic0.cuh", "csrc/crc32.cuh", "csrc/io_device.cuh", "csrc/train.cuh",
               "../include/hfpg.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(os.path.join(HERE, d)) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return SO
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3",
           "-std=c++17", "--extended-lambda", "-shared", "-Xcompiler", "-fPIC,-O3,-march=x86-64-v3,-ffp-contract=fast",
           "-o", SO + ".tmp", *[os.path.join(HERE, s) for s in SRCS], "-lz", "-lpthread"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, cwd=HERE, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc build of libhfpg.so failed")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO)
