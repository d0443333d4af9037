#!/bin/bash
# Development A/B: build paper_2605_13343_b200/variants/libhfpg_<name>.so with extra -D flags.
#   bash tools/build_variant.sh <name> -DPT_WARPS=8 -DPT_STAGES=4 -DPT_AUX=2
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2605_13343_b200"
mkdir -p variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 --extended-lambda -shared \
  -Xcompiler -fPIC,-O3,-march=x86-64-v3,-ffp-contract=fast "$@" -o variants/libhfpg_$name.so \
  csrc/hfpg_device.cu csrc/toynet.cu csrc/host_structure.cpp csrc/partition_host.cpp csrc/ic0_host.cpp -lz -lpthread
