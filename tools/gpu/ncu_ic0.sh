#!/bin/bash
# ncu launch list of one IC(0)-PCG iteration's kernels (3D 1M) + a full capture of the forward sweep
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_ic0|k_spmv" -c 12 --csv --log-file gpurun_out/ic0_launches.csv python tools/bench_ic0.py --config 3d_1m --steps 1 --cpu-iters 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ic0_forward_chunk -s 2 -c 1 -o gpurun_out/prof_ic0 python tools/bench_ic0.py --config 3d_1m --steps 1 --cpu-iters 1 > /dev/null 2>&1
ls -la gpurun_out/ | grep -i ic0
