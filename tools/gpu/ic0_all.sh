#!/bin/bash
# IC(0)-PCG timings on every config (chunked sweeps, the default) -> gpurun_out/ic0_all.jsonl
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in 3d_1m 2d_262144 2d_65536 2d_8192; do
  timeout 400 python tools/bench_ic0.py --config $c --cpu-iters 10 >> gpurun_out/ic0_all.jsonl 2>>gpurun_out/ic0_all.err
done
cat gpurun_out/ic0_all.jsonl
