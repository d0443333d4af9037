#!/bin/bash
# Bit-exact PCG: parity tests, then its cost against the graph solve -> gpurun_out/exact.jsonl
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_exact.py -q -m gpu 2>&1 | tail -3
for p in factor ic0 jacobi; do timeout 900 python tools/bench_exact.py --config 3d_1m --precond $p >> gpurun_out/exact.jsonl 2>>gpurun_out/exact.err; done
timeout 600 python tools/bench_exact.py --config 2d_65536 --precond factor >> gpurun_out/exact.jsonl 2>>gpurun_out/exact.err
cat gpurun_out/exact.jsonl; tail -3 gpurun_out/exact.err
