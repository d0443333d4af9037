#!/bin/bash
# IC(0) sweeps: parity tests, then chunked (default) vs per-row (HFPG_IC0_ROWS) timings.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ic0.py -x -q -m gpu > gpurun_out/ic0_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ic0_tests.log
for c in 2d_65536 3d_1m; do
  timeout 300 python tools/bench_ic0.py --config $c --cpu-iters 3 >> gpurun_out/ic0_ab.jsonl 2>>gpurun_out/ic0_ab.err
  HFPG_IC0_ROWS=1 timeout 300 python tools/bench_ic0.py --config $c --cpu-iters 3 | sed 's/^{/{"rows": 1, /' >> gpurun_out/ic0_ab.jsonl 2>>gpurun_out/ic0_ab.err
done
tail -3 gpurun_out/ic0_tests.log; cat gpurun_out/ic0_ab.jsonl
