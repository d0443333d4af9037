#!/bin/bash
# GPU frame generator: parity tests + timing
mkdir -p gpurun_out
python -m pytest tests/test_gpu_framegen.py -x -q 2>&1 | tail -15 > gpurun_out/framegen_tests.txt
timeout 600 python tools/framegen_bench.py --reps 5 > gpurun_out/framegen_bench.jsonl 2> gpurun_out/framegen_bench.err
cat gpurun_out/framegen_tests.txt gpurun_out/framegen_bench.jsonl; tail -5 gpurun_out/framegen_bench.err
