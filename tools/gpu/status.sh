cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config 2d_65536 > gpurun_out/bench65k.log 2>&1
timeout 300 python tools/bench_toynet.py --n 65536 > gpurun_out/bench_toynet.log 2>&1
tail -3 gpurun_out/smoke.log; tail -15 gpurun_out/pytest.log; cut -c1-400 gpurun_out/bench.log; cut -c1-400 gpurun_out/bench65k.log; tail -3 gpurun_out/bench_toynet.log
