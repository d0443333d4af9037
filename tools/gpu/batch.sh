cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_async.py tests/test_gpu_pcg.py -q -x -rf --timeout 300 -p no:cacheprovider > gpurun_out/pytest_async.log 2>&1; echo "rc $?" >> gpurun_out/pytest_async.log
tail -3 gpurun_out/pytest_async.log
timeout 1500 python bench.py --config batch_262k --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_batch.log 2>&1
grep "^{" gpurun_out/bench_batch.log | cut -c1-300
