cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_toynet.py -q -rf --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_toynet.log 2>&1; echo "rc $?" >> gpurun_out/pytest_toynet.log
timeout 300 python tools/bench_toynet.py --n 65536 > gpurun_out/bench_toynet.log 2>&1
tail -30 gpurun_out/pytest_toynet.log; cat gpurun_out/bench_toynet.log | tail -5
