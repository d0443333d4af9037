cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc $?" >> gpurun_out/bench_default.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc $?" >> gpurun_out/bench_ref.log
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt
tail -4 gpurun_out/pytest.log; cat gpurun_out/bench_default.log | cut -c1-400; cat gpurun_out/bench_ref.log | cut -c1-300; cat gpurun_out/host.txt
