cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest.log
tail -6 gpurun_out/pytest.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "rc $?" >> gpurun_out/bench_default.log
grep "^{" gpurun_out/bench_default.log | cut -c1-300
