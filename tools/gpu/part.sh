cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_partition.py tests/test_gpu_persistent.py tests/test_gpu_pcg.py tests/test_gpu_apply.py -q -rf --timeout 400 -p no:cacheprovider > gpurun_out/pytest_part.log 2>&1; echo "rc $?" >> gpurun_out/pytest_part.log
tail -25 gpurun_out/pytest_part.log
