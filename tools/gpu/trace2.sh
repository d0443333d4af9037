cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_persistent.py -x -q -rf --timeout 300 -p no:cacheprovider > gpurun_out/pytest_persist.log 2>&1; echo "rc $?" >> gpurun_out/pytest_persist.log
tail -3 gpurun_out/pytest_persist.log
for c in 2d_8192 2d_65536 2d_262144 3d_1m; do timeout 300 python tools/phase_trace.py --config $c; done > gpurun_out/trace.log 2>&1
for c in 2d_65536 3d_1m; do HFPG_NO_SPMV_TMA=1 timeout 300 python tools/phase_trace.py --config $c; done > gpurun_out/trace_direct.log 2>&1
