cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_toynet.py -q -x -rf --timeout 600 -p no:cacheprovider > gpurun_out/pytest_tn.log 2>&1; echo "rc $?" >> gpurun_out/pytest_tn.log
tail -25 gpurun_out/pytest_tn.log
timeout 300 python tools/bench_toynet.py --n 65536 > gpurun_out/bench_toynet.log 2>&1; tail -1 gpurun_out/bench_toynet.log
HFPG_ATTENTION_SIMT=1 timeout 300 python tools/bench_toynet.py --n 65536 > gpurun_out/bench_toynet_simt.log 2>&1; tail -1 gpurun_out/bench_toynet_simt.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_toynet.csv python tools/bench_toynet.py --n 65536 --reps 0 > gpurun_out/ncu_toynet.log 2>&1
