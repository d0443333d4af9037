cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_partition.py tests/test_gpu_pcg.py tests/test_gpu_apply.py tests/test_gpu_persistent.py -q -x -rf --timeout 300 -p no:cacheprovider > gpurun_out/pytest_c.log 2>&1; echo "rc $?" >> gpurun_out/pytest_c.log
tail -4 gpurun_out/pytest_c.log
for c in 3d_1m 2d_262144; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python tools/iter_driver.py --config $c --reps 3 > gpurun_out/ncu_launch_$c.log 2>&1
done
timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/b_3d1m.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --config 2d_262144 > gpurun_out/b_262k.log 2>&1
grep -h "^{" gpurun_out/b_3d1m.log gpurun_out/b_262k.log | cut -c1-160
