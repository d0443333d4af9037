cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest.log
timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --config 2d_65536 > gpurun_out/bench65k.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_3d.csv python tools/iter_driver.py --reps 3 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_leaf_fast -s 3 -c 1 -o gpurun_out/prof_leaf python tools/iter_driver.py --reps 2 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_coarse -s 3 -c 1 -o gpurun_out/prof_coarse python tools/iter_driver.py --reps 2 > gpurun_out/ncu_full2.log 2>&1
tail -2 gpurun_out/smoke.log; tail -6 gpurun_out/pytest.log; cut -c1-600 gpurun_out/bench.log; tail -3 gpurun_out/ncu_launch.log
