cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider > gpurun_out/pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "rc $?" >> gpurun_out/bench_default.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 300 python bench.py --config 2d_65536 --no-cpu-baseline > gpurun_out/bench_65k.log 2>&1
timeout 300 python bench.py --config 2d_262144 --no-cpu-baseline > gpurun_out/bench_262k.log 2>&1
timeout 300 python bench.py --config 2d_8192 --no-cpu-baseline > gpurun_out/bench_8k.log 2>&1
timeout 1500 python bench.py --config batch_262k --steps 1 --warmup 1 > gpurun_out/bench_batch.log 2>&1
timeout 1500 python bench.py --config part_16m --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_part16m.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_3d.csv python tools/iter_driver.py --reps 3 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_leaf_fast -s 1 -c 1 -o gpurun_out/prof_leaf python tools/iter_driver.py --reps 3 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_prolong_fast|k_spmv_tma|k_sums_tree|k_tiles_all" -s 4 -c 4 -o gpurun_out/prof_other python tools/iter_driver.py --reps 3 > gpurun_out/ncu_full2.log 2>&1
tail -2 gpurun_out/smoke.log; tail -6 gpurun_out/pytest.log; for f in gpurun_out/bench_*.log; do echo "== $f"; grep "^{" $f | cut -c1-250; done
