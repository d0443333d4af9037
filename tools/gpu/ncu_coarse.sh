cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 3d_1m 2d_262144; do
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__registers_per_thread --clock-control none --csv --log-file gpurun_out/launches_$c.csv python tools/iter_driver.py --config $c --reps 3 > gpurun_out/ncu_launch_$c.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tiles_all|k_sums_tree" -s 4 -c 2 -o gpurun_out/prof_coarse_1m python tools/iter_driver.py --config 3d_1m --reps 2 > gpurun_out/ncu_full_coarse.log 2>&1
tail -2 gpurun_out/ncu_full_coarse.log
