cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sums_tree -s 1 -c 1 -o gpurun_out/prof_sums_1m python tools/iter_driver.py --config 3d_1m --reps 3 > gpurun_out/ncu_sums.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tiles_all -s 1 -c 1 -o gpurun_out/prof_tiles_1m python tools/iter_driver.py --config 3d_1m --reps 3 > gpurun_out/ncu_tiles.log 2>&1
tail -n 2 gpurun_out/ncu_sums.log; tail -n 2 gpurun_out/ncu_tiles.log
