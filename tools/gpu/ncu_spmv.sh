cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spmv_tma|k_prolong_fast|k_sums_tree|k_tiles_all" -s 4 -c 4 -o gpurun_out/prof_r1b python tools/iter_driver.py --reps 3 > gpurun_out/ncu_r1b.log 2>&1
tail -3 gpurun_out/ncu_r1b.log
