cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leaf_coarse -s 1 -c 1 -o gpurun_out/prof_lc python tools/iter_driver.py --reps 2 > gpurun_out/ncu_lc.log 2>&1
tail -n 2 gpurun_out/ncu_lc.log
