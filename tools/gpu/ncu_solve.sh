cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve -s 1 -c 1 -o gpurun_out/prof_solve_${CFG:-2d_65536} python tools/solve_driver.py --config ${CFG:-2d_65536} --max-iters 300 --reps 2 > gpurun_out/ncu_solve.log 2>&1
tail -3 gpurun_out/ncu_solve.log
