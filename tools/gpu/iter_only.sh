cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/iter_driver.py --reps 5 2>&1 | tail -1
