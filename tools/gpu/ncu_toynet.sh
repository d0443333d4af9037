cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_uniform.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/launches_toynet.csv python tools/bench_toynet.py --n 65536 --reps 1 > gpurun_out/ncu_toynet.log 2>&1
tail -3 gpurun_out/ncu_toynet.log
