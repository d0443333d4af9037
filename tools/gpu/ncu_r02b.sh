# round 2 final ncu evidence for the solve: the four iteration kernels (--set full, standalone
# launches), the in-graph whole-solve DRAM (--graph-profiling graph), the bench launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/prof_*.ncu-rep gpurun_out/launches_*.csv
for k in k_spmv_tma k_leaf_fast k_coarse_coop k_prolong_tma; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k python tools/iter_driver.py --reps 3 > gpurun_out/ncu_$k.log 2>&1
  echo "$k: $(grep -c Report gpurun_out/ncu_$k.log)"
done
timeout 600 ncu --graph-profiling graph --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv --log-file gpurun_out/graph_solve.csv python tools/solve_driver.py --config 3d_1m --max-iters 100 --reps 1 --graph > gpurun_out/ncu_graph.log 2>&1
echo "graph rc $?"; tail -3 gpurun_out/graph_solve.csv
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_3d.csv python bench.py --steps 1 --warmup 1 --no-parity --no-cpu-baseline --no-inference > gpurun_out/ncu_bench.log 2>&1
echo "bench launches rc $?"
