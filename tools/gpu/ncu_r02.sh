# round 2 ncu evidence: solve kernels (--set full, standalone launches), in-graph whole-solve
# metrics (--graph-profiling graph), bench launch list; toynet kernels with tensor-pipe activity
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/prof_*.ncu-rep gpurun_out/launches_*.csv
for k in k_spmv_tma k_leaf_fast k_sums_tree k_tiles_all k_prolong_fast; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_$k python tools/iter_driver.py --reps 3 > gpurun_out/ncu_$k.log 2>&1
  echo "$k: $(grep -c Report gpurun_out/ncu_$k.log)"
done
timeout 600 ncu --graph-profiling graph --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv --log-file gpurun_out/graph_solve.csv python tools/solve_driver.py --config 3d_1m --max-iters 100 --reps 1 --graph > gpurun_out/ncu_graph.log 2>&1
echo "graph rc $?"; tail -3 gpurun_out/graph_solve.csv
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_3d.csv python bench.py --steps 1 --warmup 1 --no-parity --no-cpu-baseline --no-inference > gpurun_out/ncu_bench.log 2>&1
echo "bench launches rc $?"
timeout 900 ncu --clock-control none --kernel-name-base demangled -k "regex:pgemm|attn_tc" --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --csv --log-file gpurun_out/toynet_tc.csv python tools/bench_toynet.py --n 65536 --reps 0 > gpurun_out/ncu_tn_tc.log 2>&1
echo "toynet tc rc $?"
