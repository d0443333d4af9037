# L2 reuse of the bridges between the leaf kernel and the prolongation: ncu with the caches NOT
# flushed between kernels (--cache-control none), per bridge policy of the leaf kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for arm in ${ARMS:-last first tail10 tail20 tail30}; do
  unset HFPG_BRIDGE_FIRST HFPG_BRIDGE_TAIL HFPG_L2_PERSIST_MB HFPG_L2_WINDOW_MB
  case $arm in w*) export HFPG_L2_PERSIST_MB=80 HFPG_L2_WINDOW_MB=${arm#w};; first) export HFPG_BRIDGE_FIRST=1;; tail*) export HFPG_BRIDGE_TAIL=${arm#tail};; p*t*) export HFPG_L2_PERSIST_MB=${arm%t*}; export HFPG_L2_PERSIST_MB=${HFPG_L2_PERSIST_MB#p}; export HFPG_BRIDGE_TAIL=${arm#*t};; p*) export HFPG_L2_PERSIST_MB=${arm#p};; esac
  timeout 600 ncu --cache-control none --clock-control none -k "regex:k_leaf_fast|k_prolong|k_spmv|k_tiles|k_sums" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv --log-file gpurun_out/l2_$arm.csv python tools/iter_driver.py --reps 3 > gpurun_out/l2_$arm.log 2>&1
  grep "persisting\|window" gpurun_out/l2_$arm.log | head -2
  python tools/l2_table.py $arm
done
