# in-graph DRAM bytes of 100 iterations at 3D 1M with the leaf kernel's bridges evict_last (default)
# vs evict_first (HFPG_BRIDGE_FIRST=1): the difference is the prolongation's L2 reuse
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for arm in last first; do
  if [ $arm = first ]; then export HFPG_BRIDGE_FIRST=1; else unset HFPG_BRIDGE_FIRST; fi
  timeout 600 ncu --graph-profiling graph --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv --log-file gpurun_out/graph_l2_$arm.csv python tools/solve_driver.py --config 3d_1m --max-iters 100 --reps 1 --graph > gpurun_out/ncu_graph_$arm.log 2>&1
  python - <<PY
import csv, io
txt = [l for l in open("gpurun_out/graph_l2_$arm.csv").read().splitlines() if not l.startswith("==")]
rows = list(csv.DictReader(io.StringIO("\n".join(txt))))
print("$arm", {r["Metric Name"]: r["Metric Value"] for r in rows})
PY
done
