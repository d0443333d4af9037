# A/B: VAR=<env assignment for B> [BENCH_ARGS=...] bash tools/gpu/ab.sh
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for arm in A B; do
  if [ $arm = B ]; then export $VAR; fi
  echo "== $arm ($( [ $arm = B ] && echo $VAR ))"
  timeout 300 python tools/iter_driver.py --reps 5 2>&1 | tail -1
  timeout 600 python bench.py --no-cpu-baseline --steps 3 --warmup 3 ${BENCH_ARGS} 2>&1 | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; print('value',d['value'],'iters',d['config'].get('iterations'),'it ms', r.get('solve_ms_per_iteration'), 'dom', r.get('kernel'), round(r.get('frac',0),3), 'apply GBps', round(r.get('apply_GBps',0)))"
done
