# A/B: the leaf kernel's bridge L2 policy (evict_last, default, vs evict_first) under the TMA prolongation
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for arm in last first last first; do
  if [ $arm = last ]; then unset HFPG_BRIDGE_FIRST; else export HFPG_BRIDGE_FIRST=1; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-inference --no-cpu-baseline --no-parity > gpurun_out/bench_br_$arm.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_br_$arm.log') if l.startswith('{')][-1])
print('$arm', round(d['value'],2), d['config_details']['iterations'], {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()}, round(d['roofline'].get('apply_GBps',0)))"
done
