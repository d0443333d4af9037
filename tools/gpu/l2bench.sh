# bench A/B of the L2 policy knobs for the bridges (whole solve, graph path)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for arm in ${ARMS:-last w40 w70 last w40 w70}; do
  unset HFPG_BRIDGE_FIRST HFPG_BRIDGE_TAIL HFPG_L2_PERSIST_MB HFPG_L2_WINDOW_MB
  case $arm in w*) export HFPG_L2_PERSIST_MB=80 HFPG_L2_WINDOW_MB=${arm#w};; first) export HFPG_BRIDGE_FIRST=1;; tail*) export HFPG_BRIDGE_TAIL=${arm#tail};; esac
  timeout 600 python bench.py --steps 5 --warmup 3 --no-inference --no-cpu-baseline --no-parity > gpurun_out/bench_l2_$arm.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_l2_$arm.log') if l.startswith('{')][-1])
print('$arm', round(d['value'],2), d['config_details']['iterations'], {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()})"
done
