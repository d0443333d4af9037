cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -rf --timeout 600 -p no:cacheprovider -k "pcg or apply or exact or dropin or async or persistent" > gpurun_out/pytest_lc.log 2>&1; echo "rc $?" >> gpurun_out/pytest_lc.log
tail -5 gpurun_out/pytest_lc.log
for arm in fused staged fused staged; do
  if [ $arm = staged ]; then unset HFPG_LEAF_COARSE; else export HFPG_LEAF_COARSE=1; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-inference --no-cpu-baseline > gpurun_out/bench_$arm.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_$arm.log') if l.startswith('{')][-1])
print('$arm', round(d['value'],2), d['config_details']['iterations'], {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()}, d['parity']['exact_bit_identical_to_reference'])"
done
