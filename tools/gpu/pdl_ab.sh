# A/B of programmatic dependent launch (HFPG_PDL=1) vs plain launches (default),
# after the apply / PCG parity tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -rf --timeout 600 -p no:cacheprovider -k "pcg or apply or exact or dropin or async or persistent or part" > gpurun_out/pytest_pdl.log 2>&1; echo "rc $?" >> gpurun_out/pytest_pdl.log
tail -5 gpurun_out/pytest_pdl.log
for arm in pdl nopdl pdl nopdl; do
  if [ $arm = pdl ]; then export HFPG_PDL=1; else unset HFPG_PDL; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-inference --no-cpu-baseline > gpurun_out/bench_pdl_$arm.log 2>&1
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/bench_pdl_$arm.log') if l.startswith('{')][-1])
print('$arm', round(d['value'],2), d['config_details']['iterations'], {k: round(v*1e3,1) for k,v in d['roofline']['kernel_ms'].items()}, d['parity']['exact_bit_identical_to_reference'], round(d['roofline'].get('apply_GBps',0)))"
done
