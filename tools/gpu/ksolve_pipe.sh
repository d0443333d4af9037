# the persistent solver with pipelined leaves (default) vs sequential (HFPG_KSOLVE_PIPE=0):
# parity tests, then the 8K / 65K solves and phase traces
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_persistent.py tests/test_gpu_pcg.py tests/test_gpu_variants.py -q -x -p no:cacheprovider 2>&1 | tail -2
for arm in pipe seq; do
  if [ $arm = seq ]; then export HFPG_KSOLVE_PIPE=0; else unset HFPG_KSOLVE_PIPE; fi
  for c in 2d_8192 2d_65536; do timeout 300 python tools/phase_trace.py --config $c 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$arm', d['config'], d['iterations'], round(d['solve_ms'],2), d['loop_us_median'])"; done
done
