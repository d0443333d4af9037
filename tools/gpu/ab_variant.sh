# A/B a variant .so against the current build: V=<variant> CONFIGS="2d_65536 2d_8192" bash tools/gpu/ab_variant.sh
cd $GRAFT_REPO_ROOT
for c in $CONFIGS; do
  for arm in cur $V; do
    if [ $arm = cur ]; then unset HFPG_SO_VARIANT; else export HFPG_SO_VARIANT=$arm; fi
    timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 3 --config $c 2>&1 | grep "^{" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$c', '$arm', round(d['value'],3), d['config'].get('iterations'), d['config'].get('solver',''))"
  done
done
