cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline"
timeout 600 $B --steps 3 --warmup 3 > gpurun_out/b_3d1m.log 2>&1
timeout 300 $B --steps 3 --warmup 3 --config 2d_65536 > gpurun_out/b_65k.log 2>&1
timeout 300 $B --steps 3 --warmup 3 --config 2d_262144 > gpurun_out/b_262k_auto.log 2>&1
HFPG_SOLVER=persistent timeout 300 $B --steps 3 --warmup 3 --config 2d_262144 > gpurun_out/b_262k_pers.log 2>&1
timeout 900 $B --steps 1 --warmup 1 --config batch_262k > gpurun_out/b_batch.log 2>&1
timeout 1500 $B --steps 1 --warmup 1 --config part_16m > gpurun_out/b_part16m.log 2>&1
for f in gpurun_out/b_*.log; do echo "== $f"; python -c "
import json,sys
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); c=d['config']; print(d['value'], d['ms_per_step'], c.get('iterations', c.get('iterations_mean')), c.get('solver',''), d.get('e2e',{}).get('value'), d.get('roofline',{}).get('frac'))
" 2>&1 | tail -3; tail -2 $f | cut -c1-300; done
