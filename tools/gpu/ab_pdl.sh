cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in 3d_1m 2d_262144; do
timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --config $c > gpurun_out/ab_pdl_$c.log 2>&1
HFPG_NO_PDL=1 timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 --config $c > gpurun_out/ab_nopdl_$c.log 2>&1
done
for f in gpurun_out/ab_*.log; do echo "$f $(grep '^{' $f | cut -c60-110)"; done
