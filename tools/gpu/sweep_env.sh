# usage: NAME=VAR VALUES="a b c" bash tools/gpu/sweep_env.sh   -> iter_driver per value
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in $VALUES; do
  echo "== $NAME=$v"
  env $NAME=$v timeout 300 python tools/iter_driver.py --reps 5 --config ${CFG:-3d_1m} 2>&1 | tail -1
done
