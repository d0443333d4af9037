# usage: K=<kernel regex> NAME=<out> [CFG=3d_1m] bash tools/gpu/ncu_k.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-1} -c ${COUNT:-1} -o gpurun_out/$NAME python tools/iter_driver.py --reps 3 --config ${CFG:-3d_1m} > gpurun_out/$NAME.log 2>&1
tail -2 gpurun_out/$NAME.log
