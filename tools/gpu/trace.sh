cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in ${CONFIGS:-2d_65536 3d_1m}; do timeout 300 python tools/phase_trace.py --config $c; done > gpurun_out/trace.log 2>&1
cat gpurun_out/trace.log
