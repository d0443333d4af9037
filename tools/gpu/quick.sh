cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/iter_driver.py --reps 5 > gpurun_out/iter.log 2>&1
timeout 300 python tools/iter_driver.py --reps 5 --config 2d_262144 >> gpurun_out/iter.log 2>&1
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_pcg.py} -q -x -p no:cacheprovider > gpurun_out/qtest.log 2>&1; echo "pytest rc $?" >> gpurun_out/qtest.log
timeout 600 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/qbench.log 2>&1
cat gpurun_out/iter.log; tail -3 gpurun_out/qtest.log; grep "^{" gpurun_out/qbench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('value',d['value'],'iters',d['config']['iterations'],'kernel_ms',d['roofline']['kernel_ms'],'spmv GBps',d['roofline']['spmv_GBps'], 'it ms', d['roofline']['solve_ms_per_iteration'])"
