cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for t in iteration_kernels group_apply; do
for tool in racecheck synccheck; do
timeout 900 $CS --tool $tool --num-cuda-barriers 65536 --error-exitcode 9 python tools/sanitize_driver.py --only $t > gpurun_out/san_${tool}_$t.log 2>&1; echo "$tool $t rc $?" >> gpurun_out/san_${tool}_$t.log
done; done
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python tools/sanitize_driver.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc $?" >> gpurun_out/san_memcheck.log
for f in gpurun_out/san_*_iteration_kernels.log gpurun_out/san_*_group_apply.log gpurun_out/san_memcheck.log; do echo "== $f"; grep -v "^ok" $f | tail -n 3; done
