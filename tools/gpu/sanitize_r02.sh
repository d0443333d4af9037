# compute-sanitizer matrix on the round-2 kernels (k_prolong_tma, k_coarse_coop, persistent solver)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
out=gpurun_out/sanitizer_r02.txt
: > $out
for spec in memcheck:apply_fast memcheck:solve_graph memcheck:solve_persistent memcheck:iteration_kernels \
            memcheck:group_apply memcheck:toynet racecheck:iteration_kernels racecheck:apply_fast \
            synccheck:iteration_kernels synccheck:apply_fast initcheck:solve_graph initcheck:solve_persistent initcheck:apply_fast; do
  tool=${spec%%:*}; case=${spec#*:}
  timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_driver.py --only $case > gpurun_out/san_${tool}_${case}.log 2>&1
  rc=$?
  summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/san_${tool}_${case}.log | tail -1)
  echo "$tool $case rc=$rc $summ" | tee -a $out
done
