cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool racecheck --error-exitcode 9 python tools/sanitize_driver.py --only toynet > gpurun_out/san_racecheck_toynet.log 2>&1; echo "racecheck toynet rc $?" >> gpurun_out/san_racecheck_toynet.log
for t in apply_fast apply_generic solve_graph solve_persistent group toynet; do
timeout 900 $CS --tool synccheck --num-cuda-barriers 65536 --error-exitcode 9 python tools/sanitize_driver.py --only $t > gpurun_out/san_synccheck_$t.log 2>&1; echo "synccheck $t rc $?" >> gpurun_out/san_synccheck_$t.log
done
for t in solve_graph group; do
timeout 900 $CS --tool racecheck --error-exitcode 9 python tools/sanitize_driver.py --only $t > gpurun_out/san_racecheck_$t.log 2>&1; echo "racecheck $t rc $?" >> gpurun_out/san_racecheck_$t.log
done
for f in gpurun_out/san_racecheck_toynet.log gpurun_out/san_synccheck_*.log gpurun_out/san_racecheck_solve_graph.log gpurun_out/san_racecheck_group.log; do echo "== $f"; grep -v "^ok" $f | tail -n 6; done
