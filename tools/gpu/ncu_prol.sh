# ncu --set full of the TMA prolongation (standalone launches, tools/iter_driver.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/prof_k_prolong_tma.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_prolong_tma -s 2 -c 1 -o gpurun_out/prof_k_prolong_tma python tools/iter_driver.py --reps 3 > gpurun_out/ncu_prol.log 2>&1
echo "rc $? $(grep -c Report gpurun_out/ncu_prol.log)"
