# ncu --set full of k_coarse_coop (standalone iterations, tools/iter_driver.py)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/prof_k_coarse_coop.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_coarse_coop -s 2 -c 1 -o gpurun_out/prof_k_coarse_coop python tools/iter_driver.py --reps 3 > gpurun_out/ncu_coop.log 2>&1
echo "ncu rc $? $(grep -c Report gpurun_out/ncu_coop.log)"
