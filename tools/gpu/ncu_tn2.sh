# ncu --set full of the toynet leaf-bias and leaf-attention kernels at N = 65,536
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/prof_tn_*.ncu-rep
#timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tn_leaf_bias -c 1 -o gpurun_out/prof_tn_bias python tools/bench_toynet.py --n 65536 --reps 0 > gpurun_out/ncu_tn_bias.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tn_attn_tc -c 1 -o gpurun_out/prof_tn_attn python tools/bench_toynet.py --n 65536 --reps 0 > gpurun_out/ncu_tn_attn.log 2>&1
ls gpurun_out/prof_tn_*
