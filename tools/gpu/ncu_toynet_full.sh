cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm_tf32|k_tn_attention_tc|k_tn_leaf_bias" -c 6 -o gpurun_out/prof_toynet python tools/bench_toynet.py --n 65536 --reps 0 > gpurun_out/ncu_toynet_full.log 2>&1
tail -2 gpurun_out/ncu_toynet_full.log
