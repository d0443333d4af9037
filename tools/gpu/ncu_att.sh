cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tn_attention_tc -s 0 -c 1 -o gpurun_out/prof_att python tools/bench_toynet.py --n 65536 --reps 0 > gpurun_out/ncu_att.log 2>&1
tail -n 2 gpurun_out/ncu_att.log
