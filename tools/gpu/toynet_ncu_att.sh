cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpu/toynet_r02.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tn_attn_tc -s 2 -c 1 -o gpurun_out/prof_att128 python tools/bench_toynet.py --n 65536 --reps 0 > gpurun_out/ncu_att128.log 2>&1
tail -n 1 gpurun_out/ncu_att128.log
