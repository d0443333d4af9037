cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"pgemm_tf32<256" -s 0 -c 1 -o gpurun_out/prof_ffn1 python tools/bench_toynet.py --n 65536 --reps 0 > gpurun_out/ncu_ffn1.log 2>&1
tail -n 1 gpurun_out/ncu_ffn1.log
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"pgemm_tf32<128.*EpiStore" -s 2 -c 1 -o gpurun_out/prof_qkv python tools/bench_toynet.py --n 65536 --reps 0 > gpurun_out/ncu_qkv.log 2>&1
tail -n 1 gpurun_out/ncu_qkv.log
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"EpiResidualLN" -s 1 -c 1 -o gpurun_out/prof_oproj python tools/bench_toynet.py --n 65536 --reps 0 > gpurun_out/ncu_oproj.log 2>&1
tail -n 1 gpurun_out/ncu_oproj.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tn_leaf_bias -c 1 -o gpurun_out/prof_lbias python tools/bench_toynet.py --n 65536 --reps 0 > gpurun_out/ncu_lbias.log 2>&1
tail -n 1 gpurun_out/ncu_lbias.log
