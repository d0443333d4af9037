# ncu --set full of the toynet attention + FFN1 GEMM (one launch each, N=65,536)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for k in "k_tn_attn_tc" "k_pgemm_tf32"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_$k python tools/bench_toynet.py --n 65536 --reps 0 > gpurun_out/ncu_$k.log 2>&1
  tail -n 2 gpurun_out/ncu_$k.log
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pgemm_tf32<256" -s 0 -c 1 -o gpurun_out/prof_ffn1 python tools/bench_toynet.py --n 65536 --reps 0 > gpurun_out/ncu_ffn1.log 2>&1
tail -n 2 gpurun_out/ncu_ffn1.log
ls -la gpurun_out/*.ncu-rep
