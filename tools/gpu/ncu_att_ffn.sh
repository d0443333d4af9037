cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for spec in "ffn1:pgemm_tf32<\(int\)256:0" "att128:k_tn_attn_tc<\(int\)128:0" "hwc:k_tn_highway_chunks:0"; do
  name=${spec%%:*}; rest=${spec#*:}; rx=${rest%:*}; skip=${rest##*:}
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s $skip -c 1 -o gpurun_out/prof_$name python tools/bench_toynet.py --n 65536 --reps 0 > gpurun_out/ncu_$name.log 2>&1
  echo "$name: $(grep -c 'Report' gpurun_out/ncu_$name.log)"
done
