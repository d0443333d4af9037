# round 2: toynet parity at 256..65536 (errors -> gpurun_out/toynet_parity.jsonl), forward timing,
# launch list of one 65K forward
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/toynet_parity.jsonl
timeout 900 python -m pytest tests/test_gpu_toynet.py -q -rf --timeout 600 -p no:cacheprovider > gpurun_out/pytest_tn.log 2>&1; echo "rc $?" >> gpurun_out/pytest_tn.log
tail -15 gpurun_out/pytest_tn.log
cat gpurun_out/toynet_parity.jsonl
timeout 300 python tools/bench_toynet.py --n 65536 > gpurun_out/bench_toynet.log 2>&1; tail -1 gpurun_out/bench_toynet.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_toynet.csv python tools/bench_toynet.py --n 65536 --reps 0 > gpurun_out/ncu_toynet.log 2>&1
python tools/ncu_launch_table.py gpurun_out/launches_toynet.csv 2>&1 | tail -40
