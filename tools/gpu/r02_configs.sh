# round 2: bench lines for every config (default, reference arm, 8K, 65K, 262K, batch, 16.7M, inference)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt
rm -f gpurun_out/cfg_*.log
timeout 900 python bench.py > gpurun_out/cfg_default.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/cfg_ref.log 2>&1
timeout 300 python bench.py --config 2d_8192 --no-cpu-baseline > gpurun_out/cfg_8k.log 2>&1
timeout 300 python bench.py --config 2d_65536 --no-cpu-baseline > gpurun_out/cfg_65k.log 2>&1
timeout 300 python bench.py --config 2d_262144 --no-cpu-baseline > gpurun_out/cfg_262k.log 2>&1
timeout 300 python bench.py --config 2d_65536_infer --no-cpu-baseline > gpurun_out/cfg_infer.log 2>&1
timeout 1500 python bench.py --config batch_262k --steps 1 --warmup 1 > gpurun_out/cfg_batch.log 2>&1
timeout 1500 python bench.py --config part_16m --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/cfg_part16m.log 2>&1
for f in gpurun_out/cfg_*.log; do grep "^{" $f | tail -1; done > gpurun_out/r02_bench_configs.jsonl
wc -l gpurun_out/r02_bench_configs.jsonl
