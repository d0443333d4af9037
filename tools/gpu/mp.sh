cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29533 tools/mp_partition_check.py --same-gpu --size 16384 --max-iters 25 > gpurun_out/mp.log 2>&1; echo "rc $?" >> gpurun_out/mp.log
tail -15 gpurun_out/mp.log
nvidia-smi --query-gpu=name,memory.used --format=csv >> gpurun_out/mp.log
