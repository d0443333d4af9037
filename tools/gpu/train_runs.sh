cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_train_loop.py -q -rf --timeout 500 -p no:cacheprovider 2>&1 | tail -3
timeout 900 python tools/train_tensor.py --n 1024 --steps 3000 --log-every 250 --out gpurun_out/trained_1024.hftc > gpurun_out/train_1024.json 2>&1; tail -c 600 gpurun_out/train_1024.json
timeout 1200 python tools/train_tensor.py --n 16384 --steps 1500 --log-every 250 --out gpurun_out/trained_16384.hftc > gpurun_out/train_16384.json 2>&1; tail -c 600 gpurun_out/train_16384.json
