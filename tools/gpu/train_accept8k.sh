cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python tools/train_tensor.py --acceptance --n 8192 --out gpurun_out/trained_accept_8192.hftc > gpurun_out/train_accept_8192.json 2>&1; tail -c 300 gpurun_out/train_accept_8192.json
