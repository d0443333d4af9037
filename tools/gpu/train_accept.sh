cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/train_tensor.py --acceptance --n 1024 --out gpurun_out/trained_accept_1024.hftc > gpurun_out/train_accept_1024.json 2>&1; tail -c 400 gpurun_out/train_accept_1024.json
