cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train_loop.py tests/test_gpu_train.py -q -rf --timeout 800 -p no:cacheprovider > gpurun_out/pytest_trainloop.log 2>&1; echo "rc $?" >> gpurun_out/pytest_trainloop.log
tail -25 gpurun_out/pytest_trainloop.log
