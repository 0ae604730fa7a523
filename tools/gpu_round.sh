cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/box.log; free -g >> gpurun_out/box.log
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size_config" --durations=5 > gpurun_out/pytest_full.log 2>&1
