cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -x -k "multirank or distributed or krylov_basis or pipe_variants" > gpurun_out/pytest_mr.log 2>&1
