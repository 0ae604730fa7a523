cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/ac_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ac_pytest.log
