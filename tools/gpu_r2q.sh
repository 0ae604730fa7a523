cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sw_ or default_choice" > gpurun_out/q_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/q_pytest.log
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmv_sw --launch-skip 3 -c 1 -o gpurun_out/q_c5_spmv_sw \
  python tools/profile_run.py --config 5 > gpurun_out/q_ncu_full5.log 2>&1
