cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TE_SPMV_SW_FAR=21 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sw_ or default_choice" > gpurun_out/u_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/u_pytest.log
timeout 1200 python tools/spmv_sweep.py --config 5 --m 5 --reps 2 --variant "9:" --variant "9:TE_SPMV_SW_FAR=20" --variant "9:TE_SPMV_SW_FAR=21" \
  --variant "9:TE_SPMV_SW_FAR=22" --variant "9:TE_SPMV_SW_FAR=23" --variant "9:" > gpurun_out/u_sweep_c5.log 2>&1
