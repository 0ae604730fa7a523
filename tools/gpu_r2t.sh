cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TE_SPMV_SW_U=-1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sw_ or default_choice" > gpurun_out/t_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t_pytest.log
timeout 900 python tools/spmv_sweep.py --config 5 --m 5 --reps 2 --variant "9:TE_SPMV_SW_U=-1" --variant "9:TE_SPMV_SW_U=0" > gpurun_out/t_sweep_c5.log 2>&1
timeout 600 python tools/spmv_sweep.py --config 2 --m 5 --reps 4 --variant "9:TE_SPMV_SW_U=-1" --variant "9:TE_SPMV_SW_U=0" > gpurun_out/t_sweep_c2.log 2>&1
