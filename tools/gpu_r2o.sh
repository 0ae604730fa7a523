cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sw_ or default_choice" > gpurun_out/o_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/o_pytest.log
timeout 900 python tools/spmv_sweep.py --config 5 --m 5 --reps 2 --variant "9:" --variant "8:" > gpurun_out/o_sweep_c5.log 2>&1
timeout 600 python tools/spmv_sweep.py --config 2 --m 5 --reps 4 --variant "9:" --variant "8:" --variant "7:" > gpurun_out/o_sweep_c2.log 2>&1
timeout 600 python tools/spmv_sweep.py --config 3 --m 5 --reps 4 --variant "9:TE_SPMV_SW_FORCE=1" --variant "8:" > gpurun_out/o_sweep_c3.log 2>&1
timeout 600 python tools/spmv_sweep.py --config 6 --m 5 --reps 4 --variant "9:TE_SPMV_SW_FORCE=1" --variant "7:" > gpurun_out/o_sweep_c6.log 2>&1
