cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sw_ or default_choice or forced_parity" > gpurun_out/aa_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/aa_pytest.log
timeout 900 python -m pytest tests/test_gpu_multirank.py -m gpu -q -x > gpurun_out/aa_pytest_mr.log 2>&1; echo "rc=$?" >> gpurun_out/aa_pytest_mr.log
timeout 1200 python tools/spmv_sweep.py --config 5 --m 5 --reps 2 --variant "9:" --variant "9:TE_SPMV_SW_BITS=16" --variant "9:" > gpurun_out/aa_sweep_c5.log 2>&1
timeout 600 python tools/spmv_sweep.py --config 2 --m 5 --reps 4 --variant "9:" --variant "9:TE_SPMV_SW_BITS=16" > gpurun_out/aa_sweep_c2.log 2>&1
timeout 600 python bench.py --config 1 --spmv 7 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/aa_c1_ring.log 2>&1
timeout 600 python bench.py --config 1 --spmv 8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/aa_c1_xs.log 2>&1
