cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sw_ or default_choice or full_size" > gpurun_out/ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_pytest.log
timeout 600 python tools/spmv_sweep.py --config 2 --m 5 --reps 4 --variant "9:" --variant "9:TE_SPMV_SW_BITS=16" > gpurun_out/ab_sweep_c2.log 2>&1
timeout 1500 python bench.py > gpurun_out/ab_bench_c5.log 2>&1
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 > gpurun_out/ab_bench_c2.log 2>&1
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/ab_bench_c1.log 2>&1
