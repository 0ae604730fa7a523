cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config 1 > gpurun_out/bench_c1.log 2>&1
timeout 1800 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --config 4 > gpurun_out/bench_c4.log 2>&1
