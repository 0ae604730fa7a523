cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --config 3 > gpurun_out/bench_c3.log 2>&1
