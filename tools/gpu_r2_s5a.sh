# session-5 validation: GPU suite, smoke, default bench (config 5)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/s5a_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/s5a_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5a_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/s5a_smoke.log
timeout 1500 python bench.py > gpurun_out/s5a_bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/s5a_bench_c5.log
