# round-2 validation pass after the container restore: build, GPU tests, smoke, default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/i_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/i_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/i_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/i_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/i_smoke.log
timeout 1500 python bench.py > gpurun_out/i_bench.log 2>&1; echo "rc=$?" >> gpurun_out/i_bench.log
