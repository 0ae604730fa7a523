# round-2 first GPU pass: box facts, GPU tests, bench (config 5 default), config-4 ncu traffic
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
{ free -g; cat /sys/fs/cgroup/memory.max 2>/dev/null; nproc; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; } > gpurun_out/box.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/bench_c5.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_c5.log
