cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for pf in 0 1 2 4 8; do
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --prefetch $pf > gpurun_out/bench_pf$pf.log 2>&1
done
