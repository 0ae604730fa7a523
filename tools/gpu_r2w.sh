# validation pass: full GPU suite, smoke, default bench (config 5), config 4/2/3/6 benches, reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/w_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/w_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/w_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/w_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/w_smoke.log
timeout 1500 python bench.py > gpurun_out/w_bench.log 2>&1; echo "rc=$?" >> gpurun_out/w_bench.log
for c in 4 2 3 6; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/w_bench_c$c.log 2>&1
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/w_bench_ref.log 2>&1
