# round-2 final measurement pass (final kernels): GPU suite, smoke, bench lines for configs 1-6
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f2_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/f2_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/f2_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f2_smoke.log
timeout 1500 python bench.py > gpurun_out/f2_bench_c5.log 2>&1
for c in 1 2 3 4 6; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/f2_bench_c$c.log 2>&1
done
timeout 900 python bench.py --config 5 --ortho 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f2_bench_c5_f2.log 2>&1
timeout 900 python bench.py --config 5 --ortho 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/f2_bench_c5_f1.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f2_bench_ref.log 2>&1
