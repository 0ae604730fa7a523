cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
for t in 1 2 4; do TE_SPMV_TPR=$t timeout 1200 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --config 5 > gpurun_out/bench_c5t$t.log 2>&1; done
for t in 2 4 8; do TE_SPMV_TPR=$t timeout 1500 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --config 4 > gpurun_out/bench_c4t$t.log 2>&1; done
