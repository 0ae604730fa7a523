cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -k "krylov_basis" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for s in 1 3; do for c in 2 3; do timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --config $c --spmv $s > gpurun_out/bench_c${c}s$s.log 2>&1; done; done
