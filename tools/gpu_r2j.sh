# projection-kernel microbenchmark (register accumulators vs TMA ring) + parity of kernel set 5 + bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ./tools/micro/mb_proj_r > gpurun_out/j_mb_proj_r.log 2>&1; echo "rc=$?" >> gpurun_out/j_mb_proj_r.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "regacc" > gpurun_out/j_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/j_pytest.log
for k in 2 5; do
  timeout 300 python bench.py --config 2 --kernels $k --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/j_c2_k$k.log 2>&1
  timeout 300 python bench.py --config 3 --kernels $k --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/j_c3_k$k.log 2>&1
done
