cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ./tools/micro/mb_proj 8388608 1 > gpurun_out/z2_mb_n23.log 2>&1
timeout 600 ./tools/micro/mb_proj 1048576 1 > gpurun_out/z2_mb_n20.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "krylov_basis or maximum" > gpurun_out/z2_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/z2_pytest.log
timeout 1500 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/z2_bench_c5.log 2>&1
timeout 600 python bench.py --config 2 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/z2_bench_c2.log 2>&1
