cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sell" > gpurun_out/pytest_sell.log 2>&1 || exit 1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --spmv 6"
for c in 6 2 3 5 4; do timeout 900 $B --config $c > gpurun_out/sw_sell_c$c.log 2>&1; done
