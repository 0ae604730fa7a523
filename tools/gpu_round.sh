cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x -k "ring or multirank" > gpurun_out/pytest_ring.log 2>&1 || { echo FAIL >> gpurun_out/pytest_ring.log; exit 1; }
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
for c in 2 3 6 5; do timeout 900 $B --config $c > gpurun_out/sw_rs_c$c.log 2>&1; done
