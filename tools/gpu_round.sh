cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
for c in 2 3 6; do timeout 900 $B --config $c > gpurun_out/sw_c$c.log 2>&1; done
for c in 2 3; do timeout 900 $B --config $c --ortho 2 > gpurun_out/sw_c${c}_f2.log 2>&1; done
