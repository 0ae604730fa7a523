cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
timeout 600 $B --config 2 > gpurun_out/sw_rem_c2a.log 2>&1
timeout 600 $B --config 3 > gpurun_out/sw_rem_c3.log 2>&1
timeout 600 $B --config 2 > gpurun_out/sw_rem_c2b.log 2>&1
timeout 600 $B --config 2 --ortho 2 > gpurun_out/sw_rem_c2f2.log 2>&1
