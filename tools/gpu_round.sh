cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --config 1 --no-cpu-baseline > gpurun_out/final_c1.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --config 2 > gpurun_out/final_c2.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --config 2 --ortho 1 --no-cpu-baseline > gpurun_out/final_c2_lanczos.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --config 3 > gpurun_out/final_c3.log 2>&1
timeout 1500 python bench.py --steps 2 --warmup 1 --config 5 --no-cpu-baseline > gpurun_out/final_c5.log 2>&1
timeout 1800 python bench.py --steps 2 --warmup 1 --config 4 --no-cpu-baseline > gpurun_out/final_c4.log 2>&1
