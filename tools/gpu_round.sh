cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
for r in 1 2; do TE_SPMV_RPG=$r timeout 600 $B --config 2 > gpurun_out/sw_rpg${r}_c2.log 2>&1; done
for r in 1 2; do TE_SPMV_RPG=$r timeout 600 $B --config 3 > gpurun_out/sw_rpg${r}_c3.log 2>&1; done
for r in 1 2; do TE_SPMV_RPG=$r timeout 900 $B --config 5 > gpurun_out/sw_rpg${r}_c5.log 2>&1; done
TE_SPMV_RPG=2 TE_SPMV_TPR=8 timeout 600 $B --config 6 > gpurun_out/sw_rpg2_c6_t8.log 2>&1
TE_SPMV_RPG=1 timeout 600 $B --config 6 > gpurun_out/sw_rpg1_c6.log 2>&1
TE_SPMV_RPG=2 timeout 600 $B --config 1 > gpurun_out/sw_rpg2_c1.log 2>&1
