cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
export TE_SPMV_NF_WIDE=0
for t in 1 2; do TE_SPMV_RING_TPR=$t timeout 600 $B --config 2 > gpurun_out/sw_r23_c2_t$t.log 2>&1; done
for t in 4 8; do TE_SPMV_RING_TPR=$t timeout 600 $B --config 6 > gpurun_out/sw_r23_c6_t$t.log 2>&1; done
for t in 2 4; do TE_SPMV_RING_TPR=$t timeout 900 $B --config 5 > gpurun_out/sw_r23_c5_t$t.log 2>&1; done
for t in 2 4; do TE_SPMV_RING_TPR=$t timeout 600 $B --config 3 > gpurun_out/sw_r23_c3_t$t.log 2>&1; done
