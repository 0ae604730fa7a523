cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python tools/spmv_sweep.py --config 5 --m 5 --reps 2 --variant "9:" --variant "9:TE_SPMV_SW_U=21" --variant "9:TE_SPMV_SW_U=16" \
  --variant "9:TE_SPMV_SW_U=24" --variant "9:TE_SPMV_SW_U=161" --variant "9:TE_SPMV_SW_U=1" --variant "9:" > gpurun_out/x_sweep_c5.log 2>&1
