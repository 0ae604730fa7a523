cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/spmv_sweep.py --config 5 --m 5 --reps 2 --variant "8:" --variant "8:TE_SPMV_XS_TPR=4" --variant "8:TE_SPMV_XS_TPR=1" \
  --variant "8:TE_SPMV_XS_TPR=4,TE_SPMV_XS_DICT=1,TE_SPMV_XS_ECAP=4096,TE_SPMV_XS_STAGES=3" --variant "8:TE_SPMV_XS_TPR=4,TE_SPMV_XS_STAGES=3,TE_SPMV_XS_ECAP=3072" \
  --variant "8:TE_SPMV_XS_TPR=4,TE_SPMV_XS_NF=16" --variant "8:TE_SPMV_XS_TPR=8" > gpurun_out/n_sweep_c5.log 2>&1
timeout 900 python tools/spmv_sweep.py --config 2 --m 5 --reps 4 --variant "8:" --variant "8:TE_SPMV_XS_TPR=2" --variant "8:TE_SPMV_XS_TPR=4" --variant "7:" > gpurun_out/n_sweep_c2.log 2>&1
timeout 900 python tools/spmv_sweep.py --config 3 --m 5 --reps 4 --variant "8:" --variant "8:TE_SPMV_XS_TPR=2" --variant "8:TE_SPMV_XS_TPR=4" --variant "7:" > gpurun_out/n_sweep_c3.log 2>&1
timeout 900 python tools/spmv_sweep.py --config 6 --m 5 --reps 4 --variant "8:" --variant "8:TE_SPMV_XS_TPR=8" --variant "8:TE_SPMV_XS_TPR=4" --variant "7:" > gpurun_out/n_sweep_c6.log 2>&1
