# session-5: ncu --set full of the config-5 SpMV (8-bit slot-window) and of the TMA projection kernels at ~20 columns
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmv_sw8 --launch-skip 5 -c 1 -o gpurun_out/s5g_spmv_sw8 -f python tools/profile_run.py --config 5 > gpurun_out/s5g_ncu_spmv.log 2>&1; echo "rc=$?" >> gpurun_out/s5g_ncu_spmv.log
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_proj_tma --launch-skip 24 -c 2 -o gpurun_out/s5g_proj -f python tools/profile_run.py --config 5 > gpurun_out/s5g_ncu_proj.log 2>&1; echo "rc=$?" >> gpurun_out/s5g_ncu_proj.log
ls -la gpurun_out/*.ncu-rep
