cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmv_sw --launch-skip 3 -c 1 -o gpurun_out/s_c5_spmv_sw \
  python tools/profile_run.py --config 5 > gpurun_out/s_ncu_full5.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmv --launch-skip 3 -c 1 -o gpurun_out/s_c4_spmv \
  python tools/profile_run.py --config 4 > gpurun_out/s_ncu_full4.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_proj_tma<1" --launch-skip 12 -c 1 -o gpurun_out/s_c5_update \
  python tools/profile_run.py --config 5 > gpurun_out/s_ncu_full5u.log 2>&1
