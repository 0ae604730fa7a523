cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
TE_SPMV_XS_DICT=0 timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_spmv_xs --launch-skip 6 -c 1 -o gpurun_out/xs2_c2_nodict python tools/profile_run.py --config 2 --spmv 8 > gpurun_out/ncu_xs2a.log 2>&1
TE_SPMV_XS_DICT=1 timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_spmv_xs --launch-skip 6 -c 1 -o gpurun_out/xs2_c2_dict python tools/profile_run.py --config 2 --spmv 8 > gpurun_out/ncu_xs2b.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_spmv_ring --launch-skip 6 -c 1 -o gpurun_out/ring2_c2 python tools/profile_run.py --config 2 --spmv 7 > gpurun_out/ncu_ring2.log 2>&1
