cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ./tools/micro/mb_proj_r 8388608 > gpurun_out/k_mb_proj_r_n23.log 2>&1; echo "rc=$?" >> gpurun_out/k_mb_proj_r_n23.log
timeout 900 ./tools/micro/mb_proj_r 1048576 > gpurun_out/k_mb_proj_r_n20.log 2>&1; echo "rc=$?" >> gpurun_out/k_mb_proj_r_n20.log
