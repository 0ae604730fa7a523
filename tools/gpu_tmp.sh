cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "kernel_sets or krylov_basis or max_krylov or m64 or gram or cgs2" > gpurun_out/s5i_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s5i_pytest.log
timeout 1500 python tools/proj_sweep.py --config 5 --m 40 --reps 2 --variant "TE_PROJ_CONST_R=0" --variant "" --variant "TE_PROJ_GRP=4" --variant "TE_PROJ_GRP=8" > gpurun_out/s5i_proj_c5.log 2>&1
timeout 600 python tools/proj_sweep.py --config 2 --m 40 --reps 10 --variant "TE_PROJ_CONST_R=0" --variant "" --variant "TE_PROJ_GRP=4" --variant "TE_PROJ_GRP=8" > gpurun_out/s5i_proj_c2.log 2>&1
