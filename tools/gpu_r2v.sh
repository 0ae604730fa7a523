cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "colblk or sw_ or default_choice or option" > gpurun_out/v_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/v_pytest.log
timeout 1500 python tools/spmv_sweep.py --config 4 --m 5 --reps 2 --variant "10:TE_SPMV_COLBLK_MB=48" --variant "10:TE_SPMV_COLBLK_MB=32" --variant "10:TE_SPMV_COLBLK_MB=24" --variant "10:TE_SPMV_COLBLK_MB=16" --variant "10:TE_SPMV_COLBLK_MB=40" > gpurun_out/v_sweep_c4.log 2>&1
