# session-5: cross-slice pipelined 8-bit slot-window kernel — parity, config-5 sweep (panel x CTAs per SM)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sw_variants or config5_instantiation_L22 or sw_panel" > gpurun_out/s5h_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s5h_pytest.log
timeout 1500 python tools/spmv_sweep.py --config 5 --m 6 --reps 2 \
  --variant "9:TE_SPMV_SW_PANEL=0" --variant "9:TE_SPMV_SW_PANEL=0,TE_SPMV_SW_MINB=4" \
  --variant "9:TE_SPMV_SW_PANEL=15" --variant "9:TE_SPMV_SW_PANEL=15,TE_SPMV_SW_MINB=4" \
  --variant "9:TE_SPMV_SW_PANEL=13" --variant "9:TE_SPMV_SW_PANEL=13,TE_SPMV_SW_MINB=4" \
  --variant "9:TE_SPMV_SW_PANEL=16" --variant "9:TE_SPMV_SW_PANEL=14" \
  > gpurun_out/s5h_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/s5h_sweep.log
timeout 600 python tools/spmv_sweep.py --config 2 --m 12 --reps 5 --variant "9:" --variant "9:TE_SPMV_SW_MINB=4" > gpurun_out/s5h_sweep_c2.log 2>&1
