# session-5: panel-sweep slot-window SpMV — parity, then the config-5 sweep over panel sizes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sw_variants or config5_instantiation_L22 or sw_panel" > gpurun_out/s5b_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s5b_pytest.log
timeout 1500 python tools/spmv_sweep.py --config 5 --m 6 --reps 2 \
  --variant "9:TE_SPMV_SW_PANEL=0" --variant "9:" --variant "9:TE_SPMV_SW_PANEL=14" --variant "9:TE_SPMV_SW_PANEL=16" \
  --variant "9:TE_SPMV_SW_PANEL=17" --variant "9:TE_SPMV_SW_PANEL=13" \
  --variant "9:TE_SPMV_SW_PANEL=15,TE_SPMV_SW_PANEL_LO=4" --variant "9:TE_SPMV_SW_PANEL=15,TE_SPMV_SW_PANEL_LO=0" \
  > gpurun_out/s5b_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/s5b_sweep.log
