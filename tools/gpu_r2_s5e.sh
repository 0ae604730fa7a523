# session-5: staged-block slot-window SpMV — parity, config-5 sweep, ncu L2 traffic
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sw_staged or config5_instantiation_L22" > gpurun_out/s5e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s5e_pytest.log
timeout 1500 python tools/spmv_sweep.py --config 5 --m 6 --reps 2 \
  --variant "9:TE_SPMV_SW_PANEL=0" --variant "9:TE_SPMV_SW_PANEL=0,TE_SPMV_SW_STAGE=512" --variant "9:TE_SPMV_SW_PANEL=0,TE_SPMV_SW_STAGE=1024" \
  > gpurun_out/s5e_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/s5e_sweep.log
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active
TE_SPMV_SW_PANEL=0 TE_SPMV_SW_STAGE=1024 timeout 900 ncu --metrics $M --clock-control none -k regex:k_spmv_sw -c 4 --csv --log-file gpurun_out/s5e_ncu_staged.csv \
    python tools/spmv_sweep.py --config 5 --m 3 --reps 1 --variant "9:TE_SPMV_SW_PANEL=0,TE_SPMV_SW_STAGE=1024" > gpurun_out/s5e_ncu_staged.log 2>&1; echo "rc=$?" >> gpurun_out/s5e_ncu_staged.log
