# session-5: block walk + selective L1 allocation of the 8-bit slot-window SpMV — parity, config-5 sweep, ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sw_block_walk or (config5_instantiation_L22 and blk)" > gpurun_out/s5f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s5f_pytest.log
timeout 1500 python tools/spmv_sweep.py --config 5 --m 6 --reps 2 \
  --variant "9:TE_SPMV_SW_PANEL=0" --variant "9:TE_SPMV_SW_PANEL=0,TE_SPMV_SW_BLK=3" --variant "9:TE_SPMV_SW_PANEL=0,TE_SPMV_SW_BLK=5" \
  --variant "9:TE_SPMV_SW_PANEL=0,TE_SPMV_SW_BLK=6" --variant "9:TE_SPMV_SW_PANEL=0,TE_SPMV_SW_BLK=7" --variant "9:TE_SPMV_SW_PANEL=0,TE_SPMV_SW_BLK=8" \
  --variant "9:TE_SPMV_SW_PANEL=0,TE_SPMV_SW_BLK=10" \
  > gpurun_out/s5f_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/s5f_sweep.log
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct
TE_SPMV_SW_PANEL=0 TE_SPMV_SW_BLK=6 timeout 900 ncu --metrics $M --clock-control none -k regex:k_spmv_sw -c 4 --csv --log-file gpurun_out/s5f_ncu_blk6.csv \
    python tools/spmv_sweep.py --config 5 --m 3 --reps 1 --variant "9:" > gpurun_out/s5f_ncu_blk6.log 2>&1; echo "rc=$?" >> gpurun_out/s5f_ncu_blk6.log
