# session-5: ncu DRAM bytes / L2 hit rate / duration of the slot-window SpMV passes on config 5
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active
for P in 0 15 13; do
  TE_SPMV_SW_PANEL=$P timeout 900 ncu --metrics $M --clock-control none -k regex:k_spmv_sw -c 6 --csv --log-file gpurun_out/s5c_ncu_panel$P.csv \
    python tools/spmv_sweep.py --config 5 --m 3 --reps 1 --variant "9:" > gpurun_out/s5c_ncu_panel$P.log 2>&1; echo "rc=$?" >> gpurun_out/s5c_ncu_panel$P.log
done
