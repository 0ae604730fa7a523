cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_proj|k_spmv|k_update_norm|k_combine" --csv --log-file gpurun_out/restart_metrics.csv python tools/profile_run.py --t 2.5 > gpurun_out/ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmv_ring" -s 60 -c 1 -o gpurun_out/full_c2_spmv python tools/profile_run.py --t 2.5 > gpurun_out/ncu6.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_proj_tma" -s 60 -c 2 -o gpurun_out/full_c2 python tools/profile_run.py --t 2.5 > gpurun_out/ncu4.log 2>&1
echo done >> gpurun_out/ncu4.log
