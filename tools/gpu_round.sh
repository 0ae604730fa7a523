cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
python tools/profile_run.py --t 2.5 > gpurun_out/plain2.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_proj|k_spmv|k_update_norm|k_combine" --csv --log-file gpurun_out/restart_metrics.csv python tools/profile_run.py --t 2.5 > gpurun_out/ncu2.log 2>&1
python tools/profile_run.py --t 2.5 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_proj_tma|k_spmv_pipe|k_update_norm" -s 60 -c 4 -o gpurun_out/prof_r01d python tools/profile_run.py --t 2.5 > gpurun_out/ncu3.log 2>&1
python tools/profile_run.py --config 5 --t 1.2 > gpurun_out/plain5.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_proj|k_spmv|k_update_norm|k_combine" --csv --log-file gpurun_out/restart_metrics_c5.csv python tools/profile_run.py --config 5 --t 1.2 > gpurun_out/ncu5.log 2>&1
echo done >> gpurun_out/ncu5.log
