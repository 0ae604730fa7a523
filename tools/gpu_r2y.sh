# round-2 evidence pass: compute-sanitizer, ncu launch list of the bench command (config 5),
# per-class DRAM traffic over one restart (configs 2-6), --set full captures of the new kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 99 python tools/sanitize_run.py > gpurun_out/y_sanitize_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/y_sanitize_$tool.log
done
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/y_c5_launches.csv \
  python bench.py --steps 1 --warmup 1 --prof-steps 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/y_ncu_launches.log 2>&1
for cfg in 5 4 2 3 6; do
  timeout 1200 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/y_c${cfg}_restart_metrics.csv python tools/profile_run.py --config $cfg > gpurun_out/y_ncu_c$cfg.log 2>&1
done
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmv_ring --launch-skip 6 -c 1 -o gpurun_out/y_c4_spmv_colblk \
  python tools/profile_run.py --config 4 > gpurun_out/y_ncu_full4.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_proj_r --launch-skip 3 -c 1 -o gpurun_out/y_c2_proj_r \
  python tools/profile_run.py --config 2 > gpurun_out/y_ncu_full2r.log 2>&1
