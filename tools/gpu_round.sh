cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3"
timeout 900 $B --config 2 > gpurun_out/fin_c2.log 2>&1
timeout 900 $B --config 1 --no-cpu-baseline > gpurun_out/fin_c1.log 2>&1
timeout 900 $B --config 3 > gpurun_out/fin_c3.log 2>&1
timeout 900 $B --config 6 > gpurun_out/fin_c6.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --config 4 --no-cpu-baseline > gpurun_out/fin_c4.log 2>&1
timeout 1200 python bench.py --steps 3 --warmup 3 --config 5 --no-cpu-baseline > gpurun_out/fin_c5.log 2>&1
for c in 2 3 6; do timeout 900 $B --config $c --ortho 2 --no-cpu-baseline > gpurun_out/fin_c${c}_f2.log 2>&1; done
for c in 2 6; do timeout 900 $B --config $c --ortho 1 --no-cpu-baseline > gpurun_out/fin_c${c}_f1.log 2>&1; done
timeout 1200 python bench.py --steps 3 --warmup 3 --config 5 --ortho 2 --no-cpu-baseline > gpurun_out/fin_c5_f2.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin_ref_c2.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_proj|k_spmv|k_update_norm|k_combine" --csv --log-file gpurun_out/restart_metrics_c6.csv python tools/profile_run.py --config 6 --t 0.3 > gpurun_out/ncu3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spmv_ring" -s 20 -c 1 -o gpurun_out/full_c6_spmv python tools/profile_run.py --config 6 --t 0.3 > gpurun_out/ncu5.log 2>&1
echo done >> gpurun_out/ncu5.log
