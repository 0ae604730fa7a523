# round-2 measurement pass (from the repo root on a GPU box):
#   /usr/local/graft/bin/gpurun --timeout 5400 -- 'bash tools/gpu_r2_final.sh'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/f_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/f_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/f_bench.log 2>&1; echo "rc=$?" >> gpurun_out/f_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_bench_ref.log 2>&1
# launch list of the bench command (cold-cache serialised replay: shares, not absolute times)
timeout 1800 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_c5_launches.csv \
  python bench.py --steps 1 --warmup 1 --prof-steps 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/f_ncu_launches.log 2>&1
# DRAM traffic per launch over one restart: configs 5 and 4
for cfg in 5 4; do
  timeout 1200 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/f_c${cfg}_restart_metrics.csv python tools/profile_run.py --config $cfg > gpurun_out/f_ncu_c$cfg.log 2>&1
done
# full captures: the config-5 SpMV (staged-x) and an update_proj (TMA) launch at ~20 columns
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmv_xs --launch-skip 3 -c 1 -o gpurun_out/f_c5_spmv \
  python tools/profile_run.py --config 5 > gpurun_out/f_ncu_full1.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"k_proj_tma<1" --launch-skip 12 -c 1 -o gpurun_out/f_c5_update \
  python tools/profile_run.py --config 5 > gpurun_out/f_ncu_full2.log 2>&1
