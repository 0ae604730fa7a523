# Measurement pass on a B200 box (from the repo root; ~40 GPU-minutes):
#   /usr/local/graft/bin/gpurun --timeout 5400 -- 'bash tools/gpu_measure.sh'
# GPU suite, smoke, the bench lines of every config, the reference arm, the ncu launch list of the
# default bench command, DRAM traffic per kernel class over one restart (configs 5, 2, 3, 4, 6) and
# one --set full capture of the config-5 SpMV and of the TMA projection kernels.  Outputs land in
# gpurun_out/m_*; tools/ncu_summarize.py / make_summary.py turn them into profiles/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/m_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/m_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/m_smoke.log
timeout 1500 python bench.py > gpurun_out/m_bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/m_bench_c5.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/m_bench_ref.log 2>&1
for c in 1 2 3 4 6; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/m_bench_c$c.log 2>&1
done
timeout 900 python bench.py --config 5 --ortho 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/m_bench_c5_f2.log 2>&1
timeout 900 python bench.py --config 5 --ortho 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/m_bench_c5_f1.log 2>&1
# launch list of the bench command (cold-cache serialised replay: shares, not absolute times)
timeout 1800 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m_c5_launches.csv \
  python bench.py --steps 1 --warmup 1 --prof-steps 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/m_ncu_launches.log 2>&1
# DRAM traffic per launch over one restart
for cfg in 5 2 3 4 6; do
  timeout 1200 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/m_c${cfg}_restart_metrics.csv python tools/profile_run.py --config $cfg > gpurun_out/m_ncu_c$cfg.log 2>&1
done
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmv_sw8 --launch-skip 5 -c 1 -f -o gpurun_out/m_c5_spmv \
  python tools/profile_run.py --config 5 > gpurun_out/m_ncu_full1.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_proj_tma --launch-skip 24 -c 2 -f -o gpurun_out/m_c5_proj \
  python tools/profile_run.py --config 5 > gpurun_out/m_ncu_full2.log 2>&1
