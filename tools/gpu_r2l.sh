cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "regacc or hybrid or tma or option or maximum" > gpurun_out/l_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/l_pytest.log
timeout 600 ./tools/micro/mb_proj 1048576 > gpurun_out/l_mb_n20.log 2>&1
for k in 2 5; do
  timeout 300 python bench.py --config 2 --kernels $k --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/l_c2_k$k.log 2>&1
done
timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/l_c3.log 2>&1
timeout 900 python bench.py --config 4 --steps 2 --warmup 1 --prof-steps 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/l_c4.log 2>&1
# DRAM traffic per launch over a short evolution: configs 5 and 4
for cfg in 5 4; do
  timeout 1200 $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none --csv \
    --log-file gpurun_out/l_c${cfg}_restart_metrics.csv python tools/profile_run.py --config $cfg > gpurun_out/l_ncu_c$cfg.log 2>&1
done
# full captures of the config-5 and config-4 SpMVs
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmv --launch-skip 3 -c 1 -o gpurun_out/l_c5_spmv \
  python tools/profile_run.py --config 5 > gpurun_out/l_ncu_full5.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_spmv --launch-skip 3 -c 1 -o gpurun_out/l_c4_spmv \
  python tools/profile_run.py --config 4 > gpurun_out/l_ncu_full4.log 2>&1
