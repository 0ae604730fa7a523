# session-5: config-5 bench with the two-pass panel sweep (default panel 15, and 13) vs one pass
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for P in 15 13 0; do
  TE_SPMV_SW_PANEL=$P timeout 1500 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s5d_bench_c5_panel$P.log 2>&1; echo "rc=$?" >> gpurun_out/s5d_bench_c5_panel$P.log
done
