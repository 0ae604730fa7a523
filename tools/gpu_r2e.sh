cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_e.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_e.log
for cfg in 2 3 6; do
  for v in "7 0" "8 0" "8 1"; do
    set -- $v
    TE_SPMV_XS_XPOL=$2 timeout 300 python bench.py --config $cfg --spmv $1 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bxg_c${cfg}_s$1_p$2.log 2>&1
  done
done
for v in "8 0" "8 1"; do
  set -- $v
  TE_SPMV_XS_XPOL=$2 timeout 600 python bench.py --config 5 --spmv $1 --steps 1 --warmup 1 --prof-steps 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bxg_c5_s$1_p$2.log 2>&1
done
