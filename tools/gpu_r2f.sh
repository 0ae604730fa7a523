cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "xs or default_choice or forced_parity or basis_matches" > gpurun_out/pytest_f.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_f.log
for cfg in 2 3 6; do
  for dct in 1 0; do
    TE_SPMV_XS_DICT=$dct timeout 300 python bench.py --config $cfg --spmv 8 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bxh_c${cfg}_d$dct.log 2>&1
  done
done
TE_SPMV_XS_DICT=1 timeout 600 python bench.py --config 5 --spmv 8 --steps 1 --warmup 1 --prof-steps 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bxh_c5_d1.log 2>&1
