# staged-x SpMV: parity first, then config comparisons (short benches)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "xs or default_choice or forced_parity or basis_matches" > gpurun_out/pytest_xs.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_xs.log
for cfg in 2 3 6; do
  for sp in 7 8; do
    timeout 300 python bench.py --config $cfg --spmv $sp --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bx_c${cfg}_s${sp}.log 2>&1
  done
done
for sp in 8 7; do
  timeout 600 python bench.py --config 5 --spmv $sp --steps 2 --warmup 1 --prof-steps 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bx_c5_s${sp}.log 2>&1
done
