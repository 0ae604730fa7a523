cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "xs or default_choice or basis_matches or ring_variants or maximum or evolve_forced" > gpurun_out/pytest_d.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_d.log
for v in "7 0 0" "8 1 2" "8 1 3" "8 2 3" "8 2 2"; do
  set -- $v
  TE_SPMV_XS_TPR=$2 TE_SPMV_XS_STAGES=$3 timeout 300 python bench.py --config 2 --spmv $1 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bxf_c2_s$1_t$2_st$3.log 2>&1
done
for v in "7 0 0" "8 2 3" "8 2 2" "8 1 3"; do
  set -- $v
  TE_SPMV_XS_TPR=$2 TE_SPMV_XS_STAGES=$3 timeout 600 python bench.py --config 5 --spmv $1 --steps 1 --warmup 1 --prof-steps 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bxf_c5_s$1_t$2_st$3.log 2>&1
done
