cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "8 0" "16 0" "16 1"; do
  set -- $v
  TE_SPMV_XS_NF=$1 TE_SPMV_XS_DICT=$2 timeout 300 python bench.py --config 2 --spmv 8 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bxi_c2_nf$1_d$2.log 2>&1
  TE_SPMV_XS_NF=$1 TE_SPMV_XS_DICT=$2 timeout 300 python bench.py --config 6 --spmv 8 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bxi_c6_nf$1_d$2.log 2>&1
done
for v in "16 0" "16 1"; do
  set -- $v
  TE_SPMV_XS_NF=$1 TE_SPMV_XS_DICT=$2 timeout 600 python bench.py --config 5 --spmv 8 --steps 1 --warmup 1 --prof-steps 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bxi_c5_nf$1_d$2.log 2>&1
done
for sp in 7 8; do
  TE_SPMV_XS_NF=16 timeout 900 python bench.py --config 4 --spmv $sp --steps 1 --warmup 1 --prof-steps 1 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bxi_c4_s$sp.log 2>&1
done
