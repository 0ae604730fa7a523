# deferred gate: full GPU suite; staged-x SpMV: ncu + tile-size experiments on config 2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_c.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_c.log
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_spmv_xs --launch-skip 6 -c 1 -o gpurun_out/xs_c2 python tools/profile_run.py --config 2 --spmv 8 > gpurun_out/ncu_xs.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:k_spmv_ring --launch-skip 6 -c 1 -o gpurun_out/ring_c2 python tools/profile_run.py --config 2 --spmv 7 > gpurun_out/ncu_ring.log 2>&1
for cfgv in "2 4096" "1 4096" "4 4096" "2 6000" "1 8192"; do
  set -- $cfgv
  TE_SPMV_XS_TPR=$1 TE_SPMV_XS_ECAP=$2 timeout 300 python bench.py --config 2 --spmv 8 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bxe_c2_t$1_e$2.log 2>&1
done
