cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/proj_sweep.py --config 5 --m 40 --reps 2 --variant "" > gpurun_out/s5k_generic_c5.log 2>&1
timeout 600 python tools/proj_sweep.py --config 2 --m 40 --reps 10 --variant "" > gpurun_out/s5k_generic_c2.log 2>&1
cp paper_2205_15346_b200/lib/libtimeevolver.so /tmp/lib_keep.so
cp paper_2205_15346_b200/lib/libtimeevolver_lds.so paper_2205_15346_b200/lib/libtimeevolver.so
touch paper_2205_15346_b200/lib/libtimeevolver.so
timeout 900 python tools/proj_sweep.py --config 5 --m 40 --reps 2 --variant "" > gpurun_out/s5k_lds_c5.log 2>&1
timeout 600 python tools/proj_sweep.py --config 2 --m 40 --reps 10 --variant "" > gpurun_out/s5k_lds_c2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "krylov_basis_matches or maximum_krylov" > gpurun_out/s5k_lds_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/s5k_lds_pytest.log
