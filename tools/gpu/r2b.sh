set -x
B="python bench.py --no-cpu --no-fft-ref --no-e2e --steps 3 --warmup 3"
timeout 200 $B > gpurun_out/r2b_bench_default.log 2>&1
SRSB_SYMTAB=1 timeout 200 $B > gpurun_out/r2b_bench_symtab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -m gpu -q -x -k "solve or slab or trajectory_c1 or trajectory_c2 or trajectory_c3 or c1_final or dist_solver or teacher" > gpurun_out/r2b_pytest.log 2>&1
echo pytest_rc=$?
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_cols_solve|k_rhs_tma" -s 20 -c 4 -o gpurun_out/r2b_full -f python bench.py --steps 1 --warmup 0 --iters 3 --no-e2e --no-cpu --no-fft-ref > gpurun_out/r2b_ncu.log 2>&1
echo ncu_rc=$?
SANI_TIMEOUT=400 bash tools/run_sanitizers.sh c1 modes slab > gpurun_out/r2b_sani.log 2>&1
tail -5 gpurun_out/r2b_pytest.log
