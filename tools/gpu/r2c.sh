set -x
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x > gpurun_out/r2c_fused.log 2>&1
echo fused_rc=$?
tail -15 gpurun_out/r2c_fused.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "trajectory_c1 or trajectory_c2 or trajectory_c3 or c1_final or c2_final or chunking or monitor" > gpurun_out/r2c_parity.log 2>&1
echo parity_rc=$?
tail -5 gpurun_out/r2c_parity.log
B="python bench.py --no-cpu --no-e2e --steps 3 --warmup 3"
timeout 300 $B > gpurun_out/r2c_bench_c3.log 2>&1
SRSB_FUSE=0 timeout 300 $B --no-fft-ref > gpurun_out/r2c_bench_c3_nofuse.log 2>&1
timeout 300 $B --no-fft-ref --config c2 > gpurun_out/r2c_bench_c2.log 2>&1
timeout 300 $B --no-fft-ref --config c1 > gpurun_out/r2c_bench_c1.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_rhs_r2c|k_cols_solve|k_rows_c2r|k_wb_tma" -s 10 -c 4 -o gpurun_out/r2c_full -f python bench.py --steps 1 --warmup 0 --iters 3 --no-e2e --no-cpu --no-fft-ref > gpurun_out/r2c_ncu.log 2>&1
echo ncu_rc=$?
