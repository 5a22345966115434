timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -q -x -k "band_skip or trajectory_c1 or trajectory_c2 or trajectory_c3 or trajectory_c4_small or trajectory_c5_small or c1_final or c2_final or chunking or fused or wb_parity or rhs_parity or monitor" > gpurun_out/r2d_tests.log 2>&1
echo tests_rc=$?
tail -4 gpurun_out/r2d_tests.log
B="python bench.py --no-cpu --no-e2e --no-fft-ref --steps 3 --warmup 3"
for c in c3 c4 c5 c2 c1; do timeout 300 $B --config $c > gpurun_out/r2d_bench_$c.log 2>&1; done
SRSB_BAND_SKIP=0 timeout 300 $B > gpurun_out/r2d_bench_c3_noskip.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_rhs_tma|k_wb_tma|k_rows|k_cols" -s 20 -c 5 -o gpurun_out/r2d_full -f python bench.py --steps 1 --warmup 0 --iters 7 --no-e2e --no-cpu --no-fft-ref > gpurun_out/r2d_ncu.log 2>&1
echo ncu_rc=$?
