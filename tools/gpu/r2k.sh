# checked build over the GPU suite (shared-memory bounds asserts), 3-D skip tests, C4/C5 ncu captures
SRSB_LIB=vlib/libsrsb_checks.so timeout 1500 python -m pytest tests -m gpu -q -x -k "not fullsize and not final_masks" > gpurun_out/r2k_checked_tests.log 2>&1; echo checked_rc=$?
tail -3 gpurun_out/r2k_checked_tests.log
SRSB_LIB=vlib/libsrsb_checks.so timeout 300 python tools/sanitize_workload.py > gpurun_out/r2k_checked_workload.log 2>&1; echo checked_workload_rc=$?
timeout 600 python -m pytest tests/test_gpu_3d.py -q -x > gpurun_out/r2k_3d.log 2>&1; echo t3d_rc=$?; tail -2 gpurun_out/r2k_3d.log
timeout 300 python bench.py --config v3d --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2k_v3d.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_rhs_tma|k_wb_tma|k_rows|k_cols" -s 40 -c 5 -o gpurun_out/r2k_c4 -f python bench.py --config c4 --steps 1 --warmup 0 --iters 12 --no-e2e --no-cpu --no-fft-ref > /dev/null 2>&1; echo ncu4=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_rows|k_cols" -s 6 -c 3 -o gpurun_out/r2k_c5 -f python bench.py --config c5 --steps 1 --warmup 0 --iters 4 --no-e2e --no-cpu --no-fft-ref > /dev/null 2>&1; echo ncu5=$?
B="python bench.py --no-cpu --no-e2e --no-fft-ref --steps 2 --warmup 3"
SRSB_CPC=2 timeout 300 $B --config c4 --iters 100 > gpurun_out/r2k_c4_cpc2.log 2>&1
SRSB_BAND_SKIP=0 timeout 300 $B --config c4 --iters 100 > gpurun_out/r2k_c4_noskip.log 2>&1
timeout 300 $B --config c4 --iters 100 > gpurun_out/r2k_c4.log 2>&1
timeout 300 $B --config c5 --iters 50 > gpurun_out/r2k_c5_wide.log 2>&1
SRSB_R2C_WIDE=0 timeout 300 $B --config c5 --iters 50 > gpurun_out/r2k_c5_nowide.log 2>&1
timeout 300 $B --iters 200 > gpurun_out/r2k_c3.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "launch_shape or band_skip or trajectory_c5_small or trajectory_c1" > gpurun_out/r2k_tests2.log 2>&1; echo tests2_rc=$?; tail -2 gpurun_out/r2k_tests2.log
