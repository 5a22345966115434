# the r2c warp-shuffle split is not bitwise equal to the shared-memory split (FMA contraction differs): parity and masks with it
export OMP_NUM_THREADS=$(nproc)
SRSB_LIB=vlib/libsrsb_shfl_both.so timeout 1500 python -m pytest tests/test_gpu_parity.py -q -s -k "c3_final_masks or trajectory_c3_images or solve_parity or closed_forms" -p no:cacheprovider > gpurun_out/r2x_shfl_tests.log 2>&1; echo rc=$?
grep -E "mask agreement|passed|failed|FAILED" gpurun_out/r2x_shfl_tests.log | tail
