timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity.py::test_c3_final_masks --deselect tests/test_gpu_parity.py::test_c4_final_masks --deselect tests/test_gpu_parity.py::test_c5_final_masks --durations=15 > gpurun_out/r2e_tests.log 2>&1
echo tests_rc=$?
tail -22 gpurun_out/r2e_tests.log
timeout 400 python bench.py --steps 5 --warmup 3 > gpurun_out/r2e_bench_c3.log 2>&1
echo bench_rc=$?
tail -1 gpurun_out/r2e_bench_c3.log | cut -c1-300
