timeout 1200 python -m pytest tests/test_gpu_parity.py -q -s -k "final_masks" --deselect tests/test_gpu_parity.py::test_c4_final_masks --deselect tests/test_gpu_parity.py::test_c5_final_masks > gpurun_out/r2j_masks.log 2>&1; echo rc=$?
grep -E "mask agreement|passed|failed" gpurun_out/r2j_masks.log
