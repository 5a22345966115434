B="python bench.py --no-cpu --no-e2e --no-fft-ref --steps 2 --warmup 3"
timeout 300 $B --iters 200 > gpurun_out/r2i_c3.log 2>&1
for g in 1 2; do SRSB_G=$g timeout 300 $B --config c5 --iters 50 > gpurun_out/r2i_c5_g$g.log 2>&1; done
for g in 1 2; do SRSB_G=$g timeout 300 $B --config c4 --iters 100 > gpurun_out/r2i_c4_g$g.log 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "monitor or solve or trajectory_c1 or launch_shape or iterate_until" > gpurun_out/r2i_tests.log 2>&1; echo tests_rc=$?; tail -2 gpurun_out/r2i_tests.log
