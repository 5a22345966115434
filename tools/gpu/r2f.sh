timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_fused.py -q -x -k "solve or trajectory_c1 or trajectory_c2 or trajectory_c3 or trajectory_c5_small or trajectory_c4_small or launch_shape or slab or monitor or fused or band or chunking" > gpurun_out/r2f_tests.log 2>&1
echo tests_rc=$?
tail -3 gpurun_out/r2f_tests.log
B="python bench.py --no-cpu --no-e2e --no-fft-ref --steps 3 --warmup 3"
for c in c3 c5 c4; do timeout 300 $B --config $c > gpurun_out/r2f_bench_$c.log 2>&1; done
