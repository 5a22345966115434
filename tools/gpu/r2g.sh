B="python bench.py --no-cpu --no-e2e --no-fft-ref --steps 3 --warmup 3 --iters 100"
timeout 300 $B > gpurun_out/r2g_cur.log 2>&1
SRSB_LIB=vlib/libsrsb_regold.so timeout 300 $B > gpurun_out/r2g_regold.log 2>&1
SRSB_LIB=vlib/libsrsb_atomic.so timeout 300 $B > gpurun_out/r2g_atomic.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_rows_c2r" -s 3 -c 1 -o gpurun_out/r2g_c2r -f python bench.py --steps 1 --warmup 0 --iters 3 --no-e2e --no-cpu --no-fft-ref > /dev/null 2>&1
SRSB_LIB=vlib/libsrsb_atomic.so timeout 300 ncu --set full --import-source on --clock-control none -k regex:"k_rows_c2r" -s 3 -c 1 -o gpurun_out/r2g_c2r_atomic -f python bench.py --steps 1 --warmup 0 --iters 3 --no-e2e --no-cpu --no-fft-ref > /dev/null 2>&1
