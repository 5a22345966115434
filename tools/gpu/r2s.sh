# round-2 (second half) evidence: default bench line, launch list, ncu --set full of every C3 kernel, C4 / C5 row + column passes
export OMP_NUM_THREADS=$(nproc)
timeout 900 python bench.py > gpurun_out/r2s_bench_c3.json 2> gpurun_out/r2s_bench_c3.err; echo bench_rc=$?; cut -c1-600 gpurun_out/r2s_bench_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2s_launches_c3.csv python bench.py --steps 1 --warmup 0 --iters 20 --no-cpu --no-e2e --no-fft-ref > /dev/null 2>&1; echo ncu_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_rhs_tma|k_wb_tma|k_rows|k_cols" -s 40 -c 14 -o gpurun_out/r2s_c3 -f python bench.py --steps 1 --warmup 0 --iters 8 --no-e2e --no-cpu --no-fft-ref > /dev/null 2>&1; echo ncu3=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_rhs_tma|k_wb_tma|k_rows|k_cols" -s 40 -c 14 -o gpurun_out/r2s_c4 -f python bench.py --config c4 --steps 1 --warmup 0 --iters 8 --no-e2e --no-cpu --no-fft-ref > /dev/null 2>&1; echo ncu4=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_rows|k_cols" -s 9 -c 3 -o gpurun_out/r2s_c5 -f python bench.py --config c5 --steps 1 --warmup 0 --iters 4 --no-e2e --no-cpu --no-fft-ref > /dev/null 2>&1; echo ncu5=$?
for c in c1 c2 c4 c5; do timeout 600 python bench.py --config $c --no-cpu --no-fft-ref >> gpurun_out/r2s_bench_configs.jsonl 2>>gpurun_out/r2s_bench_configs.err; done; echo cfg_rc=$?
cut -c1-300 gpurun_out/r2s_bench_configs.jsonl
ls -la gpurun_out/*.ncu-rep
