# round-2 (second half) evidence: default bench line, launch list, ncu --set full of every C3 kernel (summaries made on the box:
# gpurun_out/ is capped at 64 MiB), C4 / C5 passes, all-config lines
export OMP_NUM_THREADS=$(nproc)
timeout 900 python bench.py > gpurun_out/r2t_bench_c3.json 2> gpurun_out/r2t_bench_c3.err; echo bench_rc=$?; cut -c1-300 gpurun_out/r2t_bench_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2t_launches_c3.csv python bench.py --steps 1 --warmup 0 --iters 20 --no-cpu --no-e2e --no-fft-ref > /dev/null 2>&1; echo ncu_rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_rhs_tma|k_wb_tma|k_rows|k_cols" -s 43 -c 7 -o gpurun_out/r2t_c3 -f python bench.py --steps 1 --warmup 0 --iters 8 --no-e2e --no-cpu --no-fft-ref > /dev/null 2>&1; echo ncu3=$?
python tools/ncu_summary.py gpurun_out/r2t_c3.ncu-rep > gpurun_out/r2t_ncu_full_c3.txt 2>&1
python tools/ncu_traffic.py gpurun_out/r2t_c3.ncu-rep gpurun_out/r2t_ncu_traffic.json c3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_rhs_tma|k_wb_tma|k_rows|k_cols" -s 43 -c 7 -o /tmp/r2t_c4 -f python bench.py --config c4 --steps 1 --warmup 0 --iters 8 --no-e2e --no-cpu --no-fft-ref > /dev/null 2>&1; echo ncu4=$?
python tools/ncu_summary.py /tmp/r2t_c4.ncu-rep > gpurun_out/r2t_ncu_full_c4.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_rhs_tma|k_wb_tma|k_rows|k_cols" -s 17 -c 7 -o /tmp/r2t_c5 -f python bench.py --config c5 --steps 1 --warmup 0 --iters 4 --no-e2e --no-cpu --no-fft-ref > /dev/null 2>&1; echo ncu5=$?
python tools/ncu_summary.py /tmp/r2t_c5.ncu-rep > gpurun_out/r2t_ncu_full_c5.txt 2>&1
for c in c1 c2 c4 c5; do timeout 600 python bench.py --config $c --no-cpu --no-fft-ref >> gpurun_out/r2t_bench_configs.jsonl 2>>gpurun_out/r2t_bench_configs.err; done; echo cfg_rc=$?
ls -la gpurun_out/*.ncu-rep; du -sh gpurun_out
