# final build of round 2 (warp-shuffle split in the H = 512 row passes): full suite, smoke, checked build over the solve paths,
# default bench line, launch list, ncu --set full of the C3 kernels, all-config lines
export OMP_NUM_THREADS=$(nproc)
timeout 3000 python -m pytest tests -m gpu -q -rfE -s -p no:cacheprovider > gpurun_out/r2y_gputests.log 2>&1; echo gputests_rc=$?
grep -E "mask agreement|passed|failed|FAILED|ERROR|xfail" gpurun_out/r2y_gputests.log | tail -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/r2y_smoke.log
SRSB_LIB=vlib/libsrsb_checks.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_3d.py tests/test_gpu_slab.py -q -k "solve or trajectory_c1 or trajectory_c2 or trajectory_c3_other or slab_group or cos_modes" -p no:cacheprovider > gpurun_out/r2y_checked.log 2>&1; echo checked_rc=$?; tail -2 gpurun_out/r2y_checked.log
timeout 900 python bench.py > gpurun_out/r2y_bench_c3.json 2> gpurun_out/r2y_bench_c3.err; echo bench_rc=$?; cut -c1-300 gpurun_out/r2y_bench_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2y_launches_c3.csv python bench.py --steps 1 --warmup 0 --iters 20 --no-cpu --no-e2e --no-fft-ref > /dev/null 2>&1; echo ncu_rc=$?
timeout 900 ncu --set full --clock-control none -k regex:"k_rhs_tma|k_wb_tma|k_rows|k_cols" -s 43 -c 14 -o /tmp/r2y_c3 -f python bench.py --steps 1 --warmup 0 --iters 8 --no-e2e --no-cpu --no-fft-ref > /dev/null 2>&1; echo ncu3=$?
python tools/ncu_summary.py /tmp/r2y_c3.ncu-rep > gpurun_out/r2y_ncu_full_c3.txt 2>&1
python tools/ncu_traffic.py /tmp/r2y_c3.ncu-rep gpurun_out/r2y_ncu_traffic.json c3 > /dev/null 2>&1
for c in c1 c2 c4 c5; do timeout 600 python bench.py --config $c --no-cpu --no-fft-ref >> gpurun_out/r2y_bench_configs.jsonl 2>>gpurun_out/r2y_bench_configs.err; done; echo cfg_rc=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2y_bench_reference.json 2>/dev/null; echo ref_rc=$?
du -sh gpurun_out
