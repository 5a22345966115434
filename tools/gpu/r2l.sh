# round-2 status: full GPU suite (no -x: every failure listed), smoke, default bench line, launch list, all configs
export OMP_NUM_THREADS=$(nproc)
timeout 2400 python -m pytest tests -m gpu -q -rfE -s -p no:cacheprovider > gpurun_out/r2l_gputests.log 2>&1; echo gputests_rc=$?
grep -E "mask agreement|passed|failed|FAILED|ERROR" gpurun_out/r2l_gputests.log | tail -40
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/r2l_smoke.log
timeout 900 python bench.py > gpurun_out/r2l_bench_c3.json 2> gpurun_out/r2l_bench_c3.err; echo bench_rc=$?; cat gpurun_out/r2l_bench_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2l_launches_c3.csv python bench.py --steps 1 --warmup 0 --iters 20 --no-cpu --no-e2e --no-fft-ref > /dev/null 2>&1; echo ncu_rc=$?
for c in c1 c2 c4 c5; do timeout 600 python bench.py --config $c --no-cpu --no-fft-ref >> gpurun_out/r2l_bench_configs.jsonl 2>>gpurun_out/r2l_bench_configs.err; done; echo cfg_rc=$?
cat gpurun_out/r2l_bench_configs.jsonl | cut -c1-400
