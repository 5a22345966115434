# r2c warp-shuffle split (bitwise check + A/B), checked build over the new kernels, then the full suite, smoke, bench
export OMP_NUM_THREADS=$(nproc)
echo "hash default   $(python tools/solve_hash.py 1024 1024 3)"
for v in shfl_both shfl_c2r; do echo "hash $v $(SRSB_LIB=vlib/libsrsb_$v.so python tools/solve_hash.py 1024 1024 3)"; done
B="python bench.py --no-cpu --no-e2e --no-fft-ref --steps 2 --warmup 3 --iters 100"
for rep in 1 2; do
  timeout 300 $B > gpurun_out/r2w_c3_base$rep.log 2>&1
  for v in shfl_both shfl_c2r; do SRSB_LIB=vlib/libsrsb_$v.so timeout 300 $B > gpurun_out/r2w_c3_${v}$rep.log 2>&1; done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2w_c3_*.log')):
    d=json.loads([l for l in open(f) if l.startswith('{')][-1]); k=d['roofline']['kernels']
    print(f.split('/')[-1], round(d['value']), {n:round(v['ms_per_launch'],4) for n,v in k.items()})
PY
SRSB_LIB=vlib/libsrsb_checks.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_3d.py tests/test_gpu_slab.py -q -x -k "solve or trajectory_c1 or trajectory_c2 or slab_group or cos_modes" -p no:cacheprovider > gpurun_out/r2w_checked.log 2>&1; echo checked_rc=$?; tail -3 gpurun_out/r2w_checked.log
timeout 3000 python -m pytest tests -m gpu -q -rfE -s -p no:cacheprovider > gpurun_out/r2w_gputests.log 2>&1; echo gputests_rc=$?
grep -E "mask agreement|passed|failed|FAILED|ERROR|xfail" gpurun_out/r2w_gputests.log | tail -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2w_smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/r2w_smoke.log
