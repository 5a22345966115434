# one-kernel cluster solve for small images: parity, C1 / C2 masks, bench; slab + fused suites with their pinned variants
export OMP_NUM_THREADS=$(nproc)
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "solve or trajectory_c1 or trajectory_c2 or degenerate or chunking or c1_final or c2_final or monitor or band_skip or launch_shape or iterate_until or host_buffers or nonfinite" -p no:cacheprovider -s > gpurun_out/r2r_tests.log 2>&1; echo tests_rc=$?; grep -E "mask agreement|passed|failed|FAILED|ERROR" gpurun_out/r2r_tests.log | tail
timeout 900 python -m pytest tests/test_gpu_slab.py tests/test_gpu_fused.py tests/test_gpu_checkpoint.py tests/test_gpu_aos.py -q -p no:cacheprovider > gpurun_out/r2r_tests2.log 2>&1; echo tests2_rc=$?; tail -3 gpurun_out/r2r_tests2.log
timeout 120 python tools/launch_floor.py > gpurun_out/r2r_launch_floor.json 2>&1; cat gpurun_out/r2r_launch_floor.json
B="python bench.py --no-cpu --no-e2e --no-fft-ref --steps 3 --warmup 3"
for c in c1 c2; do
  timeout 300 $B --config $c > gpurun_out/r2r_${c}_cl.log 2>&1
  SRSB_SOLVE_CL=0 timeout 300 $B --config $c > gpurun_out/r2r_${c}_nocl.log 2>&1
  SRSB_SOLVE_CL=5 timeout 300 $B --config $c > gpurun_out/r2r_${c}_cl5.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2r_c*_*.log')):
    try:
        d=json.loads([l for l in open(f) if l.startswith('{')][-1])
        k=d['roofline'].get('kernels') or {}
        print(f.split('/')[-1], round(d['value']), d['ms_per_step'], {n:round(v['ms_per_launch'],4) for n,v in k.items()})
    except Exception as e:
        print(f, 'ERR', e, open(f).read()[-300:])
PY
