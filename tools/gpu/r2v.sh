# 3-D lines solve (FFT j, FFT i, tridiagonal z): parity, bench vs the plane solve; C4 / C5 truncated-horizon masks
export OMP_NUM_THREADS=$(nproc)
timeout 1200 python -m pytest tests/test_gpu_3d.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/r2v_3d.log 2>&1; echo t3d_rc=$?; tail -5 gpurun_out/r2v_3d.log
timeout 300 python bench.py --config v3d --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2v_v3d_lines.json 2> gpurun_out/r2v_v3d_lines.err; echo rc=$?
SRSB_VOL_SOLVE=plane timeout 300 python bench.py --config v3d --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2v_v3d_plane.json 2> gpurun_out/r2v_v3d_plane.err; echo rc=$?
python - <<'PY'
import json
for n in ("lines","plane"):
    try:
        d=json.loads([l for l in open(f'gpurun_out/r2v_v3d_{n}.json') if l.startswith('{')][-1])
        print(n, round(d['value']), {k:round(v['ms_per_launch'],4) for k,v in (d['roofline'].get('kernels') or {}).items()})
    except Exception as e: print(n,'ERR',e, open(f'gpurun_out/r2v_v3d_{n}.err').read()[-500:])
PY
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -k "truncated" -s -p no:cacheprovider > gpurun_out/r2v_masks.log 2>&1; echo masks_rc=$?; grep -E "mask agreement|passed|failed" gpurun_out/r2v_masks.log
