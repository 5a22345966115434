# tridiagonal column pass (sr_tri.cuh): solve parity, trajectories, A/B bench on every config
export OMP_NUM_THREADS=$(nproc)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "solve or trajectory_c1 or trajectory_c2 or trajectory_c3 or launch_shape or degenerate or chunking" -p no:cacheprovider > gpurun_out/r2m_tests.log 2>&1; echo tests_rc=$?; tail -5 gpurun_out/r2m_tests.log
B="python bench.py --no-cpu --no-e2e --no-fft-ref --steps 2 --warmup 3"
for c in c3 c4 c5 c2 c1; do
  it=100; [ $c = c5 ] && it=50; [ $c = c1 ] && it=300; [ $c = c2 ] && it=500
  timeout 300 $B --config $c --iters $it > gpurun_out/r2m_${c}_tri.log 2>&1
  SRSB_COLS_TRI=0 timeout 300 $B --config $c --iters $it > gpurun_out/r2m_${c}_fft.log 2>&1
  SRSB_TRI_THREADS=128 timeout 300 $B --config $c --iters $it > gpurun_out/r2m_${c}_tri128.log 2>&1
  SRSB_TRI_THREADS=512 timeout 300 $B --config $c --iters $it > gpurun_out/r2m_${c}_tri512.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2m_c*_*.log')):
    try:
        d=json.loads([l for l in open(f) if l.startswith('{')][-1])
        k=d['roofline'].get('kernels') or {}
        print(f.split('/')[-1], round(d['value']), d['roofline']['step_model']['frac'] if 'step_model' in d['roofline'] else None, {n:round(v['ms_per_launch'],4) for n,v in k.items()})
    except Exception as e:
        print(f, 'ERR', e)
PY
