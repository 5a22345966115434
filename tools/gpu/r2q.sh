# full GPU suite on the tridiagonal / row-major build; C1 / C2 with the fused RHS + row-R2C kernel (one launch fewer per sweep)
export OMP_NUM_THREADS=$(nproc)
B="python bench.py --no-cpu --no-e2e --no-fft-ref --steps 3 --warmup 3"
for c in c1 c2; do
  timeout 300 $B --config $c > gpurun_out/r2q_${c}_base.log 2>&1
  SRSB_FUSE=1 timeout 300 $B --config $c > gpurun_out/r2q_${c}_fuse.log 2>&1
  SRSB_TMA=0 timeout 300 $B --config $c > gpurun_out/r2q_${c}_notma.log 2>&1
  SRSB_GRAPH=0 timeout 300 $B --config $c > gpurun_out/r2q_${c}_nograph.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2q_c*_*.log')):
    try:
        d=json.loads([l for l in open(f) if l.startswith('{')][-1])
        k=d['roofline'].get('kernels') or {}
        print(f.split('/')[-1], round(d['value']), d['ms_per_step'], {n:round(v['ms_per_launch'],4) for n,v in k.items()})
    except Exception as e:
        print(f, 'ERR', e, open(f).read()[-300:])
PY
timeout 3000 python -m pytest tests -m gpu -q -rfE -s -p no:cacheprovider > gpurun_out/r2q_gputests.log 2>&1; echo gputests_rc=$?
grep -E "mask agreement|passed|failed|FAILED|ERROR|xfail" gpurun_out/r2q_gputests.log | tail -40
