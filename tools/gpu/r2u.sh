# c2r variants on the row-major layout: accumulation source loaded late / own-row L2 prefetch / register caps
B="python bench.py --no-cpu --no-e2e --no-fft-ref --steps 2 --warmup 3"
for v in base c2r_late c2r_late_pf c2r_late_m10 c2r_m10; do
  L=""; [ $v != base ] && L="SRSB_LIB=vlib/libsrsb_$v.so"
  for c in c3 c4 c5; do
    case $v in *m10) [ $c != c3 ] && continue;; esac
    it=100; [ $c = c5 ] && it=50
    env $L timeout 300 $B --config $c --iters $it > gpurun_out/r2u_${c}_$v.log 2>&1
  done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2u_c*_*.log')):
    try:
        d=json.loads([l for l in open(f) if l.startswith('{')][-1])
        k=d['roofline'].get('kernels') or {}
        print(f.split('/')[-1], round(d['value']), round(d['roofline']['step_model']['frac'],4), {n:round(v['ms_per_launch'],4) for n,v in k.items()})
    except Exception as e:
        print(f, 'ERR', e, open(f).read()[-300:])
PY
