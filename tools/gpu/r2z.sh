# C5 mask at K = 100; A/B of the late + prefetched accumulation source in the warp-shuffle c2r
export OMP_NUM_THREADS=$(nproc)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "c5_masks" -p no:cacheprovider > gpurun_out/r2z_masks.log 2>&1; echo masks_rc=$?; grep -E "mask agreement|passed|failed" gpurun_out/r2z_masks.log
echo "hash default $(python tools/solve_hash.py 1024 1024 3)"; echo "hash c2r_sl  $(SRSB_LIB=vlib/libsrsb_c2r_sl.so python tools/solve_hash.py 1024 1024 3)"
B="python bench.py --no-cpu --no-e2e --no-fft-ref --steps 2 --warmup 3 --iters 100"
for rep in 1 2; do
  timeout 300 $B > gpurun_out/r2z_c3_base$rep.log 2>&1
  SRSB_LIB=vlib/libsrsb_c2r_sl.so timeout 300 $B > gpurun_out/r2z_c3_sl$rep.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2z_c3_*.log')):
    d=json.loads([l for l in open(f) if l.startswith('{')][-1]); k=d['roofline']['kernels']
    print(f.split('/')[-1], round(d['value']), {n:round(v['ms_per_launch'],4) for n,v in k.items()})
PY
