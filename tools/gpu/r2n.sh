# row passes on a row-major spectrum (G = H) vs the transposed layout: per-launch r2c / c2r times (column pass = generic FFT, ignored)
B="python bench.py --no-cpu --no-e2e --no-fft-ref --steps 1 --warmup 3"
run() { name=$1; shift; env "$@" SRSB_COLS_TRI=0 timeout 300 $B > gpurun_out/r2n_$name.log 2>&1; }
B0="$B"
B="$B0 --config c5 --iters 20"; run c5_base X=1; run c5_G4096_r2 SRSB_G=4096 SRSB_RPC=2; run c5_G4096_r1 SRSB_G=4096 SRSB_RPC=1; run c5_G8_r2 SRSB_G=8 SRSB_RPC=2
B="$B0 --config c4 --iters 50"; run c4_base X=1; run c4_G2048_r4 SRSB_G=2048 SRSB_RPC=4; run c4_G2048_r2 SRSB_G=2048 SRSB_RPC=2; run c4_G2048_r1 SRSB_G=2048 SRSB_RPC=1
B="$B0 --config c3 --iters 50"; run c3_base X=1; run c3_G512_r8 SRSB_G=512 SRSB_RPC=8; run c3_G512_r4 SRSB_G=512 SRSB_RPC=4; run c3_G512_r2 SRSB_G=512 SRSB_RPC=2; run c3_G512_r1 SRSB_G=512 SRSB_RPC=1
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2n_*.log')):
    try:
        d=json.loads([l for l in open(f) if l.startswith('{')][-1])
        k=d['roofline'].get('kernels') or {}
        print(f.split('/')[-1], round(d['value']), {n:round(v['ms_per_launch'],4) for n,v in k.items()})
    except Exception as e:
        print(f, 'ERR', e, open(f).read()[-300:])
PY
