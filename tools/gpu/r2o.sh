# row-major spectrum + k_cols_tri_rm: solve parity, trajectories, A/B bench
export OMP_NUM_THREADS=$(nproc)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "solve or trajectory_c1 or trajectory_c2 or trajectory_c3 or launch_shape or degenerate or chunking" -p no:cacheprovider > gpurun_out/r2o_tests.log 2>&1; echo tests_rc=$?; tail -5 gpurun_out/r2o_tests.log
B="python bench.py --no-cpu --no-e2e --no-fft-ref --steps 2 --warmup 3"
for c in c3 c4 c5 c2 c1; do
  it=100; [ $c = c5 ] && it=50; [ $c = c1 ] && it=300; [ $c = c2 ] && it=500
  timeout 300 $B --config $c --iters $it > gpurun_out/r2o_${c}_rm.log 2>&1
  SRSB_SPEC_RM=0 timeout 300 $B --config $c --iters $it > gpurun_out/r2o_${c}_tr.log 2>&1
  SRSB_TRI_W=8 timeout 300 $B --config $c --iters $it > gpurun_out/r2o_${c}_rm_w8.log 2>&1
  SRSB_RPC=2 timeout 300 $B --config $c --iters $it > gpurun_out/r2o_${c}_rm_rpc2.log 2>&1
  SRSB_RPC_INV=2 timeout 300 $B --config $c --iters $it > gpurun_out/r2o_${c}_rm_inv2.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/r2o_c*_*.log')):
    try:
        d=json.loads([l for l in open(f) if l.startswith('{')][-1])
        k=d['roofline'].get('kernels') or {}
        print(f.split('/')[-1], round(d['value']), round(d['roofline']['step_model']['frac'],4), {n:round(v['ms_per_launch'],4) for n,v in k.items()})
    except Exception as e:
        print(f, 'ERR', e, open(f).read()[-300:])
PY
