# fp64 perturbation ensembles of the C3 final masks on the GPU box's host cores (tools/oracle_masks.py,
# oracle only); records land in gpurun_out/masks/ and are copied into tests/golden/masks/.
export OMP_NUM_THREADS=$(nproc)
mkdir -p gpurun_out/masks
python tools/oracle_masks.py c3 --images 1 0 2 3 --ensemble 3 --out gpurun_out/masks > gpurun_out/masks/c3_ens.log 2>&1
echo rc=$?
tail -20 gpurun_out/masks/c3_ens.log
