# The (y, z)-mapped fused pass on 32 packed walkers (1,048,576 voxels, nz = 16):
# one `ncu --set full` capture past the tuner.
mkdir -p gpurun_out
TAG=${1:-r13}
CMD="python bench.py --config C4 --batch 32 --engine fused --steps 40 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/yz_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_step_fused_yz" -s 400 -c 1 \
  -o gpurun_out/yz_prof_$TAG $CMD > gpurun_out/yz_ncu_full_$TAG.log 2>&1
echo full rc=$?
