# Collision kernels of C3 (self collision): launch list past the tuners, and one
# `ncu --set full` capture each of k_contact and a rebuilding k_broadphase.
mkdir -p gpurun_out
TAG=${1:-r12}
CMD="python bench.py --config C3 --steps 300 --warmup 3 --no-cpu --no-e2e --engine fused"
$CMD > gpurun_out/c3_plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 1400 -c 1200 --csv \
  --log-file gpurun_out/c3_launches_$TAG.csv $CMD > gpurun_out/c3_ncu_launch_$TAG.log 2>&1
echo launches rc=$?
ncu --set full --clock-control none -k regex:"k_contact|k_broadphase" -s 600 -c 6 \
  -o gpurun_out/c3_prof_$TAG $CMD > gpurun_out/c3_ncu_full_$TAG.log 2>&1
echo full rc=$?
