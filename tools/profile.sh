# usage: bash tools/profile.sh <tag>   (one GPU; never multi-rank)
mkdir -p gpurun_out
TAG=${1:-r01}
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo launches rc=$?
$CMD > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bonds|k_integrate" -s 4 -c 2 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo full rc=$?
