# round-2 evidence run (one GPU): GPU suite (+ parity log), checked suite, bench,
# ncu launch list of the bench command and one --set full capture of the fused pass
mkdir -p gpurun_out
TAG=${1:-r14}
export VX_PARITY_LOG=$PWD/gpurun_out/${TAG}_parity_log.jsonl
rm -f $VX_PARITY_LOG
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/${TAG}_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/${TAG}_pytest.log
unset VX_PARITY_LOG
VX_LIB=checked timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_checked_pytest.log 2>&1; echo checked rc=$?; tail -1 gpurun_out/${TAG}_checked_pytest.log
VX_LIB=checked timeout 900 python tools/sanitize_cases.py > gpurun_out/${TAG}_checked_cases.log 2>&1; echo cases rc=$?
for c in n96 n96_ty1 tall300; do VX_LIB=oldparity timeout 300 python tools/sanitize_cases.py $c > gpurun_out/${TAG}_oldparity_$c.log 2>&1; echo "oldparity $c rc=$? $(grep -o 'device check failed.*' gpurun_out/${TAG}_oldparity_$c.log | head -1)"; done
timeout 900 python bench.py --steps 200 --warmup 5 > gpurun_out/${TAG}_bench.log 2>&1; echo bench rc=$?
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --repeats 1"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo launches rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k_step_fused" -s 3 -c 1 -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1; echo full rc=$?
