# round-2: the GPU suite with the per-test parity log
mkdir -p gpurun_out
rm -f gpurun_out/parity_log.jsonl
export VX_PARITY_LOG=$PWD/gpurun_out/parity_log.jsonl
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/b_pytest.log 2>&1; echo pytest rc=$?
tail -40 gpurun_out/b_pytest.log
