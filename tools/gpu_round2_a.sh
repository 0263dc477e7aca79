# round-2 first pass: GPU tests + a quick bench (one GPU)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/a_pytest.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu > gpurun_out/a_bench.log 2>&1; echo bench rc=$?
tail -3 gpurun_out/a_pytest.log
