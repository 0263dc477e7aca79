mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py --steps 100 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1; python bench.py --steps 100 --warmup 3 --no-cpu --no-e2e --engine two_pass > gpurun_out/bench2.log 2>&1; echo bench rc=$?
