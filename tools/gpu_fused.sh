mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fused.py -q -p no:cacheprovider -x > gpurun_out/pytest_fused.log 2>&1; echo pytest rc=$?
