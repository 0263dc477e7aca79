mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_owned_io.py tests/test_gpu_bench_contract.py -q -p no:cacheprovider > gpurun_out/c_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/c_pytest.log
timeout 900 python tools/scale_predict.py 2 4 8 > gpurun_out/c_scale.log 2>&1; echo scale rc=$?; cat gpurun_out/c_scale.log
