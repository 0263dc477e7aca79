mkdir -p gpurun_out
timeout 600 python bench.py --steps 100 --warmup 3 --no-cpu --no-e2e ${@} > gpurun_out/benchq.log 2>&1; echo bench rc=$?
