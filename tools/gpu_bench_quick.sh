mkdir -p gpurun_out
timeout 900 python bench.py --steps ${STEPS:-200} --warmup 5 ${@} > gpurun_out/bq.log 2>&1; echo bench rc=$?
tail -c 3000 gpurun_out/bq.log
