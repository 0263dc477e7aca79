# compute-sanitizer over tools/sanitize_cases.py (one GPU): memcheck, racecheck,
# initcheck, synccheck; logs in gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
CASES=${@:-}
for tool in memcheck racecheck initcheck synccheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  timeout 2400 compute-sanitizer --tool $tool $extra --print-limit 200 --error-exitcode 99 \
     python tools/sanitize_cases.py $CASES > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
  tail -3 gpurun_out/sanitize_$tool.log
done
