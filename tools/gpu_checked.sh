# The GPU suite on the checked build (device bounds checks + shared-memory race
# tags, vx_common.cuh), the sanitize cases on it, and the race probe's positive
# control (round 1's zrec parity restored) -- compute-sanitizer is closed on this pool.
mkdir -p gpurun_out
VX_LIB=checked timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/checked_pytest.log 2>&1; echo checked pytest rc=$?
tail -4 gpurun_out/checked_pytest.log
VX_LIB=checked timeout 900 python tools/sanitize_cases.py > gpurun_out/checked_cases.log 2>&1; echo checked cases rc=$?
tail -3 gpurun_out/checked_cases.log
for c in n96 n96_ty1 tall300 c2c; do
  VX_LIB=oldparity timeout 300 python tools/sanitize_cases.py $c > gpurun_out/oldparity_$c.log 2>&1; echo "oldparity $c rc=$?"
  tail -2 gpurun_out/oldparity_$c.log
done
