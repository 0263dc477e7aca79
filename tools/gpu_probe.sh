mkdir -p gpurun_out
for c in n96 n96_ty1 tall300; do
  VX_LIB=oldparity timeout 300 python tools/sanitize_cases.py $c > gpurun_out/oldparity_$c.log 2>&1; echo "oldparity $c rc=$?"
  tail -2 gpurun_out/oldparity_$c.log
  VX_LIB=checked timeout 300 python tools/sanitize_cases.py $c > gpurun_out/checked_$c.log 2>&1; echo "checked $c rc=$?"
  tail -1 gpurun_out/checked_$c.log
done
