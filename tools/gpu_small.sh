mkdir -p gpurun_out
for cfg in "C1" "C1 --batch 4096" "C2" "C2 --batch 64" "C3" "C4" "C4 --batch 32"; do
  name=$(echo $cfg | tr ' ' '_')
  timeout 300 python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu > gpurun_out/small_$name.log 2>&1
  echo "$cfg rc=$?"
done
