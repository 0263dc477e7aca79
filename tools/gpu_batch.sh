# Batched small scenes, x-only packing vs z stacking (fp32, auto engine): bash tools/gpu_batch.sh
mkdir -p gpurun_out
for zs in 1 auto; do
for cfg in "C1 --batch 4096" "C2 --batch 64" "C4 --batch 32" "C3 --batch 16"; do
  name=$(echo $cfg | tr ' ' '_')
  VX_FUSED_TUNE_LOG=1 timeout 300 python bench.py --config $cfg --z-stack $zs --steps 200 --warmup 5 --no-cpu --no-e2e > gpurun_out/batch_${zs}_$name.log 2>&1
  python - "z_stack=$zs $cfg" gpurun_out/batch_${zs}_$name.log <<'PY'
import json, sys
line = [l for l in open(sys.argv[2]) if l.startswith("{")]
d = json.loads(line[-1]) if line else {}
print(sys.argv[1], d.get("config", {}).get("engine"), "us/step", round(d.get("ms_per_step", float("nan")) * 1e3, 2), "value", d.get("value"))
PY
done
done
