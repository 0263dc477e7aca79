# Both engines on the small configs (fp32): bash tools/gpu_engines.sh
mkdir -p gpurun_out
for eng in fused two_pass; do
for cfg in "C1" "C1 --batch 4096" "C2" "C2 --batch 64" "C3" "C4" "C4 --batch 32"; do
  name=$(echo $cfg | tr ' ' '_')
  timeout 300 python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu --no-e2e --engine $eng > gpurun_out/eng_${eng}_$name.log 2>&1
  python - "$eng $cfg" gpurun_out/eng_${eng}_$name.log <<'PY'
import json, sys
line = [l for l in open(sys.argv[2]) if l.startswith("{")]
d = json.loads(line[-1]) if line else {}
print(sys.argv[1], "us/step", round(d.get("ms_per_step", float("nan")) * 1e3, 2), "value", d.get("value"))
PY
done
done
