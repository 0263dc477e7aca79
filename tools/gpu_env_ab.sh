# A/B of environment settings on the in-tree library: bash tools/gpu_env_ab.sh "VAR=a" "VAR=b" ...
mkdir -p gpurun_out
for kv in "$@"; do
  for rep in 1 2; do
    env $kv timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --engine fused > gpurun_out/envab.log 2>&1
    python - "$kv" gpurun_out/envab.log <<'PY'
import json, sys
line = [l for l in open(sys.argv[2]) if l.startswith("{")]
d = json.loads(line[-1]) if line else {}
print(sys.argv[1], d.get("ms_per_step"), d.get("value"), d.get("clocks", {}).get("sm_mhz"))
PY
  done
done
