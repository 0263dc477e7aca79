# bash tools/gpu_env_cfg.sh CONFIG "VAR=a ..." "VAR=b ..." : bench step time of CONFIG per env setting
mkdir -p gpurun_out
cfg=$1; shift
for kv in "$@"; do
  env $kv timeout 300 python bench.py --config $cfg --steps 2000 --warmup 20 --no-cpu --no-e2e --engine fused > gpurun_out/envcfg.log 2>&1
  python - "$cfg $kv" gpurun_out/envcfg.log <<'PY'
import json, sys
line = [l for l in open(sys.argv[2]) if l.startswith("{")]
d = json.loads(line[-1]) if line else {}
print(sys.argv[1], round(1e3 * d.get("ms_per_step", 0), 2), "us/step", d.get("value"))
PY
done
