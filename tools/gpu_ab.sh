# A/B timing of library variants: bash tools/gpu_ab.sh name1 name2 ... (libs in .exp/<name>.so)
mkdir -p gpurun_out
for n in "$@"; do
  cp .exp/$n.so paper_1212_2845_b200/libvoxsim.so
  touch paper_1212_2845_b200/libvoxsim.so
  for rep in 1 2; do
    timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --engine fused > gpurun_out/ab_$n.$rep.log 2>&1
    python - "$n" gpurun_out/ab_$n.$rep.log <<'PY'
import json, sys
line = [l for l in open(sys.argv[2]) if l.startswith("{")]
d = json.loads(line[-1]) if line else {}
print(sys.argv[1], d.get("ms_per_step"), d.get("value"), d.get("clocks", {}).get("sm_mhz"))
PY
  done
done
