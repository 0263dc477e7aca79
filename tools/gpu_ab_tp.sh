# A/B of library variants on the two-pass engine: bash tools/gpu_ab_tp.sh name1 name2 ...
mkdir -p gpurun_out
for n in "$@"; do
  cp .exp/$n.so paper_1212_2845_b200/libvoxsim.so
  touch paper_1212_2845_b200/libvoxsim.so
  for rep in 1 2; do
    timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --engine two_pass > gpurun_out/abtp_$n.$rep.log 2>&1
    python - "$n" gpurun_out/abtp_$n.$rep.log <<'PY'
import json, sys
line = [l for l in open(sys.argv[2]) if l.startswith("{")]
d = json.loads(line[-1]) if line else {}
k = d.get("roofline", {}).get("kernels", {})
print(sys.argv[1], d.get("ms_per_step"), {a: round(b["ms_per_step"], 4) for a, b in k.items()})
PY
  done
done
