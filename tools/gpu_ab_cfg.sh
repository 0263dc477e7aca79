# A/B of library variants on small configs: bash tools/gpu_ab_cfg.sh "C1 C2c C4" lib1 lib2 ...
mkdir -p gpurun_out
cfgs=$1; shift
for n in "$@"; do
  cp .exp/$n.so paper_1212_2845_b200/libvoxsim.so
  touch paper_1212_2845_b200/libvoxsim.so
  for c in $cfgs; do
    for rep in 1 2; do
      timeout 300 python bench.py --config $c --steps 3000 --warmup 30 --no-cpu --no-e2e --engine fused > gpurun_out/abc.log 2>&1
      python - "$n $c" gpurun_out/abc.log <<'PY'
import json, sys
line = [l for l in open(sys.argv[2]) if l.startswith("{")]
d = json.loads(line[-1]) if line else {}
print(sys.argv[1], round(1e3 * d.get("ms_per_step", 0), 2), "us/step")
PY
    done
  done
done
