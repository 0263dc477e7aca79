# bench.py over the other configs / options (one GPU): one JSON line each
mkdir -p gpurun_out
for a in "--config C1" "--config C2c" "--config C3" "--config C4" "--config C4 --batch 32" "--config C1 --batch 4096" "--precision 64" "--impl reference --steps 3"; do
  timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu $a > /tmp/b.log 2>&1; rc=$?
  python - "$a" "$rc" <<'PY'
import json, sys
a, rc = sys.argv[1], sys.argv[2]
line = [l for l in open("/tmp/b.log") if l.startswith("{")]
if not line:
    print(a, "rc", rc, open("/tmp/b.log").read()[-500:]); sys.exit()
d = json.loads(line[-1])
r = d.get("roofline") or {}
print(f"{a:28s} rc={rc} value={d['value']:.3e} ms/step={d['ms_per_step']:.4f} engine={d['config'].get('engine')} "
      f"frac={r.get('frac', float('nan')):.3f} e2e={(d.get('e2e') or {}).get('value', 0):.3e} digest={(d.get('e2e') or {}).get('final_state_digest')}")
PY
done
