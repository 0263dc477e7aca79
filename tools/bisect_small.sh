for d in .wt/c6cf467 .wt/3c2869e .wt/285e1c1 .wt/1d9abe4 .; do
  for cfg in C1 C2 C4; do
    (cd $d && timeout 300 python bench.py --config $cfg --engine fused --steps 2000 --warmup 5 --no-cpu --no-e2e 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$d', '$cfg', round(d['ms_per_step']*1e3,2))")
  done
done
