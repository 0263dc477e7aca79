"""Sub-box of C5 around a diverging region: does the GPU path diverge, and does
the fp64 oracle diverge at the same step?  python tools/stab_sub.py [zeta]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1212_2845_b200 import DivergedError, from_scene  # noqa: E402

zeta = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
full = W.block()
x0, y0, z0, n = 48, 184, 144, 48
sub = W.Scene("C5-sub", np.ascontiguousarray(full.cells[z0:z0 + n, y0:y0 + n, x0:x0 + n]), full.lattice_dim,
              full.materials, dict(full.env), steps=1200)
NSTEP = int(os.environ.get("NSTEP", "1200"))
sub.env["zeta_bond"] = zeta
sub.env["gravity"] = 9.81
sub.env["floor_on"] = 1
print("materials present:", np.unique(sub.cells, return_counts=True), flush=True)
for prec in (64, 32):
    lat = from_scene(sub, precision=prec, engine="fused")
    done = 0
    try:
        while done < NSTEP:
            lat.step(500)
            done += 500
            st = lat.read_state()
            print(prec, done, f"max|P| {np.abs(st.linmom).max():.3e}", flush=True)
    except DivergedError as e:
        print(prec, "DIVERGED", e, flush=True)
if "--oracle" in sys.argv:
    from oracle import OracleSim
    o = OracleSim(sub.cells, sub.lattice_dim, sub.materials, sub.env, sub.origin)
    o.set_threads(os.cpu_count() or 1)
    o.set_state(*sub.initial_state())
    for s in range(NSTEP // 100):
        try:
            o.step(100)
        except Exception as e:  # noqa: BLE001
            print("oracle DIVERGED near", (s + 1) * 100, e, flush=True)
            break
        st = o.read_state()
        print("oracle", (s + 1) * 100, f"max|P| {np.abs(st.linmom).max():.3e}", flush=True)
