"""Long runs of the configs (and C5 variants) to check the damped step's stability:
python tools/stab.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1212_2845_b200 import DivergedError, from_scene  # noqa: E402


def run(sc, steps, prec=32, chunk=500):
    lat = from_scene(sc, precision=prec, engine="fused" if sc.cells.shape[0] >= 32 else "two_pass")
    done = 0
    p0 = None
    try:
        while done < steps:
            n = min(chunk, steps - done)
            lat.step(n)
            done += n
        st = lat.read_state()
        return f"ok {done} max|P| {np.abs(st.linmom).max():.3e}"
    except DivergedError as e:
        return f"DIVERGED {e}"
    finally:
        lat.destroy()


which = sys.argv[1:] or ["C2", "C2c", "C4", "C5z1", "C5z09", "C5z05"]
for name in which:
    if name.startswith("C5"):
        z = {"C5z1": 1.0, "C5z09": 0.9, "C5z08": 0.8, "C5z05": 0.5}[name]
        sc = W.block(128, 256, 256)
        sc.env["zeta_bond"] = z
        print(name, run(sc, 3000), flush=True)
    elif name == "homog":
        sc = W.block(128, 256, 256)
        sc.cells[:] = 1
        print(name, run(sc, 3000), flush=True)
    else:
        sc = W.get(name)
        print(name, run(sc, sc.steps), flush=True)
