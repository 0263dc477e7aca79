"""Run C5 (or a smaller block of its recipe) for many steps and report the step
of divergence, per engine/precision: python tools/c5_long.py ENGINE PREC STEPS [NX]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1212_2845_b200 import DivergedError, from_scene  # noqa: E402

eng, prec, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
nx = int(sys.argv[4]) if len(sys.argv) > 4 else 512
sc = W.block(nx, 256, 256, precision=prec) if nx != 512 else W.block(precision=prec)
lat = from_scene(sc, precision=prec, engine=eng)
print("dt", lat.dt, flush=True)
done = 0
try:
    while done < steps:
        lat.step(50)
        done += 50
        if done % 250 == 0:
            st = lat.read_state()
            v = np.abs(st.linmom).max()
            print(f"step {done}: max|P| {v:.3e} max|phi| {np.abs(st.angmom).max():.3e}", flush=True)
    print(eng, prec, "ok", done)
except DivergedError as e:
    print(eng, prec, "DIVERGED", e)
