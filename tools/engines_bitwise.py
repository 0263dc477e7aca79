"""Are the two engines bitwise equal after 150 steps? (fp32 / fp64, several scenes)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, workloads as W
from paper_1212_2845_b200 import from_scene
def flat(st): return np.concatenate([st.pos.ravel(), st.quat.ravel(), st.linmom.ravel(), st.angmom.ravel(), st.latch.astype(float)])
w = W.walker(16, 8, 8); w.env["T_freq"] = 1000.0
for name, sc in [("C2c", W.get("C2c")), ("walker-fast", w), ("block", W.block(37, 9, 11)), ("two-bodies", W.two_bodies()), ("C3", W.hollow_sphere()), ("C1", W.cantilever()), ("tall", W.block(6, 5, 300))]:
    for prec in (32, 64):
        a = from_scene(sc, precision=prec, engine="two_pass"); b = from_scene(sc, precision=prec, engine="fused")
        a.step(150); b.step(150)
        fa, fb = flat(a.read_state()), flat(b.read_state())
        print(name, prec, "bitwise" if np.array_equal(fa, fb) else f"differ max {np.abs(fa-fb).max():.3e}")
