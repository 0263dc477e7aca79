import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import workloads as W
from parity import oracle_for
from paper_1212_2845_b200 import from_scene
np.set_printoptions(precision=4, linewidth=200)
def cmp(sc, prec, steps=4):
    lat = from_scene(sc, precision=prec); o = oracle_for(sc)
    print(sc.name, "dt", lat.dt, o.dt)
    for s in range(steps):
        lat.step(1); o.step(1)
        g = lat.read_state(); r = o.read_state()
        print(f"step {s+1}")
        for name in ("pos", "quat", "linmom", "angmom"):
            a, b = getattr(g, name), getattr(r, name)
            if name == "pos": a = a - sc.initial_state()[0]; b = b - sc.initial_state()[0]
            print(" ", name, "maxabs gpu", np.abs(a).max(), "orc", np.abs(b).max(), "diff", np.abs(a-b).max())
        if s == 0:
            print("  P gpu", g.linmom[:6]); print("  P orc", r.linmom[:6])
            print("  phi gpu", g.angmom[:6]); print("  phi orc", r.angmom[:6])
cmp(W.cantilever(), 64)
sc = W.cube(contact_variant=True, n=3); sc.env["gravity"]=0; sc.env["floor_on"]=0
rng = np.random.default_rng(0)
pos, quat, P, phi, latch = sc.initial_state()
P = rng.normal(size=P.shape)*1e-9; phi = rng.normal(size=phi.shape)*1e-16
sc.initial_state = lambda: (pos, quat, P, phi, latch)
cmp(sc, 64, 3)
