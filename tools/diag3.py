import sys, os, numpy as np
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import workloads as W
from parity import oracle_for
from paper_1212_2845_b200 import from_scene
np.set_printoptions(precision=4, linewidth=200)
sc = W.cube()
p0 = sc.initial_state()[0]
o = oracle_for(sc); g32 = from_scene(sc, precision=32); g64 = from_scene(sc, precision=64)
done = 0
for n in (1, 2, 5, 10, 30, 100):
    k = n - done; done = n
    o.step(k); g32.step(k); g64.step(k)
    r = o.read_state(); a = g32.read_state(); b = g64.read_state()
    du = r.pos - p0
    print(n, "orc |u|max", np.abs(du).max(), "mean uz", du[:,2].mean(), "std uz", du[:,2].std())
    for nm, s in (("f32", a), ("f64", b)):
        e = np.abs(s.pos - r.pos); i = np.argmax(e.max(1))
        print("  ", nm, "pos err max", e.max(), "at", i, "P err", np.abs(s.linmom - r.linmom).max(), "P orc max", np.abs(r.linmom).max(), "phi err", np.abs(s.angmom-r.angmom).max(), "phi orc", np.abs(r.angmom).max())
