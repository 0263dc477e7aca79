import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_1212_2845_b200 import from_scene
np.set_printoptions(precision=5, linewidth=200)
sc = W.cube(contact_variant=True, n=3)
for prec in (64, 32):
    lat = from_scene(sc, precision=prec)
    g = lat.read_state()
    pos, quat, P, phi, latch = sc.initial_state()
    print(prec, "roundtrip pos", np.abs(g.pos-pos).max(), "quat", np.abs(g.quat-quat).max(), "P", np.abs(g.linmom-P).max())
    print(g.quat[:4]); print(g.pos[:4]); print(pos[:4])
    v = lat.read_voxels(np.arange(4)); print("rv", v.quat, v.pos)
