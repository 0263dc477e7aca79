import sys, os, numpy as np
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import workloads as W
from parity import oracle_for
from paper_1212_2845_b200 import from_scene
np.set_printoptions(precision=5, linewidth=220)
def show(sc, ids):
    o = oracle_for(sc); g = from_scene(sc, precision=32)
    o.step(1); g.step(1)
    r = o.read_state(); a = g.read_state()
    mats = sc.cells.ravel()[sc.cells.ravel() > 0]
    for i in ids:
        print(i, sc.voxel_coords()[i], mats[i], "gpu", a.linmom[i], "orc", r.linmom[i])
sc = W.cube(); show(sc, list(range(0, 25)) + [399, 400, 7999])
sc = W.cube(n=3); show(sc, range(27))
