import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_1212_2845_b200 import from_scene
for prec in (32, 64):
    for zb in (0.0, 1.0):
        sc = W.cantilever(n=20, force=3e-5, zeta_ground=0.003)
        sc.env['zeta_bond'] = zb
        lat = from_scene(sc, precision=prec)
        res = []
        for blk in range(16):
            lat.step(10000)
            st = lat.read_state()
            res.append(np.abs(st.linmom).max() / 1e-6)
        # jitter of the tip over the last 2000 steps
        z = []
        for s in range(200):
            lat.step(10); z.append(lat.read_state().pos[-1, 2])
        print(prec, zb, ['%.1e' % r for r in res], 'tip z std %.2e' % np.std(z))
