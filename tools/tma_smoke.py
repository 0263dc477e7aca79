import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_1212_2845_b200 import from_scene
for sc in (W.block(23, 12, 10), W.walker(16, 8, 8), W.get("C2c")):
    a = from_scene(sc, precision=32, engine="fused"); a.step(20)
    b = from_scene(sc, precision=32, engine="two_pass"); b.step(20)
    sa, sb = a.read_state(), b.read_state()
    disp = np.abs(sb.pos - sc.initial_state()[0]).max()
    print(sc.name, "max pos diff / disp", np.abs(sa.pos - sb.pos).max() / disp, "bitwise", np.array_equal(sa.pos, sb.pos))
