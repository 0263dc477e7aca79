"""C5 fused step time over a (TY, SX) grid, tuning off, best of 3 short regions
(least power-capped): python tools/geo_grid2.py "3,4,5" "8,16,32,64" """
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1212_2845_b200 import from_scene  # noqa: E402

tys = [int(x) for x in sys.argv[1].split(",")]
sxs = [int(x) for x in sys.argv[2].split(",")]
sc = W.block(precision=32)
res = []
for ty in tys:
    for sx in sxs:
        os.environ["VX_FUSED_TY"], os.environ["VX_FUSED_SX"] = str(ty), str(sx)
        lat = from_scene(sc, precision=32, engine="fused", init_state=False)
        lat.step(5)
        lat.prepare_steps(40)
        s = torch.cuda.ExternalStream(lat.stream)
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            lat.step(40)
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 40)
        lat.destroy()
        res.append((min(ts), ty, sx))
        print(f"TY={ty} SX={sx}: best {min(ts) * 1e3:.1f} us/step {[round(t * 1e3, 1) for t in ts]}", flush=True)
res.sort()
print("best:", [(round(t * 1e3, 1), ty, sx) for t, ty, sx in res[:6]])
