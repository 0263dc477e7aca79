"""C5 fused step time over an explicit (TY, SX) grid (tuning off):
python tools/geo_grid.py "5,6,7,8" "8,10,12,14,16,20,24,32" """
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1212_2845_b200 import from_scene  # noqa: E402

tys = [int(x) for x in sys.argv[1].split(",")]
sxs = [int(x) for x in sys.argv[2].split(",")]
sc = W.block(precision=32)
for ty in tys:
    for sx in sxs:
        os.environ["VX_FUSED_TY"], os.environ["VX_FUSED_SX"] = str(ty), str(sx)
        lat = from_scene(sc, precision=32, engine="fused")
        lat.step(5)
        s = torch.cuda.ExternalStream(lat.stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        lat.step(60)
        e1.record(s)
        torch.cuda.synchronize()
        print(f"TY={ty} SX={sx}: {e0.elapsed_time(e1) / 60 * 1e3:.1f} us/step", flush=True)
        lat.destroy()
