"""C5 fused step time of the library in place (A/B of build variants):
python tools/ab_time.py [label]  -- median of 3 regions of 100 steps."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1212_2845_b200 import from_scene  # noqa: E402

lat = from_scene(W.block(), precision=32, engine="fused", init_state=False)
lat.step(10)
lat.prepare_steps(100)
s = torch.cuda.ExternalStream(lat.stream)
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    lat.step(100)
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 100)
print(f"{sys.argv[1] if len(sys.argv) > 1 else ''}: {np.median(ts) * 1e3:.1f} us/step  {[round(t * 1e3, 1) for t in ts]}",
      flush=True)
