"""Time the phases of bench's end-to-end episode (set_state, step(K), read_state)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1212_2845_b200 import State, from_scene  # noqa: E402

sc = W.block(precision=32)
lat = from_scene(sc, precision=32, engine="fused")
lat.step(5)
st0 = sc.initial_state()
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa
hin = [pin(a) for a in st0]
hout = State(*[pin(np.empty_like(a)) for a in st0])
for rep in range(3):
    t0 = time.perf_counter(); lat.set_state(*hin); t1 = time.perf_counter()
    lat.set_step(0); lat.step(200); t2 = time.perf_counter()
    lat.read_state(hout); t3 = time.perf_counter()
    print(f"set_state {1e3*(t1-t0):.1f} ms  step(200) {1e3*(t2-t1):.1f} ms  read_state {1e3*(t3-t2):.1f} ms", flush=True)
