"""Live cost of a broadphase rebuild on C3: one step right after set_state
(which forces a rebuild) versus one ordinary step, both as prepared 1-step
graphs timed with CUDA events on the library's stream."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1212_2845_b200 import from_scene  # noqa: E402

sc = W.hollow_sphere()
lat = from_scene(sc, precision=32)
lat.step(20)
stream = torch.cuda.ExternalStream(lat.stream)
lat.prepare_steps(1)


def one(force):
    if force:
        st = lat.read_state()
        lat.set_state(st.pos, st.quat, st.linmom, st.angmom, st.latch)
        lat.step(1)                                  # pack + rebuild outside the timing
        st = lat.read_state()
        lat.set_state(st.pos, st.quat, st.linmom, st.angmom, st.latch)
        lat.prepare_steps(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    r0 = lat.num_rebuilds
    e0.record(stream)
    lat.step(1)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3, lat.num_rebuilds - r0


plain = [one(False) for _ in range(30)]
reb = [one(True) for _ in range(30)]
p = np.median([t for t, r in plain if r == 0])
q = np.median([t for t, r in reb if r == 1])
print(f"engine {lat.engine}: ordinary step {p:.1f} us, step with rebuild {q:.1f} us, "
      f"rebuild ~{q - p:.1f} us ({sum(r for _, r in reb)} / {len(reb)} rebuilt)")
