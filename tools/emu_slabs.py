"""Step time of C5 with P emulated x-slabs on one GPU (per-slab launch split of
the NCCL ranks, run back to back): python tools/emu_slabs.py P [P ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1212_2845_b200 import from_scene  # noqa: E402

sc = W.block(precision=32)
for P in map(int, sys.argv[1:]):
    lat = from_scene(sc, precision=32, nranks=P, engine="fused")
    lat.step(10)
    s = torch.cuda.ExternalStream(lat.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    lat.step(50)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    lat.set_instrumentation(True)
    lat.step(10)
    kt = lat.kernel_times()
    lat.set_instrumentation(False)
    print(f"P={P}: {ms:.3f} ms/step (sum over slabs); per step: fused {kt['integrate'][0] / 10:.3f} ms "
          f"in {kt['integrate'][1] // 10} launches, other {kt['other'][0] / 10:.3f} ms", flush=True)
    lat.destroy()
