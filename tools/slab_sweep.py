"""Per-rank fused-step time of one x-slab of C5 (nx planes of 256 x 256) for
launch-geometry settings: python tools/slab_sweep.py NX [NX ...]
(env VX_FUSED_WAVES / VX_FUSED_TY are read at lattice creation)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1212_2845_b200 import from_scene  # noqa: E402


def run(nx, steps=100):
    sc = W.block(nx, 256, 256)
    lat = from_scene(sc, precision=32, engine="fused")
    lat.step(10)
    s = torch.cuda.ExternalStream(lat.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    lat.step(steps)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    lat.destroy()
    return ms, sc.num_voxels


waves_list = [int(x) for x in os.environ.get("SWEEP_WAVES", "1,2,4").split(",")]
sx_list = [os.environ.get("VX_FUSED_TUNE", "1")]
for nx in map(int, sys.argv[1:]):
    for waves in waves_list:
        for sxm in sx_list:
            os.environ["VX_FUSED_WAVES"], os.environ["VX_FUSED_TUNE"] = str(waves), str(sxm)
            ms, n = run(nx)
            print(f"nx={nx} waves={waves} tune={sxm}: {ms * 1e3:.1f} us/step, {n * 1e3 / ms:.3e} voxel-steps/s")
