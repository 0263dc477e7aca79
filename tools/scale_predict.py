"""Per-rank time of C5's x-slabs, measured on one GPU, for DESIGN.md §7's
multi-GPU prediction:
  * the whole lattice (N = 1), fused step;
  * one rank's slab as its own lattice (512/P planes; what a rank computes,
    without the boundary-plane split);
  * P emulated slabs in one process (the NCCL ranks' launches -- interior pass
    plus the two boundary planes -- run back to back; step / P = the mean
    per-rank time with the split, without the overlap the comm stream gives);
prints ms per step and the implied efficiency t_1 / (P t_rank).
    python tools/scale_predict.py [P ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1212_2845_b200 import from_scene  # noqa: E402


def timed(lat, steps=60, warm=10):
    lat.step(warm)
    lat.prepare_steps(steps)
    s = torch.cuda.ExternalStream(lat.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    lat.step(steps)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


out = {}
full = from_scene(W.block(), precision=32, engine="fused", init_state=False)
t1 = timed(full)
full.destroy()
out["t1_ms"] = t1
for P in map(int, sys.argv[1:] or ["2", "4", "8"]):
    nx = 512 // P
    lat = from_scene(W.block(nx, 256, 256), precision=32, engine="fused", init_state=False)
    tr = timed(lat)
    lat.destroy()
    emu = from_scene(W.block(), precision=32, engine="fused", init_state=False, nranks=P)
    te = timed(emu)
    emu.destroy()
    out[P] = dict(slab_ms=tr, emulated_step_ms=te, emulated_per_rank_ms=te / P,
                  eff_slab=t1 / (P * tr), eff_emulated=t1 / te)
    print(f"P={P}: slab-as-lattice {tr * 1e3:.1f} us, emulated {te * 1e3:.1f} us / step "
          f"({te / P * 1e3:.1f} per rank); t1 {t1 * 1e3:.1f} us -> efficiency "
          f"{t1 / (P * tr):.3f} (slab) / {t1 / te:.3f} (emulated split)", flush=True)
print(json.dumps(out))
