"""Per-class device time of one config's step (instrumented, events per launch):
python tools/kernel_split.py C3 [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1212_2845_b200 import from_scene  # noqa: E402

name = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
sc = W.get(name)
lat = from_scene(sc, precision=32, engine="fused")
lat.step(20)
lat.set_instrumentation(True)
lat.step(steps)
kt = lat.kernel_times()
for k, (ms, n) in kt.items():
    print(f"{name} {k:10s} {1e3 * ms / steps:8.2f} us/step  ({n} launches)")
print("rebuilds", lat.num_rebuilds, "pairs", lat.num_contact_pairs, "surface", lat.num_surface)
