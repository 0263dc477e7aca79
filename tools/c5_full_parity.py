"""C5 at full size (512 x 256 x 256, 33.5M voxels) against the fp64 oracle:
100 steps from a strained start (workloads.strained, floor contact on), the
GPU in the bench's launch configuration (fused engine, CUDA-graph chunks) in
fp32 and fp64, the oracle on the host cores (~10 min, ~30 GB).  Prints and
writes the parity errors of tests/parity.py (SURVEY 8(c) normaliser).
    python tools/c5_full_parity.py [steps] [out.json]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from paper_1212_2845_b200 import from_scene  # noqa: E402
from parity import TOL, TOL_QPPHI, errors, oracle_for  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
out_path = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "c5_full_parity.json")
sc = W.block(precision=32)
st0 = W.strained(sc, seed=11, lift=False)
res = {"workload": "C5 512x256x256, strained start (workloads.strained seed 11, floor contact)",
       "steps": steps, "voxels": sc.num_voxels}
gpu = {}
for prec in (32, 64):
    t = time.time()
    lat = from_scene(sc, precision=prec, engine="fused", init_state=False)
    lat.set_state(*st0)
    lat.step(3)                    # bench-style: a short chunk, then graph chunks
    lat.step(steps - 3)
    gpu[prec] = lat.read_state()
    res[f"gpu_fp{prec}_dt"] = lat.dt
    res[f"gpu_fp{prec}_s"] = time.time() - t
    lat.destroy()
    print(f"gpu fp{prec} done in {time.time() - t:.1f} s", flush=True)
t = time.time()
o = oracle_for(sc, state=st0)
res["oracle_create_s"] = time.time() - t
res["oracle_dt"] = o.dt
assert res["gpu_fp32_dt"] == o.dt and res["gpu_fp64_dt"] == o.dt
t = time.time()
o.step(steps)
res["oracle_step_s"] = time.time() - t
res["oracle_threads"] = os.cpu_count()
r = o.read_state()
print(f"oracle {steps} steps in {res['oracle_step_s']:.0f} s", flush=True)
for prec in (64, 32):
    e = errors(gpu[prec], r, st0[0], sc.lattice_dim, prec, init=st0)
    e["bar_eD"] = TOL[prec]
    e["bar_qPphi"] = TOL_QPPHI[prec]
    e["pass"] = bool(e["eD"] <= TOL[prec] and max(e["eq"], e["eP"], e["ephi"]) <= TOL_QPPHI[prec]
                     and e["latch_flips"] == 0)
    res[f"fp{prec}"] = e
    print(f"fp{prec}: {e}", flush=True)
res["floor_contact_voxels_end"] = int(np.count_nonzero(r.pos[:, 2] < 0.5 * sc.lattice_dim))
res["latched_end"] = int(np.count_nonzero(r.latch))
json.dump(res, open(out_path, "w"), indent=1)
print(json.dumps(res))
