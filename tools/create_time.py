"""Set-up time of C5: recipe, vx_create_lattice, set_materials, set_environment,
first step (incl. geometry tuning)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_1212_2845_b200 import Lattice  # noqa: E402

t0 = time.time()
sc = W.block()
t1 = time.time()
lat = Lattice.create_lattice(sc.cells, sc.lattice_dim, sc.origin, 32, 0)
t2 = time.time()
lat.set_materials(sc.materials)
t3 = time.time()
lat.set_environment(sc.env)
lat.set_engine("fused")
t4 = time.time()
lat.step(1)
t5 = time.time()
print(f"recipe {t1-t0:.2f}s create {t2-t1:.2f}s materials {t3-t2:.2f}s env {t4-t3:.2f}s "
      f"first step {t5-t4:.2f}s")
