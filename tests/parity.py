"""Helpers shared by the GPU parity tests: run a scene through the CUDA path
(C ABI via the binding) and through the fp64 oracle on the same seeded input,
and measure the normalised position error of SURVEY §8(c):

    e_D = max_i |D_i^gpu - D_i^orc| / max(max_i |D_i^orc - D_i^0|, 1e-9 l)
"""
import os

import numpy as np

from oracle import OracleSim
from paper_1212_2845_b200 import from_scene

THREADS = os.cpu_count() or 1


def oracle_for(scene, threads=THREADS):
    o = OracleSim(scene.cells, scene.lattice_dim, scene.materials, scene.env, scene.origin)
    o.set_threads(threads)
    if scene.fixed is not None or scene.fext is not None:
        o.set_boundary(scene.fixed, scene.fext)
    for kind, org, size, force in scene.extra.get("regions", []):
        o.add_region(kind, org, size, force)
    o.set_state(*scene.initial_state())
    return o


def errors(gpu, orc, pos0, l):
    # The oracle stores absolute positions D in fp64, so its own resolution of
    # a displacement is ~eps |D|.  The scale is floored at 1e-6 |D|max (10 nm at
    # 1 cm), where a 1e-9 criterion means ~5 ulp of D.
    scale = max(np.abs(orc.pos - pos0).max(), 1e-6 * np.abs(orc.pos).max(), 1e-9 * l)
    eD = np.linalg.norm(gpu.pos - orc.pos, axis=1).max() / scale
    Pscale = max(np.abs(orc.linmom).max(), 1e-300)
    eP = np.abs(gpu.linmom - orc.linmom).max() / Pscale
    # quaternion sign is fixed by continuity from identity
    dq = np.abs(gpu.quat - orc.quat).max()
    return dict(eD=eD, eP=eP, dq=dq)


def run_pair(scene, steps, precision, chunks=1, threads=THREADS, engine=None):
    """(gpu state, oracle state, initial positions, lattice, oracle)."""
    pos0 = scene.initial_state()[0]
    lat = from_scene(scene, precision=precision, engine=engine)
    o = oracle_for(scene, threads)
    assert abs(lat.dt - o.dt) <= 1e-15 * o.dt
    per = steps // chunks
    for c in range(chunks):
        n = per if c < chunks - 1 else steps - per * (chunks - 1)
        lat.step(n)
        o.step(n)
    return lat.read_state(), o.read_state(), pos0, lat, o
