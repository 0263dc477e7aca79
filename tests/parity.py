"""Helpers shared by the GPU parity tests: run a scene through the CUDA path
(C ABI via the binding) and through the fp64 oracle on the same seeded input,
and measure the normalised errors of SURVEY §8(c):

    e_D = max_i |D_i^gpu - D_i^orc| / max(max_i |D_i^orc - D_i^0|, 1e-9 l)

and q, P, phi the same way (each normalised by its own largest change).
Floors of the normalisers (the resolution of the stored values over the bar):
  * fp64 positions: 1e-6 max|D| -- the oracle stores absolute positions in
    fp64, so its own resolution of a displacement is ~eps |D| (at 10 nm of
    motion on a 1 cm body a 1e-9 criterion is ~5 ulp of D);
  * fp32 positions: none beyond 1e-9 l (the GPU stores u = D - D_rest, so its
    resolution scales with the displacement itself);
  * q, P, phi: 1e-6 (fp64) / 1e-3 (fp32) of the quantity's magnitude, i.e. an
    error at the storage resolution (~1e-16 / ~1e-7 relative) never fails.
"""
import json
import os

import numpy as np

from oracle import OracleSim
from paper_1212_2845_b200 import from_scene

THREADS = os.cpu_count() or 1
TOL = {64: 1e-9, 32: 1e-4}


def oracle_for(scene, threads=THREADS, state=None):
    o = OracleSim(scene.cells, scene.lattice_dim, scene.materials, scene.env, scene.origin)
    o.set_threads(threads)
    if scene.fixed is not None or scene.fext is not None:
        o.set_boundary(scene.fixed, scene.fext)
    for kind, org, size, force in scene.extra.get("regions", []):
        o.add_region(kind, org, size, force)
    o.set_state(*(state if state is not None else scene.initial_state()))
    return o


def _rel(g, o, x0, floor):
    scale = max(np.abs(o - x0).max(initial=0.0), floor * np.abs(o).max(initial=0.0), 1e-300)
    return float(np.abs(g - o).max(initial=0.0) / scale)


def errors(gpu, orc, pos0, l, prec=64, init=None):
    """e_D (max over voxels of the position error norm) and e_q, e_P, e_phi
    (max abs component error), each over its normaliser (module docstring).
    `init` = the initial (pos, quat, linmom, angmom, ...) the run started from
    (default: rest orientation and zero momenta)."""
    floor_d = 1e-6 if prec == 64 else 0.0
    scale = max(np.abs(orc.pos - pos0).max(), floor_d * np.abs(orc.pos).max(), 1e-9 * l)
    eD = float(np.linalg.norm(gpu.pos - orc.pos, axis=1).max() / scale)
    n = len(pos0)
    if init is None:
        q0 = np.zeros((n, 4)); q0[:, 0] = 1.0
        P0 = np.zeros((n, 3)); phi0 = np.zeros((n, 3))
    else:
        q0, P0, phi0 = init[1], init[2], init[3]
    f = 1e-6 if prec == 64 else 1e-3
    # quaternion sign is fixed by continuity from the start on both sides
    e = dict(eD=eD, eq=_rel(gpu.quat, orc.quat, q0, f), eP=_rel(gpu.linmom, orc.linmom, P0, f),
             ephi=_rel(gpu.angmom, orc.angmom, phi0, f),
             latch_flips=int(np.count_nonzero(gpu.latch != orc.latch)))
    log = os.environ.get("VX_PARITY_LOG")
    if log:
        with open(log, "a") as fh:
            fh.write(json.dumps(dict(test=os.environ.get("PYTEST_CURRENT_TEST", ""), prec=prec,
                                     **e)) + "\n")
    return e


def assert_parity(e, prec, what=""):
    """The bar: e_D within north_star's tolerance, q / P / phi within the same
    relative tolerance of their own change, latch flags identical."""
    tol = TOL[prec]
    assert e["eD"] <= tol, (what, prec, e)
    assert e["eq"] <= tol and e["eP"] <= tol and e["ephi"] <= tol, (what, prec, e)
    assert e["latch_flips"] == 0, (what, prec, e)


def run_pair(scene, steps, precision, chunks=1, threads=THREADS, engine=None, state=None):
    """(gpu state, oracle state, initial positions, lattice, oracle)."""
    st0 = state if state is not None else scene.initial_state()
    lat = from_scene(scene, precision=precision, engine=engine, init_state=state is None)
    if state is not None:
        lat.set_state(*st0)
    o = oracle_for(scene, threads, state=st0)
    assert abs(lat.dt - o.dt) <= 1e-15 * o.dt
    per = steps // chunks
    for c in range(chunks):
        n = per if c < chunks - 1 else steps - per * (chunks - 1)
        lat.step(n)
        o.step(n)
    return lat.read_state(), o.read_state(), st0[0], lat, o
