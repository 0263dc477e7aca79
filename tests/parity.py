"""Helpers shared by the GPU parity tests: run a scene through the CUDA path
(C ABI via the binding) and through the fp64 oracle on the same seeded input,
and measure the normalised errors of SURVEY §8(c):

    e_D = max_i |D_i^gpu - D_i^orc| / max(max_i |D_i^orc - D_i^0|, 1e-9 l)

and q, P, phi the same way (each normalised by its own largest change, see
errors()).  Floor of the position normaliser: fp64 1e-6 max|D| -- the oracle
stores absolute positions in fp64, so its own resolution of a displacement is
~eps |D| (at 10 nm of motion on a 1 cm body a 1e-9 criterion is ~5 ulp of D;
DESIGN.md §6); fp32 none beyond 1e-9 l (the GPU stores u = D - D_rest, so its
resolution scales with the displacement itself).
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


def errors(gpu, orc, pos0, l, prec=64, init=None):
    """e_D (max over voxels of the position error norm) and e_q, e_P, e_phi
    (max abs component error), each over its normaliser (module docstring).
    `init` = the initial (pos, quat, linmom, angmom, ...) the run started from
    (default: rest orientation and zero momenta).

    Normalisers: s_D = max(max|D_o - D_0|, [fp64] 1e-6 max|D|, 1e-9 l); with
    r = s_D / max|D_o - D_0| >= 1 the factor by which the position floor loosens
    e_D, the other quantities get the same floor (the oracle's absolute-position
    resolution propagates into its loads): s_P = r max|P_o - P_0|,
    s_q = max(r max|q_o - q_0|, s_D / l) (the rotation equivalent of the
    position scale), s_phi = max(r max|phi_o - phi_0|, s_P l / 2) (the angular
    momentum of s_P at the lever of half a voxel) -- so a quantity that barely
    changes (no rotation in a free fall) is measured on the motion's scale."""
    n = len(pos0)
    if init is None:
        q0 = np.zeros((n, 4)); q0[:, 0] = 1.0
        P0 = np.zeros((n, 3)); phi0 = np.zeros((n, 3))
    else:
        q0, P0, phi0 = init[1], init[2], init[3]
    floor_d = 1e-6 if prec == 64 else 0.0
    dD = np.abs(orc.pos - pos0).max(initial=0.0)
    sD = max(dD, floor_d * np.abs(orc.pos).max(initial=0.0), 1e-9 * l)
    r = sD / dD if dD > 0 else 1.0
    sP = max(r * np.abs(orc.linmom - P0).max(initial=0.0), 1e-300)
    sq = max(r * np.abs(orc.quat - q0).max(initial=0.0), sD / l)
    sphi = max(r * np.abs(orc.angmom - phi0).max(initial=0.0), sP * l / 2)
    mx = lambda a, b: float(np.abs(a - b).max(initial=0.0))   # noqa: E731
    # quaternion sign is fixed by continuity from the start on both sides
    e = dict(eD=float(np.linalg.norm(gpu.pos - orc.pos, axis=1).max(initial=0.0) / sD),
             eq=mx(gpu.quat, orc.quat) / sq, eP=mx(gpu.linmom, orc.linmom) / sP,
             ephi=mx(gpu.angmom, orc.angmom) / sphi,
             latch_flips=int(np.count_nonzero(gpu.latch != orc.latch)))
    log = os.environ.get("VX_PARITY_LOG")
    if log:
        with open(log, "a") as fh:
            fh.write(json.dumps(dict(test=os.environ.get("PYTEST_CURRENT_TEST", ""), prec=prec,
                                     **e)) + "\n")
    return e


# q, P, phi bars (north_star fixes only the position bar): fp32 the same 1e-4;
# fp64 1e-8 -- the fp64 oracle's loads inherit its absolute-position resolution
# (eps |D| k per bond), which on a block sagging by nanometres is ~2e-9 of the
# momentum change (measured maximum 2.4e-9 over the GPU suite; positions 7.8e-10)
TOL_QPPHI = {64: 1e-8, 32: 1e-4}


def assert_parity(e, prec, what="", qpphi_tol=None):
    """The bar: e_D within north_star's tolerance, q / P / phi within
    TOL_QPPHI of their own change (or `qpphi_tol`), latch flags identical."""
    tol = TOL[prec]
    t2 = qpphi_tol if qpphi_tol is not None else TOL_QPPHI[prec]
    assert e["eD"] <= tol, (what, prec, e)
    assert e["eq"] <= t2 and e["eP"] <= t2 and e["ephi"] <= t2, (what, prec, e)
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
