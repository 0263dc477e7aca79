"""The fused pass's launch geometry (rows per block TY, planes per segment via
the wave count, the boundary-plane launch of slabs) changes which copy of the
bond arithmetic -- a halo recomputation or a row of the sweep -- evaluates a
bond, never its result: states are bitwise identical (vx_common.cuh, explicit
rounding)."""
import os

import numpy as np
import pytest

import workloads as W
from paper_1212_2845_b200 import from_scene

pytestmark = pytest.mark.gpu


def _flat(st):
    return np.concatenate([st.pos.ravel(), st.quat.ravel(), st.linmom.ravel(),
                           st.angmom.ravel(), st.latch.astype(float)])


def _run(sc, prec, steps, ty=None, waves=None, nranks=1):
    old = {k: os.environ.get(k) for k in ("VX_FUSED_TY", "VX_FUSED_WAVES")}
    try:
        for k, v in (("VX_FUSED_TY", ty), ("VX_FUSED_WAVES", waves)):
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = str(v)
        lat = from_scene(sc, precision=prec, engine="fused", nranks=nranks)
        lat.step(steps)
        out = _flat(lat.read_state())
        lat.destroy()
        return out
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _scenes():
    b = W.block(37, 21, 40)
    b.env["zeta_ground"] = 0.0
    w = W.walker(24, 12, 40)
    w.env["T_freq"] = 1000.0
    cells = np.ones((300, 5, 6), np.uint8)          # nz > 256: two z chunks
    cells[150:] = 2
    tall = W.Scene("tall", cells, 1e-3, [dict(E=1e6, nu=0.35, rho=1000.0, mu_s=0.5, mu_d=0.5),
                                        dict(E=5e6, nu=0.35, rho=1200.0, mu_s=0.5, mu_d=0.5)],
                   W._env(gravity=9.81, floor_on=1, zeta_bond=1.0))
    return {"block": (b, 60), "walker": (w, 60), "C2c": (W.get("C2c"), 120),
            "sphere": (W.hollow_sphere(n=14, r_in=4, r_out=7), 200), "tall": (tall, 80)}


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("name", ["block", "walker", "C2c", "sphere", "tall"])
def test_geometry_bitwise(name, prec):
    sc, steps = _scenes()[name]
    ref = _run(sc, prec, steps)
    for ty, waves in ((1, 4), (3, 1), (8, 64), (2, 16)):
        assert np.array_equal(_run(sc, prec, steps, ty, waves), ref), (name, prec, ty, waves)
    assert np.array_equal(_run(sc, prec, steps, nranks=3), ref), (name, prec, "slabs")
