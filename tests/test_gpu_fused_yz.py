"""The fused pass for shallow lattices (nz < 64, vx_fused_yz.cuh): G rows side
by side per block, the -y record through a shared ring.  Same per-voxel
arithmetic and slot order as the one-row-at-a-time pass, so the two give the
same state bit for bit; both are checked against the oracle elsewhere
(test_gpu_fused.py, test_gpu_parity.py run the fused engine on these scenes)."""
import os

import numpy as np
import pytest

import workloads as W
from paper_1212_2845_b200 import from_scene

pytestmark = pytest.mark.gpu


def _flat(st):
    return np.concatenate([st.pos.ravel(), st.quat.ravel(), st.linmom.ravel(),
                           st.angmom.ravel(), st.latch.astype(float)])


def _run(sc, prec, yz, steps, nranks=1, **env):
    old = {k: os.environ.get(k) for k in ["VX_FUSED_YZ", *env]}
    os.environ["VX_FUSED_YZ"] = "1" if yz else "0"
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        lat = from_scene(sc, precision=prec, engine="fused", nranks=nranks)
        lat.step(steps)
        return _flat(lat.read_state())
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _scenes():
    w = W.walker(16, 8, 8)
    w.env["T_freq"] = 1000.0
    s = W.hollow_sphere(n=14, r_in=4, r_out=7)
    s.v0 = np.array([0.0, 0.0, -3.0])
    return {"C2c": W.get("C2c"), "C4": W.walker(), "walker-fast": w, "sphere-small": s,
            "two-bodies": W.two_bodies(), "block-37x9x11": W.block(37, 9, 11),
            "block-5x40x3": W.block(5, 40, 3), "C3": W.hollow_sphere()}


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("name", ["C2c", "C4", "walker-fast", "sphere-small", "two-bodies",
                                  "block-37x9x11", "block-5x40x3", "C3"])
def test_yz_pass_equals_row_pass(name, prec):
    sc = _scenes()[name]
    assert sc.cells.shape[0] < 64
    a = _run(sc, prec, True, 90)
    b = _run(sc, prec, False, 90)
    assert np.array_equal(a, b), name


@pytest.mark.parametrize("ty,sx", [(1, 1), (2, 3), (8, 32)])
def test_yz_pass_any_geometry(ty, sx):
    sc = _scenes()["block-37x9x11"]
    ref = _run(sc, 32, False, 40)
    got = _run(sc, 32, True, 40, VX_FUSED_TY=ty, VX_FUSED_SX=sx)
    assert np.array_equal(got, ref)


def test_yz_pass_emulated_slabs():
    sc = _scenes()["walker-fast"]
    ref = _run(sc, 64, False, 60)
    for P in (2, 3, 5):
        assert np.array_equal(_run(sc, 64, True, 60, nranks=P), ref), P
