"""VX_ENGINE_AUTO (the default engine): resolved at the first step to the
faster engine for the lattice (include/voxsim.h, vx_engine).  Choosing times
both engines on the current state; that must leave no trace: the run equals,
bit for bit, a run with the chosen engine set explicitly -- including the
clock, the motion budget and the surface table of a self-colliding scene."""
import numpy as np
import pytest

import workloads as W
from paper_1212_2845_b200 import from_scene
from paper_1212_2845_b200.batch import pack

pytestmark = pytest.mark.gpu


def _flat(st):
    return np.concatenate([st.pos.ravel(), st.quat.ravel(), st.linmom.ravel(),
                           st.angmom.ravel(), st.latch.astype(float)])


def _sphere():
    s = W.hollow_sphere(n=14, r_in=4, r_out=7)
    s.v0 = np.array([0.0, 0.0, -3.0])
    return s


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("name", ["C1", "C2c", "C4", "sphere", "block-tall"])
def test_auto_equals_the_engine_it_picks(name, prec):
    sc = {"C1": W.cantilever(), "C2c": W.get("C2c"), "C4": W.walker(),
          "sphere": _sphere(), "block-tall": W.block(6, 5, 70)}[name]
    a = from_scene(sc, precision=prec)
    assert a.engine == "auto"
    a.step(37)
    chosen = a.engine
    assert chosen in ("fused", "two_pass")
    b = from_scene(sc, precision=prec, engine=chosen)
    b.step(37)
    assert np.array_equal(_flat(a.read_state()), _flat(b.read_state())), (name, chosen)
    assert a.steps_done == b.steps_done and a.num_rebuilds == b.num_rebuilds
    a.step(20)
    b.step(20)
    assert np.array_equal(_flat(a.read_state()), _flat(b.read_state()))


def test_auto_takes_fused_for_large_deep_lattices():
    lat = from_scene(W.block(64, 256, 256), precision=32)   # 2^22 cells, nz = 256
    lat.step(2)
    assert lat.engine == "fused"


def test_auto_picks_two_pass_for_packed_cantilevers():
    # 4096 packed cantilevers (nz = 1): the fused pass runs 1 of 32 lanes per
    # warp (44 us / step), the two-pass kernels full warps (9 us / step)
    bt = pack([W.cantilever()] * 4096, precision=32, z_stack=1)
    bt.lattice.step(3)
    assert bt.lattice.engine == "two_pass"


def test_auto_can_be_requested_again():
    sc = W.get("C2c")
    a = from_scene(sc, precision=32, engine="two_pass")
    a.step(5)
    a.set_engine("auto")
    assert a.engine == "auto"
    a.step(5)
    assert a.engine in ("fused", "two_pass")
    with pytest.raises(Exception):
        a.set_engine(7)


@pytest.mark.parametrize("name", ["C2c", "sphere"])
def test_prepare_steps_does_not_advance(name):
    sc = {"C2c": W.get("C2c"), "sphere": _sphere()}[name]
    a = from_scene(sc, precision=32)
    a.step(3)
    s0 = _flat(a.read_state())
    a.prepare_steps(77)                 # engine resolved, graphs built, nothing run
    assert a.engine in ("fused", "two_pass")
    assert np.array_equal(_flat(a.read_state()), s0) and a.steps_done == 3
    a.step(77)
    b = from_scene(sc, precision=32, engine=a.engine)
    b.step(80)
    assert np.array_equal(_flat(a.read_state()), _flat(b.read_state()))
