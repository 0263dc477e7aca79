"""The fused single-pass engine: same physics as K3 + K4 with
the bond loads kept on chip.  Checked against the oracle on the parity
scenes, against the two-pass engine, across emulated slabs, and for C5 at
full size on sampled voxels (test_gpu_c5.py runs both engines)."""
import numpy as np
import pytest

import workloads as W
from parity import assert_parity, errors, oracle_for
from paper_1212_2845_b200 import from_scene

pytestmark = pytest.mark.gpu

TOL = {64: 1e-9, 32: 1e-4}


def _flat(st):
    return np.concatenate([st.pos.ravel(), st.quat.ravel(), st.linmom.ravel(),
                           st.angmom.ravel(), st.latch.astype(float)])


def _scenes():
    w = W.walker(16, 8, 8)
    w.env["T_freq"] = 1000.0
    s = W.hollow_sphere(n=14, r_in=4, r_out=7)
    s.v0 = np.array([0.0, 0.0, -3.0])
    return {"C1": W.cantilever(), "C2c": W.get("C2c"), "C3": W.hollow_sphere(),
            "C4": W.walker(), "walker-fast": w, "sphere-small": s, "two-bodies": W.two_bodies(),
            "block-37x9x11": W.block(37, 9, 11), "block-5x40x3": W.block(5, 40, 3),
            "appA-1N": _app_a_1n()}


def _app_a_1n():
    sc = W.app_a_beam()
    sc.extra["regions"][1] = ("forced", (0, 0.99, 0), (1.0, 0.01, 1.0), (0, 0, -1.0))
    return sc


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("name", ["C1", "C2c", "C3", "C4", "walker-fast", "sphere-small",
                                  "two-bodies", "block-37x9x11", "block-5x40x3", "appA-1N"])
def test_fused_matches_oracle(name, prec):
    sc = _scenes()[name]
    steps = 300 if name in ("two-bodies", "sphere-small") else 100
    lat = from_scene(sc, precision=prec, engine="fused")
    # clock + fused pass, + broadphase / contact with self collision (the surface
    # table is written by the update itself)
    col = bool(sc.env.get("self_collision"))
    assert lat.engine == "fused" and lat.launches_per_step == (4 if col else 2)
    o = oracle_for(sc)
    lat.step(steps // 2)
    lat.step(steps - steps // 2)
    o.step(steps)
    g, r = lat.read_state(), o.read_state()
    e = errors(g, r, sc.initial_state()[0], sc.lattice_dim, prec, init=sc.initial_state())
    assert_parity(e, prec, name)


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("name", ["C1", "C2c", "C3", "walker-fast", "block-37x9x11", "two-bodies",
                                  "block-5x40x3"])
def test_fused_vs_two_pass(name, prec):
    # same bond function, same per-voxel update, same slot order, explicit
    # rounding: the engines agree bit for bit (shallow scenes run the (y, z) pass)
    sc = _scenes()[name]
    a = from_scene(sc, precision=prec, engine="two_pass")
    b = from_scene(sc, precision=prec, engine="fused")
    a.step(150)
    b.step(150)
    assert np.array_equal(_flat(a.read_state()), _flat(b.read_state())), name


@pytest.mark.parametrize("prec", [32, 64])
def test_fused_slabs_bitwise(prec):
    sc = W.block(23, 12, 10)
    ref = from_scene(sc, precision=prec, engine="fused")
    ref.step(77)
    r = _flat(ref.read_state())
    o = oracle_for(sc)
    o.step(77)
    orc = o.read_state()
    for P in (2, 3, 5, 8):
        lat = from_scene(sc, precision=prec, nranks=P, engine="fused")
        lat.step(77)
        assert np.array_equal(_flat(lat.read_state()), r), P
        init = sc.initial_state()
        assert_parity(errors(lat.read_state(), orc, init[0], sc.lattice_dim, prec, init=init),
                      prec, P)


def test_fused_engine_switch_and_checkpoint():
    sc = W.get("C2c")
    a = from_scene(sc, precision=32, engine="fused")
    a.step(33)                        # odd: the other state copy is current
    blob = a.save_checkpoint()
    a.step(40)
    ref = _flat(a.read_state())
    b = from_scene(sc, precision=32, engine="fused")
    b.load_checkpoint(blob)
    b.step(40)
    assert np.array_equal(_flat(b.read_state()), ref)
    # switching engines mid-run keeps the state
    c = from_scene(sc, precision=32, engine="fused")
    c.step(33)
    c.set_engine("two_pass")
    c.step(40)
    d = np.abs(c.read_state().pos - a.read_state().pos).max()
    assert d <= 1e-5 * np.abs(a.read_state().pos - sc.initial_state()[0]).max()


@pytest.mark.parametrize("prec", [64, 32])
def test_fused_tall_z_chunks_match_oracle(prec):
    """nz > 256: the sweep runs z chunks of 256 (each chunk's lowest lane
    recomputes its -z bond); two-material column on the floor under gravity."""
    nz = 300
    cells = np.ones((nz, 2, 3), np.uint8)
    cells[nz // 2:] = 2
    sc = W.Scene("tall", cells, 1e-3, [dict(E=1e6, nu=0.35, rho=1000.0, mu_s=0.5, mu_d=0.5),
                                      dict(E=5e6, nu=0.35, rho=1200.0, mu_s=0.5, mu_d=0.5)],
                 W._env(gravity=9.81, floor_on=1, zeta_bond=1.0))
    lat = from_scene(sc, precision=prec, engine="fused")
    assert lat.engine == "fused"
    o = oracle_for(sc)
    lat.step(100)
    o.step(100)
    g, r = lat.read_state(), o.read_state()
    e = errors(g, r, sc.initial_state()[0], sc.lattice_dim, prec, init=sc.initial_state())
    assert_parity(e, prec, "tall")
