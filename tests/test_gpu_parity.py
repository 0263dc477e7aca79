"""GPU (CUDA, through the C ABI) vs the fp64 oracle, element by element.

Tolerances (BASELINE.json north_star): fp64 e_D <= 1e-9 after 100 steps;
fp32 e_D <= 1e-4 after 100 steps; fp32 settled cantilever deflection within
1e-3 relative.  e_D is the max position error normalised by the largest
displacement (tests/parity.py)."""
import math

import numpy as np
import pytest

import workloads as W
from parity import assert_parity, errors, oracle_for, run_pair
from paper_1212_2845_b200 import DivergedError, from_scene

pytestmark = pytest.mark.gpu

TOL = {64: 1e-9, 32: 1e-4}


def _check(scene, steps, prec, chunks=1):
    g, o, p0, lat, orc = run_pair(scene, steps, prec, chunks)
    e = errors(g, o, p0, scene.lattice_dim, prec, init=scene.initial_state())
    assert_parity(e, prec, scene.name)
    return g, o, e


@pytest.mark.parametrize("prec", [64, 32])
def test_c1_cantilever_100_steps(prec):
    _check(W.cantilever(), 100, prec, chunks=3)


def test_c1_cantilever_settled_fp32():
    sc = W.cantilever()
    g, o, p0, lat, orc = run_pair(sc, sc.steps, 32)
    dg = p0[-1, 2] - g.pos[-1, 2]
    do = p0[-1, 2] - o.pos[-1, 2]
    assert abs(dg - do) / abs(do) <= 1e-3, (dg, do)


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("name", ["C2", "C2c"])
def test_c2_cube_100_steps(name, prec):
    g, o, e = _check(W.get(name), 100, prec)
    if name == "C2c":   # the floor contact window is inside the 100 steps
        assert np.any(g.latch)


@pytest.mark.parametrize("prec", [64, 32])
def test_c3_sphere_self_collision_100_steps(prec):
    _check(W.hollow_sphere(), 100, prec)


@pytest.mark.parametrize("prec", [64, 32])
def test_small_sphere_self_contact_long(prec):
    # a small shell driven fast into the floor: self contacts, rebuilds
    sc = W.hollow_sphere(n=14, r_in=4, r_out=7)
    sc.v0 = np.array([0.0, 0.0, -3.0])
    g, o, e = _check(sc, 600, prec, chunks=4)


@pytest.mark.parametrize("prec", [64, 32])
def test_two_bodies_collide_and_separate(prec):
    sc = W.two_bodies()
    g, o, e = _check(sc, 300, prec, chunks=6)
    # they collided (momenta reversed) and total momentum is conserved
    i = sc.voxel_coords()[:, 0]
    assert g.linmom[i < 3, 0].sum() < 0 < g.linmom[i >= 3, 0].sum()
    assert abs(g.linmom[:, 0].sum()) <= 1e-6 * np.abs(g.linmom[:, 0]).sum()


@pytest.mark.parametrize("prec", [64, 32])
def test_c4_walker_100_steps(prec):
    _check(W.walker(), 100, prec)


@pytest.mark.parametrize("prec", [64, 32])
def test_walker_fast_actuation(prec):
    # thermal actuation exercised within the window: a quarter period in 100 steps
    sc = W.walker(16, 8, 8)
    o = oracle_for(sc)
    sc.env["T_freq"] = 1.0 / (400 * o.dt)
    _check(sc, 100, prec)


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("dims", [(13, 7, 5), (37, 9, 11), (5, 40, 3)])
def test_block_ragged_multi_tile(dims, prec):
    _check(W.block(*dims, precision=prec), 100, prec)


@pytest.mark.parametrize("prec", [64, 32])
def test_app_a_regions(prec):
    """App. A as printed: 1 kN on a 5x5 mm section of a 10 MPa
    beam is far past the model's range -- both sides diverge at the same step."""
    sc = W.app_a_beam()
    n = 140 if prec == 64 else 50     # fp32 vs fp64 decorrelate on the way to blow-up
    g, o, p0, lat, orc = run_pair(sc, n, prec, chunks=2)
    e = errors(g, o, p0, sc.lattice_dim, prec, init=sc.initial_state())
    assert e["eD"] <= TOL[prec], e
    with pytest.raises(FloatingPointError) as eo:
        orc.step(400 - n)
    with pytest.raises(DivergedError) as eg:
        lat.step(400 - n)
    so, sg = str(eo.value), str(eg.value)
    assert "at step 149" in so
    if prec == 64:
        assert so.split("diverged: ")[1] == sg.split("diverged: ")[1]
    else:
        assert 140 <= int(sg.rsplit("step ", 1)[1]) <= 160


@pytest.mark.parametrize("prec", [64, 32])
def test_app_a_regions_reduced_load(prec):
    sc = W.app_a_beam()
    sc.extra["regions"][1] = ("forced", (0, 0.99, 0), (1.0, 0.01, 1.0), (0, 0, -1.0))
    _check(sc, 400, prec, chunks=2)


def test_empty_lattice_and_single_voxel():
    sc = W.cantilever()
    sc.cells = np.zeros((2, 2, 2), np.uint8)
    sc.fixed = sc.fext = None
    lat = from_scene(sc, precision=32)
    assert lat.num_voxels == 0
    lat.step(10)
    # single voxel in free fall: semi-implicit Euler closed form
    sc = W.Scene("one", np.ones((1, 1, 1), np.uint8), 1e-3, [dict(E=1e6, nu=0.35, rho=1000.0)],
                 W._env(gravity=9.81))
    lat = from_scene(sc, precision=64)
    z0 = lat.read_state().pos[0, 2]
    lat.step(1000)
    st = lat.read_state()
    n, dt = 1000, lat.dt
    assert st.pos[0, 2] == pytest.approx(z0 - 9.81 * dt * dt * n * (n + 1) / 2, rel=1e-13)


def test_all_fixed_nothing_moves():
    sc = W.cube(n=5)
    sc.fixed = np.ones(sc.num_voxels, np.uint8)
    lat = from_scene(sc, precision=32)
    p0 = lat.read_state().pos.copy()
    lat.step(50)
    assert np.array_equal(lat.read_state().pos, p0)


def test_divergence_reports_voxel_and_step():
    sc = W.cantilever()
    lat = from_scene(sc, precision=64)
    pos, quat, P, phi, latch = sc.initial_state()
    P[5, 1] = np.nan
    lat.set_state(pos, quat, P, phi, latch)
    with pytest.raises(DivergedError, match="voxel 4 at step 0"):
        lat.step(5)
