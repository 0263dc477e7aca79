"""Properties of the CUDA path that hold independently of the oracle:
determinism, bitwise resume, conservation, rigid-motion nullity, and the
collision shortlist against brute force."""
import math

import numpy as np
import pytest

import workloads as W
from paper_1212_2845_b200 import from_scene

pytestmark = pytest.mark.gpu


def _flat(st):
    return np.concatenate([st.pos.ravel(), st.quat.ravel(), st.linmom.ravel(),
                           st.angmom.ravel(), st.latch.astype(float)])


@pytest.mark.parametrize("prec", [32, 64])
def test_bitwise_determinism(prec):
    sc = W.hollow_sphere(n=14, r_in=4, r_out=7)
    sc.v0 = np.array([0.0, 0.0, -3.0])
    outs = []
    for _ in range(2):
        lat = from_scene(sc, precision=prec)
        lat.step(300)
        outs.append(_flat(lat.read_state()))
        lat.destroy()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("name", ["C2c-6", "walker-fast", "sphere-small"])
def test_resume_is_bitwise(name, prec):
    if name == "C2c-6":
        sc = W.cube(contact_variant=True, n=6)
    elif name == "walker-fast":
        sc = W.walker(16, 8, 8)
        sc.env["T_freq"] = 1000.0
    else:
        sc = W.hollow_sphere(n=14, r_in=4, r_out=7)
        sc.v0 = np.array([0.0, 0.0, -3.0])
    a = from_scene(sc, precision=prec)
    a.step(200)
    ref = _flat(a.read_state())
    b = from_scene(sc, precision=prec)
    b.step(77)
    blob = b.save_checkpoint()
    st = b.read_state()
    b.destroy()
    c = from_scene(sc, precision=prec)
    c.load_checkpoint(blob)
    assert c.steps_done == 77
    c.step(123)
    assert np.array_equal(_flat(c.read_state()), ref)
    # through absolute fp64 positions the resume is exact only to rounding
    d = from_scene(sc, precision=prec)
    d.set_state(st.pos, st.quat, st.linmom, st.angmom, st.latch)
    d.set_step(77)
    d.step(123)
    sd = d.read_state()
    disp = np.abs(a.read_state().pos - sc.initial_state()[0]).max()
    assert np.abs(sd.pos - a.read_state().pos).max() <= (1e-3 if prec == 32 else 1e-9) * disp


def test_linear_momentum_conserved_free_body_fp64():
    rng = np.random.default_rng(3)
    sc = W.cube(n=5)
    sc.env.update(gravity=0.0, floor_on=0)
    pos, quat, P, phi, latch = sc.initial_state()
    pos = pos + rng.normal(size=pos.shape) * 2e-6
    P = rng.normal(size=P.shape) * 1e-9
    lat = from_scene(sc, precision=64)
    lat.set_state(pos, quat, P, phi, latch)
    P0 = P.sum(0)
    lat.step(3000)
    st = lat.read_state()
    assert np.abs(st.linmom.sum(0) - P0).max() <= 1e-12 * np.abs(st.linmom).sum()


def test_rigid_motion_nullity_fp64():
    rng = np.random.default_rng(1)
    sc = W.cube(n=4)
    sc.env.update(gravity=0.0, floor_on=0)
    pos, quat, P, phi, latch = sc.initial_state()
    ax = rng.normal(size=3); ax /= np.linalg.norm(ax)
    a = 1.1
    q = np.r_[math.cos(a / 2), math.sin(a / 2) * ax]
    w, x, y, z = q
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    c = pos.mean(0)
    pos2 = (pos - c) @ R.T + c + 0.003
    omega = np.array([20.0, -5.0, 40.0])
    m = np.where(sc.cells.ravel()[sc.cells.ravel() > 0] == 1, 1000.0, 1200.0) * 1e-9
    P2 = m[:, None] * (np.cross(omega, pos2 - c) + np.array([0.2, 0.0, -0.1]))
    phi2 = (m * 1e-6 / 6)[:, None] * omega
    lat = from_scene(sc, precision=64)
    lat.set_state(pos2, np.tile(q, (len(pos), 1)), P2, phi2, latch)
    lat.step(1)
    st = lat.read_state()
    fscale = 1e8 * 1e-3 * 1e-2 * lat.dt     # a stiff bond at 1% strain, one step
    assert np.abs(st.linmom - P2).max() <= 1e-11 * fscale
    assert np.abs(st.angmom - phi2).max() <= 1e-11 * fscale * 1e-3


def _surface_and_coords(sc):
    c = np.pad(sc.cells > 0, 1)
    nb = (c[1:-1, 1:-1, 2:].astype(int) + c[1:-1, 1:-1, :-2] + c[1:-1, 2:, 1:-1]
          + c[1:-1, :-2, 1:-1] + c[2:, 1:-1, 1:-1] + c[:-2, 1:-1, 1:-1])
    surf_cell = ((sc.cells > 0) & (nb < 6)).ravel()
    filled = sc.cells.ravel() > 0
    surf = np.nonzero(surf_cell[filled])[0]
    return surf, sc.voxel_coords()


def _brute_pairs(pos, surf, ijk, cutoff):
    out = []
    for x in range(len(surf)):
        a = surf[x]
        d = np.linalg.norm(pos[surf[x + 1:]] - pos[a], axis=1)
        man = np.abs(ijk[surf[x + 1:]] - ijk[a]).sum(1)
        for b in surf[x + 1:][(d < cutoff) & (man > 3)]:
            out.append((a, b))
    return sorted(out)


def test_shortlist_equals_brute_force_at_rebuild():
    rng = np.random.default_rng(5)
    cells = (rng.random((6, 7, 9)) < 0.55).astype(np.uint8)
    sc = W.Scene("rnd", cells, 1e-3, [dict(E=1e6, nu=0.35, rho=1000.0)],
                 W._env(self_collision=1, horizon_voxels=2.0, zeta_col=0.5))
    pos, quat, P, phi, latch = sc.initial_state()
    pos = pos + rng.normal(size=pos.shape) * 0.35e-3
    lat = from_scene(sc, precision=64)
    lat.set_state(pos, quat, P, phi, latch)
    lat.step(1)                      # rebuild from S_0 at the start of step 0
    surf, ijk = _surface_and_coords(sc)
    cutoff = 2 * 0.5e-3 + 2.0 * 1e-3
    expect = _brute_pairs(pos, surf, ijk, cutoff)
    got = [tuple(p) for p in lat.contact_pairs()]
    assert got == expect and len(expect) > 10
    assert lat.num_contact_pairs == len(expect)


@pytest.mark.parametrize("prec", [32, 64])
def test_shortlist_covers_every_overlap_each_step(prec):
    sc = W.two_bodies()
    lat = from_scene(sc, precision=prec)
    surf, ijk = _surface_and_coords(sc)
    seen_overlap = 0
    for _ in range(260):
        st = lat.read_state()        # S_n; step n uses the list as of its start
        lat.step(1)
        short = set(tuple(p) for p in lat.contact_pairs())
        over = _brute_pairs(st.pos, surf, ijk, 1e-3)       # r_a + r_b = l (alpha = 0)
        seen_overlap += len(over)
        missing = [p for p in over if p not in short]
        assert not missing, missing[:5]
    assert lat.num_rebuilds >= 2
    assert seen_overlap > 0


@pytest.mark.parametrize("engine", ["fused", "two_pass"])
@pytest.mark.parametrize("prec", [32, 64])
def test_quaternion_sign_invariance(prec, engine):
    """q and -q are one orientation (R7): negating every voxel's quaternion of a
    strained block leaves positions and momenta bit for bit unchanged over 60
    steps (the bond's w >= 0 fold, R(q) = R(-q)); the quaternions stay negated."""
    sc = W.block(10, 9, 70, precision=prec)
    pos, quat, P, phi, latch = W.strained(sc, seed=9, lift=False)
    out = []
    for sgn in (1.0, -1.0):
        lat = from_scene(sc, precision=prec, engine=engine, init_state=False)
        lat.set_state(pos, sgn * quat, P, phi, latch)
        lat.step(60)
        out.append(lat.read_state())
    a, b = out
    assert np.array_equal(a.pos, b.pos) and np.array_equal(a.linmom, b.linmom)
    assert np.array_equal(a.angmom, b.angmom) and np.array_equal(a.latch, b.latch)
    assert np.array_equal(a.quat, -b.quat)
