"""Degenerate cases of the method on the CUDA path, against the oracle where
the oracle defines the result.

* coincident centres of a contact pair (reading R16): the normal falls
  back to +z for the voxel with the lower external id, -z for the other --
  chosen here so that the lattice's internal (x-slowest) order disagrees with
  the external (x-fastest) one;
* a non-positive thermal rest length (Eq. 40) is a fault
  reported as DIVERGED naming the first step where it occurs, the same step
  the oracle stops at;
* a contact pair list over its capacity returns VX_ERR_STATE without a CUDA
  fault (the library stays usable)."""
import math

import numpy as np
import pytest

import workloads as W
from parity import assert_parity, errors, oracle_for, run_pair
from paper_1212_2845_b200 import DivergedError, VoxError, from_scene
from paper_1212_2845_b200 import _native as N

pytestmark = pytest.mark.gpu
L = 1e-3


def _coincident_scene():
    # A = (0, 1, 0), B = (5, 0, 0): external ids 6 and 5 (B lower), internal
    # box ids 1 and 10 (A lower); lattice Manhattan distance 6 > 3
    cells = np.zeros((1, 2, 6), np.uint8)
    cells[0, 1, 0] = 1
    cells[0, 0, 5] = 2
    mats = [dict(E=1e6, nu=0.35, rho=1000.0), dict(E=3e6, nu=0.35, rho=1500.0)]
    sc = W.Scene("coincident", cells, L, mats, W._env(self_collision=1, zeta_col=0.3))
    pos, quat, P, phi, latch = sc.initial_state()
    ijk = sc.voxel_coords()
    a = int(np.nonzero((ijk[:, 0] == 0))[0][0])
    b = 1 - a
    pos[b] = pos[a]
    state = (pos, quat, P, phi, latch)
    return sc, state, a, b


@pytest.mark.parametrize("prec", [64, 32])
def test_coincident_centres_fall_back_to_z(prec):
    sc, st0, a, b = _coincident_scene()
    assert b < a                                     # B has the lower external id
    g, o, p0, lat, orc = run_pair(sc, 1, prec, state=st0)
    assert g.linmom[b, 2] > 0 > g.linmom[a, 2]       # +z on the lower external id
    assert np.abs(g.linmom[:, :2]).max() == 0.0
    assert g.linmom[b, 2] == pytest.approx(o.linmom[b, 2], rel={64: 1e-12, 32: 1e-6}[prec])
    assert g.linmom[a, 2] == pytest.approx(o.linmom[a, 2], rel={64: 1e-12, 32: 1e-6}[prec])
    lat.step(40)                                     # they separate along z
    orc.step(40)
    e = errors(lat.read_state(), orc.read_state(), p0, L, prec, init=st0)
    assert_parity(e, prec, "coincident")


def _thermal_fault_scene(cross=37.5):
    """alpha = -0.02, dT = 60 sin(2 pi f t): the rest length l (1 - 1.2 sin)
    reaches 0 at sin = 1/1.2, placed `cross` steps in (mid-step: no tie)."""
    cells = np.ones((1, 1, 3), np.uint8)
    mats = [dict(E=1e6, nu=0.35, rho=1000.0, cte=-0.02)]
    sc = W.Scene("thermal-fault", cells, L, mats, W._env(T_amp=60.0, zeta_bond=1.0))
    dt = 1 / (2 * math.pi * math.sqrt(1e6 * L / 1e-6))       # Eq. 31-32, one material
    sc.env["T_freq"] = math.asin(1 / 1.2) / (2 * math.pi * cross * dt)
    return sc


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("engine", ["fused", "two_pass"])
def test_nonpositive_rest_length_is_diverged_at_the_oracle_step(prec, engine):
    sc = _thermal_fault_scene()
    o = oracle_for(sc)
    with pytest.raises(FloatingPointError) as eo:
        o.step(100)
    step_o = int(str(eo.value).rsplit("step ", 1)[1])
    assert step_o == 38
    lat = from_scene(sc, precision=prec, engine=engine)
    assert lat.dt == o.dt
    lat.step(step_o)                                 # steps 0 .. 37 are fine
    with pytest.raises(DivergedError, match=f"non-positive thermal rest length at step {step_o} "):
        lat.step(5)


def test_pair_list_overflow_is_state_error_not_a_fault():
    """512 isolated surface voxels (no bonds: lattice spacing 4, Manhattan
    distance > 3 between any two) all placed within one voxel of each other:
    512 x 511 partner entries exceed the list capacity (max(2^16, 128 per
    surface row) = 65,536).  vx_step must return VX_ERR_STATE and leave the
    CUDA context usable."""
    cells = np.zeros((32, 32, 32), np.uint8)
    cells[::4, ::4, ::4] = 1
    sc = W.Scene("crowd", cells, L, [dict(E=1e6, nu=0.35, rho=1000.0)],
                 W._env(self_collision=1, zeta_col=0.5))
    assert sc.num_voxels == 512
    pos, quat, P, phi, latch = sc.initial_state()
    rng = np.random.default_rng(2)
    pos = pos[0] + rng.normal(size=pos.shape) * 0.1 * L          # all within one voxel
    lat = from_scene(sc, precision=32, init_state=False)
    assert lat.num_bonds == 0 and lat.num_surface == 512
    lat.set_state(pos, quat, P, phi, latch)
    with pytest.raises(VoxError) as ei:
        lat.step(3)
    assert ei.value.status == N.VX_ERR_STATE and "capacity" in str(ei.value)
    st = lat.read_state()                            # the context is alive
    assert np.all(np.isfinite(st.pos))
    lat.destroy()
    ok = from_scene(W.cantilever(), precision=32)
    ok.step(10)
    assert np.all(np.isfinite(ok.read_state().pos))
