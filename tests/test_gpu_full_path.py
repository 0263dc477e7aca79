"""The path bench.py times, against the fp64 oracle at the north_star bar.

bench.py steps C5 (512 x 256 x 256) with the fused engine: `k_step_fused`,
whose warp-uniform FULL row copy computes every row of 32 filled, free voxels
with all four x/y neighbours (the interior of a solid -- almost all of C5),
and, for nz > 256, its z-chunk form.  These tests run dense C5-recipe blocks
that take those paths (nz = 96, 256, 300 with ny, nx >= 8) from a strained
state (workloads.strained: displacements ~1e-2 l, rotations ~1e-2 rad,
velocities and spins), so every term of Eq. 13-24 and 33-35 is loaded from
the first step, for 100 steps (P:100 synchronous steps), fp64 and fp32,
against the oracle, and bit for bit against the two-pass engine.  A
64 x 256 x 256 sub-block of C5 itself (4.2M voxels, the bench's y-z plane)
runs 100 steps in both precisions against the oracle with the oracle's own
dt, which is also C5's dt."""
import numpy as np
import pytest

import workloads as W
from parity import assert_parity, errors, oracle_for, run_pair
from paper_1212_2845_b200 import from_scene

pytestmark = pytest.mark.gpu

BLOCKS = {"n96": (8, 8, 96), "n256": (9, 10, 256), "n300": (8, 8, 300)}


def _flat(st):
    return np.concatenate([st.pos.ravel(), st.quat.ravel(), st.linmom.ravel(),
                           st.angmom.ravel(), st.latch.astype(float)])


@pytest.mark.parametrize("floor_contact", [False, True])
@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("name", list(BLOCKS))
def test_fused_full_rows_strained_vs_oracle(name, prec, floor_contact):
    sc = W.block(*BLOCKS[name], precision=prec)
    st0 = W.strained(sc, seed=3, lift=not floor_contact)
    g, o, p0, lat, orc = run_pair(sc, 100, prec, chunks=2, engine="fused", state=st0)
    assert lat.engine == "fused"
    e = errors(g, o, p0, sc.lattice_dim, prec, init=st0)
    assert_parity(e, prec, (name, floor_contact))
    if floor_contact:
        assert np.any(o.latch) or np.any(np.abs(o.pos[:, 2] - 0.5e-3) < 0.5e-3)


@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("name", list(BLOCKS))
def test_fused_full_rows_bitwise_two_pass(name, prec):
    """Same bond function, same per-voxel update, same slot order, explicit
    rounding: the FULL row copy and the z chunks equal K3 + K4 bit for bit."""
    sc = W.block(*BLOCKS[name], precision=prec)
    st0 = W.strained(sc, seed=5, lift=False)
    out = []
    for engine in ("two_pass", "fused"):
        lat = from_scene(sc, precision=prec, engine=engine, init_state=False)
        lat.set_state(*st0)
        lat.step(61)
        lat.step(39)
        assert lat.engine == engine
        out.append(_flat(lat.read_state()))
    assert np.array_equal(out[0], out[1]), name


def _pairs(cells):
    """Material pairs (a, b) of face-neighbour bonds, a on the negative side."""
    c = cells.astype(np.int64)
    out = set()
    for ax in range(3):
        a = np.moveaxis(c, 2 - ax, 0)
        x, y = a[:-1].ravel(), a[1:].ravel()
        keep = (x > 0) & (y > 0)
        out |= set(zip(x[keep].tolist(), y[keep].tolist()))
    return out


def test_c5_subblock_100_steps_vs_oracle():
    """64 x 256 x 256 of the C5 recipe (4,194,304 voxels; the bench's y-z
    plane, so the same block shape and tuned launch geometry class), strained,
    floor contact on, 100 steps: GPU fp32 and fp64 against one oracle run.
    The oracle's dt is computed from this grid and equals C5's (the sub-block
    holds every material pair of the full block)."""
    sub = W.block(64, 256, 256, precision=32)
    full = W.block(precision=32)
    assert _pairs(sub.cells) == _pairs(full.cells)
    st0 = W.strained(sub, seed=7, lift=False)
    o = oracle_for(sub, state=st0)
    lat_full = from_scene(full, precision=32, init_state=False)
    assert lat_full.dt == o.dt          # C5's dt (GPU, full grid) == the oracle's own dt
    lat_full.destroy()
    gpu = {}
    for prec in (32, 64):
        lat = from_scene(sub, precision=prec, engine="fused", init_state=False)
        assert lat.dt == o.dt
        lat.set_state(*st0)
        lat.step(3)
        lat.step(97)
        gpu[prec] = lat.read_state()
        lat.destroy()
    o.step(100)
    r = o.read_state()
    for prec in (64, 32):
        e = errors(gpu[prec], r, st0[0], sub.lattice_dim, prec, init=st0)
        assert_parity(e, prec, "C5 sub-block")
    assert np.any(r.pos[:, 2] < 0.5 * sub.lattice_dim)     # floor contact in the run
