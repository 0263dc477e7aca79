"""Batched independent scenes: K scenes packed along x with
separator planes, stepped by one launch per step, each evolving as it does
alone -- including self collision, which vx_set_batch keeps inside a scene."""
import numpy as np
import pytest

import workloads as W
from parity import assert_parity, errors, oracle_for
from paper_1212_2845_b200 import VoxError, from_scene
from paper_1212_2845_b200.batch import pack

pytestmark = pytest.mark.gpu


def _vs_oracle(b, s, sc, st, steps, prec):
    """Scene s of the batch against its own fp64 oracle run (each
    packed design is one independent physical evaluation)."""
    o = oracle_for(sc)
    o.step(steps)
    init = sc.initial_state()
    e = errors(b.state_of(s, st), o.read_state(), init[0], sc.lattice_dim, prec, init=init)
    assert_parity(e, prec, (sc.name, s))


def _cube_variants(K, n=6):
    rng = np.random.default_rng(11)
    out = []
    for s in range(K):
        sc = W.cube(contact_variant=True, n=n)
        sc.cells = rng.integers(1, 3, size=sc.cells.shape).astype(np.uint8)   # a new design
        out.append(sc)
    return out


@pytest.mark.parametrize("z_stack", [1, 2, "auto"])
@pytest.mark.parametrize("engine", ["fused", "two_pass"])
@pytest.mark.parametrize("prec", [32, 64])
def test_batch_equals_each_scene_alone(engine, prec, z_stack):
    # the cubes rest on the floor (C2c): with z stacking each scene's floor
    # lies under its own lowest layer
    scenes = _cube_variants(5)
    b = pack(scenes, precision=prec, engine=engine, z_stack=z_stack)
    kz = {1: 1, 2: 2, "auto": 5}[z_stack]
    assert b.z_stack == kz and b.lattice.num_scenes == (5 if kz != 2 else 6)
    b.lattice.step(120)
    st = b.lattice.read_state()
    for s, sc in enumerate(scenes):
        lat = from_scene(sc, precision=prec, engine=engine)
        assert lat.dt == b.lattice.dt
        lat.step(120)
        ref = lat.read_state()
        u_ref = ref.pos - sc.initial_state()[0]
        u = b.displacement_of(s, st)
        scale = np.abs(u_ref).max()
        assert np.abs(u - u_ref).max() <= (1e-12 if prec == 64 else 1e-5) * scale, s
        assert np.array_equal(st.latch[b.ext_of[s]], ref.latch)
        _vs_oracle(b, s, sc, st, 120, prec)


@pytest.mark.parametrize("z_stack", [1, "auto"])
def test_batch_self_collision_stays_inside_each_scene(z_stack):
    # two-body collisions in every scene; bodies of neighbouring scenes are one
    # plane (or layer) apart, within the horizon, but must never be paired
    scenes = [W.two_bodies(v=v) for v in (1.5, 2.0, 2.5)]
    b = pack(scenes, precision=64, z_stack=z_stack)
    if z_stack == "auto":
        assert b.z_stack == 3
    b.lattice.step(300)
    st = b.lattice.read_state()
    pairs = b.lattice.contact_pairs()
    scene_of = np.empty(sum(b.counts), int)
    for s, ids in enumerate(b.ext_of):
        scene_of[ids] = s
    assert len(pairs) and np.all(scene_of[pairs[:, 0]] == scene_of[pairs[:, 1]])
    for s, sc in enumerate(scenes):
        lat = from_scene(sc, precision=64)
        lat.step(300)
        u_ref = lat.read_state().pos - sc.initial_state()[0]
        assert np.abs(b.displacement_of(s, st) - u_ref).max() <= 1e-12 * np.abs(u_ref).max()
        _vs_oracle(b, s, sc, st, 300, 64)


def test_batch_rejects_filled_separator():
    sc = W.cube(n=4)
    lat = from_scene(sc, precision=32)
    with pytest.raises(VoxError):
        lat.set_batch(2)


def test_batch_rejects_filled_separator_layer():
    sc = W.cube(n=4)
    lat = from_scene(sc, precision=32)
    with pytest.raises(VoxError):
        lat.set_batch_z(2)
    lat.set_batch_z(0)



@pytest.mark.parametrize("prec", [32, 64])
def test_batch_y_stacked_cantilevers_equal_alone(prec):
    # 10 x 1 x 1 cantilevers (a fixed end, a tip load, ground damping) stacked
    # along y: every scene evolves as alone
    scenes = [W.cantilever(force=f) for f in (1e-3, 2e-3, 5e-4, 1.5e-3, 3e-3, 1e-4, 2.5e-3)]
    b = pack(scenes, precision=prec, engine="fused")
    assert b.y_stack == 7 and b.lattice.num_scenes == 7
    b.lattice.step(400)
    st = b.lattice.read_state()
    for s, sc in enumerate(scenes):
        lat = from_scene(sc, precision=prec, engine="fused")
        lat.step(400)
        u_ref = lat.read_state().pos - sc.initial_state()[0]
        u = b.displacement_of(s, st)
        assert np.abs(u - u_ref).max() <= (1e-12 if prec == 64 else 1e-5) * np.abs(u_ref).max(), s
        _vs_oracle(b, s, sc, st, 400, prec)


def test_batch_rejects_filled_separator_row():
    sc = W.cube(n=4)
    lat = from_scene(sc, precision=32)
    with pytest.raises(VoxError):
        lat.set_batch_y(2)
    lat.set_batch_y(0)
