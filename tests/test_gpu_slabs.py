"""x-slab decomposition on one GPU: P slabs emulated inside one
handle (ghost planes by device copies, the same slab arithmetic the NCCL
ranks run) must reproduce the single-domain run bit for bit."""
import numpy as np
import pytest

import workloads as W
from parity import assert_parity, errors, oracle_for
from paper_1212_2845_b200 import from_scene
from paper_1212_2845_b200 import slab_planes as slab

pytestmark = pytest.mark.gpu


def _oracle(sc, steps):
    o = oracle_for(sc)
    o.step(steps)
    return o.read_state()


def _vs_oracle(lat, sc, ref, prec, what):
    """A slab-split run against the fp64 oracle itself (not only against the
    single-domain GPU run)."""
    init = sc.initial_state()
    e = errors(lat.read_state(), ref, init[0], sc.lattice_dim, prec, init=init)
    assert_parity(e, prec, what)


def _flat(st):
    return np.concatenate([st.pos.ravel(), st.quat.ravel(), st.linmom.ravel(),
                           st.angmom.ravel(), st.latch.astype(float)])


def _scenes():
    b = W.block(23, 12, 10)
    b.env["zeta_ground"] = 0.0
    w = W.walker(16, 8, 8)
    w.env["T_freq"] = 1000.0
    c = W.cube(contact_variant=True, n=6)
    rng = np.random.default_rng(3)
    pos, quat, P, phi, latch = c.initial_state()
    P = P + rng.normal(size=P.shape) * 1e-10
    c.initial_state = (lambda s=(pos, quat, P, phi, latch): s)
    return {"block": b, "walker": w, "cube": c, "cantilever": W.cantilever()}


@pytest.mark.parametrize("engine", ["two_pass", "fused"])
@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("name", ["block", "walker", "cube", "cantilever"])
def test_slabs_bitwise_equal_single_domain(name, prec, engine):
    sc = _scenes()[name]
    ref = from_scene(sc, precision=prec, engine=engine)
    ref.step(150)
    r = _flat(ref.read_state())
    nx = sc.cells.shape[2]
    orc = _oracle(sc, 150)
    for P in sorted(p for p in {2, 3, 4, 5, 7, 8} if p <= nx):
        lat = from_scene(sc, precision=prec, nranks=P, engine=engine)
        if engine == "two_pass":
            assert lat.launches_per_step == 1 + 2 * P
        else:   # interior + one launch for the two boundary planes per slab
            w = [b - a for a, b in (slab(nx, P, r) for r in range(P))]
            assert lat.launches_per_step == 1 + sum(2 if x >= 3 else 1 for x in w)
        lat.step(150)
        assert np.array_equal(_flat(lat.read_state()), r), (name, prec, P)
        _vs_oracle(lat, sc, orc, prec, (name, P))
        lat.destroy()


def test_slabs_read_voxels_and_checkpoint():
    sc = W.block(23, 12, 10)
    lat = from_scene(sc, precision=32, nranks=4)
    lat.step(40)
    ids = np.array([0, 5, 600, 1500, sc.num_voxels - 1])
    v = lat.read_voxels(ids)
    full = lat.read_state()
    assert np.array_equal(v.pos, full.pos[ids]) and np.array_equal(v.quat, full.quat[ids])
    blob = lat.save_checkpoint()
    lat.step(30)
    after = _flat(lat.read_state())
    lat2 = from_scene(sc, precision=32, nranks=4)
    lat2.load_checkpoint(blob)
    lat2.step(30)
    assert np.array_equal(_flat(lat2.read_state()), after)


def test_slabs_divergence_and_rejections():
    from paper_1212_2845_b200 import DivergedError, VoxError
    sc = W.cantilever()
    lat = from_scene(sc, precision=64, nranks=3)
    pos, quat, P, phi, latch = sc.initial_state()
    P[7, 2] = np.inf
    lat.set_state(pos, quat, P, phi, latch)
    with pytest.raises(DivergedError, match="voxel 6 at step 0"):
        lat.step(3)


@pytest.mark.parametrize("engine", ["two_pass", "fused"])
@pytest.mark.parametrize("prec", [32, 64])
@pytest.mark.parametrize("name", ["two_bodies", "sphere"])
def test_slabs_self_collision_bitwise(name, prec, engine):
    """self collision across slabs.  The surface table carries
    every slab's surface voxels to every slab, the budget is global, so the
    pair lists, rebuild steps and states equal the single-domain run."""
    if name == "two_bodies":
        sc, steps = W.two_bodies(n=4, gap=2, v=2.0), 160
    else:
        sc, steps = W.hollow_sphere(n=14, r_in=4, r_out=7), 320
    ref = from_scene(sc, precision=prec, engine=engine)
    ref.step(steps)
    r = _flat(ref.read_state())
    pairs = ref.contact_pairs()
    assert ref.num_rebuilds >= 2 and len(pairs) > 0
    nx = sc.cells.shape[2]
    orc = _oracle(sc, steps)
    for P in (2, 3, 4, 5):
        if P > nx:
            continue
        lat = from_scene(sc, precision=prec, nranks=P, engine=engine)
        lat.step(steps)
        assert lat.num_rebuilds == ref.num_rebuilds, (name, P)
        assert np.array_equal(lat.contact_pairs(), pairs), (name, P)
        assert lat.num_contact_pairs == ref.num_contact_pairs
        assert np.array_equal(_flat(lat.read_state()), r), (name, prec, P)
        _vs_oracle(lat, sc, orc, prec, (name, P))
        lat.destroy()


def test_two_bodies_contact_crosses_slabs():
    """The two cubes of two_bodies sit in different slabs at P = 2 and still
    collide: momentum along x reverses and total momentum is conserved."""
    sc = W.two_bodies(n=4, gap=2, v=2.0)
    lat = from_scene(sc, precision=64, nranks=2)
    a, b = lat.owned_planes()
    assert (a, b) == (0, 10)      # emulated: the handle owns both slabs
    st0 = lat.read_state()
    lat.step(300)
    st = lat.read_state()
    i = sc.voxel_coords()[:, 0]
    left = i < 4
    assert st.linmom[left, 0].sum() < 0 < st0.linmom[left, 0].sum()
    assert abs(st.linmom[:, 0].sum()) <= 1e-12 * abs(st0.linmom[left, 0].sum())
