"""The NCCL slab path with a single rank (VX_FORCE_NCCL=1, one-rank
communicator): the ghost-plane exchange (empty), the interior / boundary-plane
launch split with the boundary planes on the comm stream, one-rank broadcasts
and reductions, NCCL calls captured in CUDA graphs -- the multi-rank code
running on one GPU.  States must equal the plain single-domain run bit for bit."""
import os

import numpy as np
import pytest

import workloads as W
from paper_1212_2845_b200 import from_scene, nccl_unique_id

pytestmark = pytest.mark.gpu


def _flat(st):
    return np.concatenate([st.pos.ravel(), st.quat.ravel(), st.linmom.ravel(),
                           st.angmom.ravel(), st.latch.astype(float)])


def _scenes():
    b = W.block(24, 16, 40)
    w = W.walker(16, 8, 40)
    w.env["T_freq"] = 1000.0
    return {"block": (b, 120), "walker": (w, 120), "C2c": (W.get("C2c"), 150),
            "two_bodies": (W.two_bodies(n=4, gap=2, v=2.0), 160),
            "sphere": (W.hollow_sphere(n=14, r_in=4, r_out=7), 320)}


@pytest.mark.parametrize("engine", ["fused", "two_pass"])
@pytest.mark.parametrize("name", ["block", "walker", "C2c", "two_bodies", "sphere"])
def test_one_rank_nccl_path_bitwise(name, engine):
    sc, steps = _scenes()[name]
    ref = from_scene(sc, precision=32, engine=engine)
    ref.step(steps)
    r = _flat(ref.read_state())
    old = os.environ.get("VX_FORCE_NCCL")
    os.environ["VX_FORCE_NCCL"] = "1"
    try:
        lat = from_scene(sc, precision=32, engine=engine, nranks=1, nccl_id=nccl_unique_id())
    finally:
        if old is None:
            os.environ.pop("VX_FORCE_NCCL", None)
        else:
            os.environ["VX_FORCE_NCCL"] = old
    if engine == "fused" and sc.cells.shape[2] >= 3:
        assert lat.launches_per_step >= 3          # clock + interior + boundary planes
    lat.step(steps // 2)
    lat.step(steps - steps // 2)
    assert np.array_equal(_flat(lat.read_state()), r), (name, engine)
    if sc.env.get("self_collision"):
        assert lat.num_contact_pairs == ref.num_contact_pairs
        assert np.array_equal(lat.contact_pairs(), ref.contact_pairs())
    lat.destroy()
