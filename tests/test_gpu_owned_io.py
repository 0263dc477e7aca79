"""Owned-voxel state I/O (vx_num_owned / vx_owned_ids / vx_set_state_owned /
vx_read_state_owned): with one rank (or emulated slabs in one process) the
owned voxels are all N, in external order, and the calls equal the full-state
ones bit for bit."""
import numpy as np
import pytest

import workloads as W
from paper_1212_2845_b200 import from_scene

pytestmark = pytest.mark.gpu


def _flat(st):
    return np.concatenate([st.pos.ravel(), st.quat.ravel(), st.linmom.ravel(),
                           st.angmom.ravel(), st.latch.astype(float)])


@pytest.mark.parametrize("nranks", [1, 3])
@pytest.mark.parametrize("prec", [32, 64])
def test_owned_io_equals_full_state(prec, nranks):
    sc = W.block(12, 6, 70, precision=prec)
    st0 = W.strained(sc, seed=2, lift=False)
    a = from_scene(sc, precision=prec, nranks=nranks, init_state=False)
    ids = a.owned_ids()
    assert np.array_equal(ids, np.arange(sc.num_voxels))
    a.set_state_owned(*[x[ids] for x in st0])
    b = from_scene(sc, precision=prec, nranks=nranks, init_state=False)
    b.set_state(*st0)
    assert np.array_equal(_flat(a.read_state_owned()), _flat(b.read_state()))
    a.step(40)
    b.step(40)
    assert np.array_equal(_flat(a.read_state_owned()), _flat(b.read_state()))
    with pytest.raises(ValueError):
        a.set_state_owned(st0[0][:-1])
