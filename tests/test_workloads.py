"""Input generators: shapes, counts and recipe invariants."""
import numpy as np
import pytest

import workloads as W


def _face_pairs(cells):
    c = cells > 0
    return (int(np.sum(c[:, :, 1:] & c[:, :, :-1])), int(np.sum(c[:, 1:, :] & c[:, :-1, :])),
            int(np.sum(c[1:, :, :] & c[:-1, :, :])))


def _surface(cells):
    c = np.pad(cells > 0, 1)
    nb = (c[1:-1, 1:-1, 2:].astype(int) + c[1:-1, 1:-1, :-2] + c[1:-1, 2:, 1:-1]
          + c[1:-1, :-2, 1:-1] + c[2:, 1:-1, 1:-1] + c[:-2, 1:-1, 1:-1])
    return int(np.sum((cells > 0) & (nb < 6)))


@pytest.mark.parametrize("name,nv,nb,ns", [
    ("C1", 10, 9, 10), ("C2", 8000, 22800, 2168), ("C3", 12880, 32112, 7184),
    ("C4", 32768, 94720, 6728)])
def test_counts(name, nv, nb, ns):
    s = W.get(name)
    assert s.num_voxels == nv
    assert sum(_face_pairs(s.cells)) == nb
    assert _surface(s.cells) == ns


def test_c5_counts_and_recipe():
    s = W.block()
    assert s.cells.shape == (256, 256, 512)
    assert s.num_voxels == 33_554_432
    assert _face_pairs(s.cells) == (33_488_896, 33_423_360, 33_423_360)
    Es = [m["E"] for m in s.materials]
    rhos = [m["rho"] for m in s.materials]
    assert all(1e5 <= E <= 1e8 for E in Es) and all(900 <= r <= 1500 for r in rhos)
    # constant material over every 8^3 cell
    c = s.cells[:8, :8, :8]
    assert np.all(c == c[0, 0, 0])
    assert set(np.unique(s.cells)) == {1, 2, 3}


def test_generators_are_deterministic():
    a, b = W.cube(), W.cube()
    assert np.array_equal(a.cells, b.cells)
    # C2 is ~50/50 two-material
    frac = np.mean(a.cells == 1)
    assert 0.45 < frac < 0.55


def test_sphere_and_walker_geometry():
    s = W.hollow_sphere()
    pos = s.initial_state()[0]
    assert pos[:, 2].min() - 0.5 * s.lattice_dim == pytest.approx(0.5 * s.lattice_dim)
    w = W.walker()
    assert np.all(w.cells[:4] == 1) and set(np.unique(w.cells[4:])) == {2, 3}


def test_clapper_recipe():
    s = W.clapper()
    assert s.cells.shape == (7, 2, 14) and s.num_voxels == 118
    assert int(s.fixed.sum()) == 14                     # the base column
    ctes = sorted(m["cte"] for m in s.materials)
    assert ctes == [-0.002, 0.0, 0.002] and s.env["self_collision"] == 1
