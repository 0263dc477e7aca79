"""TEST INFRASTRUCTURE ONLY -- linear direct stiffness method (Table 1).

Assembles the 12-DOF beam element of Eq. 6-7 (printed for a +X
beam; the DOF vector's repeated theta_y1 at P:153 read as theta_z1, SURVEY
§8(c) #2) for every bond of a voxel lattice, rotated to the bond's lattice
axis by the cyclic permutation of reading R5, and solves K u = f with the
fixed voxels' six DOFs eliminated.  Bond constants come from Eq. 1-12 via
the oracle library (``oracle.composite`` / ``oracle.beam_constants``).

Per-node DOF order: X, Y, Z, theta_x, theta_y, theta_z.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import beam_constants, composite


def element_matrix_x(a1, a2, b1, b2, b3):
    """Eq. 7 as printed (upper triangle, symmetric completion)."""
    U = np.zeros((12, 12))
    rows = [
        # col: 1    2    3    4    5     6     7    8    9    10   11    12
        [a1, 0, 0, 0, 0, 0, -a1, 0, 0, 0, 0, 0],
        [None, b1, 0, 0, 0, b2, 0, -b1, 0, 0, 0, b2],
        [None, None, b1, 0, -b2, 0, 0, 0, -b1, 0, -b2, 0],
        [None, None, None, a2, 0, 0, 0, 0, 0, -a2, 0, 0],
        [None, None, None, None, 2 * b3, 0, 0, 0, b2, 0, b3, 0],
        [None, None, None, None, None, 2 * b3, 0, -b2, 0, 0, 0, b3],
        [None] * 6 + [a1, 0, 0, 0, 0, 0],
        [None] * 7 + [b1, 0, 0, 0, -b2],
        [None] * 8 + [b1, 0, b2, 0],
        [None] * 9 + [a2, 0, 0],
        [None] * 10 + [2 * b3, 0],
        [None] * 11 + [2 * b3],
    ]
    for i, r in enumerate(rows):
        for j, v in enumerate(r):
            if v is not None:
                U[i, j] = v
    K = np.triu(U) + np.triu(U, 1).T
    return K


def _perm_matrix(axis):
    """Pi: world -> bond frame (x-bond identity, y: (x,y,z)->(y,z,x), z: ->(z,x,y))."""
    P = np.zeros((3, 3))
    order = {0: (0, 1, 2), 1: (1, 2, 0), 2: (2, 0, 1)}[axis]
    for r, c in enumerate(order):
        P[r, c] = 1.0
    return P


def element_matrix(axis, consts):
    K = element_matrix_x(*consts)
    P = _perm_matrix(axis)
    T = np.kron(np.eye(4), P)       # local = T @ world for (u1, th1, u2, th2)
    return T.T @ K @ T


def assemble(cells, l, materials):
    """Global stiffness over filled cells (x-fastest ids); returns (K, coords)."""
    cells = np.asarray(cells)
    nz, ny, nx = cells.shape
    ids = -np.ones(cells.shape, dtype=np.int64)
    kk, jj, ii = np.nonzero(cells)
    order = np.lexsort((ii, jj, kk))   # x fastest
    kk, jj, ii = kk[order], jj[order], ii[order]
    ids[kk, jj, ii] = np.arange(len(ii))
    coords = np.stack([ii, jj, kk], 1)
    N = len(ii)
    rows, cols, vals = [], [], []
    for v in range(N):
        i, j, k = coords[v]
        for axis, (di, dj, dk) in enumerate(((1, 0, 0), (0, 1, 0), (0, 0, 1))):
            i2, j2, k2 = i + di, j + dj, k + dk
            if i2 >= nx or j2 >= ny or k2 >= nz or cells[k2, j2, i2] == 0:
                continue
            w = ids[k2, j2, i2]
            ma = materials[cells[k, j, i] - 1]
            mb = materials[cells[k2, j2, i2] - 1]
            Ec, Gc, _ = composite(ma["E"], ma["nu"], mb["E"], mb["nu"])
            Ke = element_matrix(axis, beam_constants(Ec, Gc, l))
            dofs = np.r_[6 * v:6 * v + 6, 6 * w:6 * w + 6]
            r, c = np.meshgrid(dofs, dofs, indexing="ij")
            rows.append(r.ravel()); cols.append(c.ravel()); vals.append(Ke.ravel())
    if rows:
        K = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                          shape=(6 * N, 6 * N))
    else:
        K = sp.csr_matrix((6 * N, 6 * N))
    return K, coords


def solve(cells, l, materials, fixed, forces):
    """Solve K u = f; ``fixed`` (N,) bool, ``forces`` (N,3) N.  Returns u (N,6)."""
    K, coords = assemble(cells, l, materials)
    N = len(coords)
    f = np.zeros(6 * N)
    f.reshape(N, 6)[:, :3] = forces
    free = np.ones(6 * N, bool)
    for v in np.nonzero(np.asarray(fixed))[0]:
        free[6 * v:6 * v + 6] = False
    u = np.zeros(6 * N)
    Kf = K[free][:, free].tocsc()
    u[free] = spla.spsolve(Kf, f[free])
    return u.reshape(N, 6)
