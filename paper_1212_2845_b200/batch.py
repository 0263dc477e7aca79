"""Batched independent scenes: pack K scenes of one shape into
one lattice along x with an empty separator plane after each, step them with
one launch per step, and map states back.  Marshalling only -- the packed
lattice runs the same kernels; ``vx_set_batch`` keeps self collision inside
each scene.

Every scene must share the grid shape, lattice dimension, origin and
environment (one clock and one stable time step for the batch).  Scene s sits
at x offset s * stride * l; the physics is invariant under that translation.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .lattice import Lattice, State


@dataclass
class Batch:
    lattice: Lattice
    stride: int                 # planes per scene (nx + 1)
    counts: list                # voxels per scene
    ext_of: list                # per scene: packed external ids of its voxels (scene order)
    offset: float               # x offset between consecutive scenes (m)

    rest: list = None           # per scene: packed rest sites of its voxels
    own: list = None            # per scene: its own rest sites (origin + l (ijk + 1/2))

    def state_of(self, s, st: State | None = None) -> State:
        """Scene s's state; positions as displacements from its packed rest sites
        added to its own rest sites (origin + l (ijk + 1/2))."""
        st = st or self.lattice.read_state()
        ids = self.ext_of[s]
        pos = self.own[s] + (st.pos[ids] - self.rest[s])
        return State(pos, st.quat[ids].copy(), st.linmom[ids].copy(), st.angmom[ids].copy(),
                     st.latch[ids].copy())

    def displacement_of(self, s, st: State | None = None):
        """u = D - D_rest of scene s's voxels (exact in the lattice's frame)."""
        st = st or self.lattice.read_state()
        return st.pos[self.ext_of[s]] - self.rest[s]


def pack(scenes, precision=32, engine=None, device=0) -> Batch:
    """Build one lattice holding every scene (see module docstring)."""
    s0 = scenes[0]
    nz, ny, nx = s0.cells.shape
    for sc in scenes:
        if sc.cells.shape != s0.cells.shape or sc.lattice_dim != s0.lattice_dim:
            raise ValueError("batched scenes must share grid shape and lattice dimension")
        if sc.env != s0.env or tuple(sc.origin) != tuple(s0.origin):
            raise ValueError("batched scenes must share environment and origin")
    stride = nx + 1
    K = len(scenes)
    # material palette: union in first-seen order
    palette, remap = [], []
    for sc in scenes:
        m = []
        for mat in sc.materials:
            if mat not in palette:
                palette.append(mat)
            m.append(palette.index(mat) + 1)
        remap.append(np.array([0] + m, np.uint8))
    cells = np.zeros((nz, ny, K * stride - 1), np.uint8)
    for s, sc in enumerate(scenes):
        cells[:, :, s * stride:s * stride + nx] = remap[s][sc.cells]
    # packed external ids (x-fastest over the packed grid) of every scene voxel
    pid = -np.ones(cells.shape, np.int64)
    filled = cells > 0
    pid[filled] = np.arange(int(filled.sum()))
    ext_of = []
    for s, sc in enumerate(scenes):
        kk, jj, ii = np.nonzero(sc.cells)
        ext_of.append(pid[kk, jj, ii + s * stride])
    N = int(filled.sum())
    l = s0.lattice_dim
    lat = Lattice.create_lattice(cells, l, s0.origin, precision, device)
    lat.set_materials(palette)
    lat.set_environment(s0.env)
    if engine is not None:
        lat.set_engine(engine)
    lat.set_batch(stride)
    fixed = np.zeros(N, np.uint8)
    fext = np.zeros((N, 3))
    pos = np.zeros((N, 3)); quat = np.zeros((N, 4)); lin = np.zeros((N, 3))
    ang = np.zeros((N, 3)); latch = np.zeros(N, np.uint8)
    any_bc = False
    org = np.asarray(s0.origin, np.float64)[None, :]
    rest, owns = [], []
    for s, sc in enumerate(scenes):
        ids = ext_of[s]
        if sc.fixed is not None:
            fixed[ids] = sc.fixed
            any_bc = True
        if sc.fext is not None:
            fext[ids] = sc.fext
            any_bc = True
        p, q, P, phi, la = sc.initial_state()
        ijk = sc.voxel_coords().astype(np.float64)
        own = org + l * (ijk + 0.5)                         # the scene's own rest sites
        ijk[:, 0] += s * stride
        packed = org + l * (ijk + 0.5)                      # its rest sites in the batch
        rest.append(packed)
        owns.append(own)
        pos[ids] = packed + (p - own)
        quat[ids], lin[ids], ang[ids], latch[ids] = q, P, phi, la
    if any_bc:
        lat.set_boundary(fixed, fext)
    lat.set_state(pos, quat, lin, ang, latch)
    return Batch(lat, stride, [len(e) for e in ext_of], ext_of, stride * l, rest, owns)
