"""Batched independent scenes: pack K scenes of one shape into
one lattice along x with an empty separator plane after each, step them with
one launch per step, and map states back.  Marshalling only -- the packed
lattice runs the same kernels; ``vx_set_batch`` keeps self collision inside
each scene.

Every scene must share the grid shape, lattice dimension, origin and
environment (one clock and one stable time step for the batch).  Scenes sit on
a grid of x blocks (``stride`` planes) and, for shallow scenes, z blocks
(``stride_z`` layers, ``vx_set_batch_z``): the fused engine runs one thread per
z, so stacking shallow scenes (nz < 32) up to ~256 layers keeps its warps full.
The physics is invariant under the x translation; along z each scene's floor is
placed under its own lowest layer by the library, so the z translation is
invariant too.
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
    offset: float               # x offset between consecutive x blocks (m)

    rest: list = None           # per scene: packed rest sites of its voxels
    own: list = None            # per scene: its own rest sites (origin + l (ijk + 1/2))
    stride_z: int = 0           # layers per z block (nz + 1), 0: no z stacking
    z_stack: int = 1            # scenes per z column
    stride_y: int = 0           # rows per y block (ny + 1), 0: no y stacking
    y_stack: int = 1            # scenes per y row of blocks (scene s: y block
                                # (s // z_stack) % y_stack, z block s % z_stack,
                                # x block s // (y_stack z_stack))

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


def z_stack_for(K, nz, max_layers=256):
    """Scenes per z column: 1 for nz >= 32; else as many as fit ``max_layers``
    layers, balanced so the x blocks are evenly filled."""
    if nz >= 32 or K <= 1:
        return 1
    kz = max(1, min(K, max_layers // (nz + 1)))
    kx = -(-K // kz)
    return -(-K // kx)


def y_stack_for(K, ny, nz, max_rows=256):
    """Scenes per y row of blocks: for scenes whose y-z plane is under a warp
    (ny nz < 32, e.g. a 10 x 1 x 1 cantilever) as many as fit ``max_rows``
    rows, so the (y, z)-mapped fused pass gets full warps; else 1."""
    if ny * nz >= 32 or K <= 1:
        return 1
    ky = max(1, min(K, max_rows // (ny + 1)))
    kx = -(-K // ky)
    return -(-K // kx)


def pack(scenes, precision=32, engine=None, device=0, z_stack=1, y_stack="auto") -> Batch:
    """Build one lattice holding every scene (see module docstring).
    ``z_stack``: scenes per z column (1: x only, the default; "auto":
    ``z_stack_for``).  ``y_stack``: scenes per y row ("auto": ``y_stack_for``,
    which stacks only scenes whose y-z plane is under a warp).  Measured (fp32,
    one B200): z stacking helps the fused engine (32 walkers
    99 -> 78 us / step) but the two-pass engine, faster for most mid-size
    batches, gains nothing from it; y stacking gives 4096 cantilevers full warps."""
    s0 = scenes[0]
    nz, ny, nx = s0.cells.shape
    for sc in scenes:
        if sc.cells.shape != s0.cells.shape or sc.lattice_dim != s0.lattice_dim:
            raise ValueError("batched scenes must share grid shape and lattice dimension")
        if sc.env != s0.env or tuple(sc.origin) != tuple(s0.origin):
            raise ValueError("batched scenes must share environment and origin")
    stride = nx + 1
    K = len(scenes)
    kz = z_stack_for(K, nz) if z_stack == "auto" else max(1, min(int(z_stack), K))
    ky = (y_stack_for(-(-K // kz), ny, nz) if y_stack == "auto"
          else max(1, min(int(y_stack), -(-K // kz))))
    kx = -(-K // (kz * ky))
    stride_z = nz + 1 if kz > 1 else 0
    stride_y = ny + 1 if ky > 1 else 0
    # (x block, y block, z block) of scene s
    blk = [(s // (ky * kz), (s // kz) % ky, s % kz) for s in range(K)]
    # material palette: union in first-seen order
    palette, remap = [], []
    for sc in scenes:
        m = []
        for mat in sc.materials:
            if mat not in palette:
                palette.append(mat)
            m.append(palette.index(mat) + 1)
        remap.append(np.array([0] + m, np.uint8))
    cells = np.zeros((kz * (nz + 1) - 1, ky * (ny + 1) - 1, kx * stride - 1), np.uint8)
    for s, sc in enumerate(scenes):
        bx, by, bz = blk[s]
        cells[bz * (nz + 1):bz * (nz + 1) + nz, by * (ny + 1):by * (ny + 1) + ny,
              bx * stride:bx * stride + nx] = remap[s][sc.cells]
    # packed external ids (x-fastest over the packed grid) of every scene voxel
    pid = -np.ones(cells.shape, np.int64)
    filled = cells > 0
    pid[filled] = np.arange(int(filled.sum()))
    ext_of = []
    for s, sc in enumerate(scenes):
        kk, jj, ii = np.nonzero(sc.cells)
        bx, by, bz = blk[s]
        ext_of.append(pid[kk + bz * (nz + 1), jj + by * (ny + 1), ii + bx * stride])
    N = int(filled.sum())
    l = s0.lattice_dim
    lat = Lattice.create_lattice(cells, l, s0.origin, precision, device)
    lat.set_materials(palette)
    lat.set_environment(s0.env)
    if engine is not None:
        lat.set_engine(engine)
    lat.set_batch(stride)
    if stride_z:
        lat.set_batch_z(stride_z)
    if stride_y:
        lat.set_batch_y(stride_y)
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
        ijk[:, 0] += blk[s][0] * stride
        ijk[:, 1] += blk[s][1] * (ny + 1)
        ijk[:, 2] += blk[s][2] * (nz + 1)
        packed = org + l * (ijk + 0.5)                      # its rest sites in the batch
        rest.append(packed)
        owns.append(own)
        pos[ids] = packed + (p - own)
        quat[ids], lin[ids], ang[ids], latch[ids] = q, P, phi, la
    if any_bc:
        lat.set_boundary(fixed, fext)
    lat.set_state(pos, quat, lin, ang, latch)
    return Batch(lat, stride, [len(e) for e in ext_of], ext_of, stride * l, rest, owns,
                 stride_z, kz, stride_y, ky)
