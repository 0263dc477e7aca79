"""Seeded synthetic workloads C1-C5 (BASELINE.json configs[0..4]).

Shared by the oracle side and the CUDA side of every test and of bench.py.
This module holds only the input recipes of SURVEY.md §8(d) -- grids,
palettes, environment constants and initial conditions; none of the
method's arithmetic.  All generators use numpy PCG64(12122845), a fresh
generator per config.

Grid convention: ``cells`` has shape (nz, ny, nx), so its flat C order is
x-fastest; 0 = empty, k>=1 selects ``materials[k-1]``.  Voxel ids are
the filled cells in that flat order.  Voxel (i,j,k) sits at
origin + l*(i+1/2, j+1/2, k+1/2).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED = 12122845
L = 1e-3           # lattice dimension, m (all configs)
NU = 0.35


def _rng():
    return np.random.Generator(np.random.PCG64(SEED))


def _mat(E, rho, nu=NU, cte=0.0, mu=0.0):
    return dict(E=float(E), nu=float(nu), rho=float(rho), cte=float(cte), mu_s=float(mu),
                mu_d=float(mu))


def _env(**kw):
    env = dict(gravity=0.0, floor_on=0, floor_z=0.0, T_ref=0.0, T_amp=0.0, T_freq=0.0,
               T_phase=0.0, zeta_bond=1.0, zeta_ground=0.0, zeta_col=0.0,
               horizon_voxels=2.0, dt_safety=1.0, self_collision=0)
    env.update(kw)
    return env


@dataclass
class Scene:
    name: str
    cells: np.ndarray                 # (nz, ny, nx) uint8
    lattice_dim: float
    materials: list
    env: dict
    origin: tuple = (0.0, 0.0, 0.0)
    fixed: np.ndarray | None = None   # (N,) uint8 in voxel-id order
    fext: np.ndarray | None = None    # (N,3) N
    v0: np.ndarray | None = None      # (3,) or (N,3) initial velocities, m/s
    steps: int = 100                  # the config's step count
    precision: int = 64
    notes: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def shape_xyz(self):
        nz, ny, nx = self.cells.shape
        return nx, ny, nz

    @property
    def num_voxels(self):
        return int(np.count_nonzero(self.cells))

    def voxel_coords(self):
        """(N,3) integer (i,j,k) of the filled cells in voxel-id order."""
        kk, jj, ii = np.nonzero(self.cells)   # C order of (k,j,i) == x-fastest ids
        return np.stack([ii, jj, kk], 1)

    def initial_state(self):
        """Rest lattice sites, identity orientation, P = rho l^3 v0, phi = 0."""
        ijk = self.voxel_coords().astype(np.float64)
        l = self.lattice_dim
        pos = np.asarray(self.origin, np.float64)[None, :] + l * (ijk + 0.5)
        n = len(ijk)
        quat = np.zeros((n, 4)); quat[:, 0] = 1.0
        linmom = np.zeros((n, 3))
        if self.v0 is not None:
            mats = self.cells.ravel()[np.flatnonzero(self.cells.ravel())]
            rho = np.array([m["rho"] for m in self.materials])[mats - 1]
            v0 = np.asarray(self.v0, np.float64)
            linmom = (rho * l ** 3)[:, None] * (v0[None, :] if v0.ndim == 1 else v0)
        angmom = np.zeros((n, 3))
        latch = np.zeros(n, np.uint8)
        return pos, quat, linmom, angmom, latch


def cantilever(n=10, force=1e-3, zeta_ground=0.013, E=1e6):
    """C1: n x 1 x 1, voxel (0,0,0) fixed, tip force (0,0,-force) on (n-1,0,0)."""
    cells = np.ones((1, 1, n), np.uint8)
    fixed = np.zeros(n, np.uint8); fixed[0] = 1
    fext = np.zeros((n, 3)); fext[n - 1, 2] = -force
    return Scene("C1-cantilever", cells, L, [_mat(E, 1000.0)],
                 _env(zeta_bond=1.0, zeta_ground=zeta_ground), fixed=fixed, fext=fext,
                 steps=20000, notes="g=0, floor off; zeta_g=0.013 (SURVEY 8c #13)")


def cube(contact_variant=False, n=20):
    """C2 (and C2c): n^3 two-material cube dropped on the floor."""
    rng = _rng()
    ids = rng.integers(1, 3, size=n ** 3).astype(np.uint8)
    cells = ids.reshape(n, n, n)
    mats = [_mat(1e6, 1000.0, mu=0.5), _mat(1e8, 1200.0, mu=0.5)]
    env = _env(gravity=9.81, floor_on=1, zeta_bond=1.0, zeta_col=0.5)
    if contact_variant:
        return Scene("C2c-cube-contact", cells, L, mats, env, origin=(0.0, 0.0, 1e-5),
                     v0=np.array([0.0, 0.0, -0.1981]), steps=5000,
                     notes="bottom face 10 um above floor, v0 = 2 mm drop impact speed")
    return Scene("C2-cube", cells, L, mats, env, origin=(0.0, 0.0, 2e-3), steps=5000,
                 notes="bottom face 2 mm above floor")


def hollow_sphere(n=40, r_in=17, r_out=20):
    """C3: n^3 box, filled iff r_in*l <= |c| < r_out*l (c from the box centre)."""
    idx = np.arange(n) + 0.5 - n / 2.0
    z, y, x = np.meshgrid(idx, idx, idx, indexing="ij")
    r = np.sqrt(x * x + y * y + z * z)
    cells = ((r >= r_in) & (r < r_out)).astype(np.uint8)
    kmin = int(np.nonzero(cells.any(axis=(1, 2)))[0].min())
    # lowest voxel's bottom face 0.5 l above the floor
    oz = 0.5 * L - kmin * L
    env = _env(gravity=9.81, floor_on=1, zeta_bond=1.0, zeta_col=0.5, self_collision=1,
               horizon_voxels=2.0)
    return Scene("C3-hollow-sphere", cells, L, [_mat(5e5, 1000.0, mu=0.5)], env,
                 origin=(0.0, 0.0, oz), v0=np.array([0.0, 0.0, -1.0]), steps=10000)


def walker(nx=64, ny=32, nz=16):
    """C4: passive base (k<4, E=1e7) under 4^3 checker blocks of +-CTE actuators."""
    k = np.arange(nz)[:, None, None]
    j = np.arange(ny)[None, :, None]
    i = np.arange(nx)[None, None, :]
    parity = (i // 4 + j // 4 + k // 4) % 2
    cells = np.where(k < 4, 1, np.where(parity == 0, 2, 3)).astype(np.uint8)
    cells = np.broadcast_to(cells, (nz, ny, nx)).copy()
    mats = [_mat(1e7, 1000.0, mu=0.8), _mat(1e6, 1000.0, cte=0.01, mu=0.8),
            _mat(1e6, 1000.0, cte=-0.01, mu=0.8)]
    env = _env(gravity=9.81, floor_on=1, zeta_bond=1.0, T_amp=10.0, T_freq=5.0)
    return Scene("C4-walker", cells, L, mats, env, steps=20000,
                 notes="resting on the floor; T = 10 sin(2 pi 5 t) K")


def block(nx=512, ny=256, nz=256, precision=32):
    """C5 recipe on an nx x ny x nz box (default = the scaling block)."""
    rng = _rng()
    uE = rng.random(3)
    uR = rng.random(3)
    cx, cy, cz = 64, 32, 32                      # cell draw is always the full 8^3 grid
    cell = rng.integers(1, 4, size=cx * cy * cz).astype(np.uint8).reshape(cz, cy, cx)
    E = 10.0 ** (5 + 3 * uE)
    rho = 900.0 + 600.0 * uR
    mats = [_mat(E[q], rho[q], mu=0.5) for q in range(3)]
    ci = np.arange(nx) // 8
    cj = np.arange(ny) // 8
    ck = np.arange(nz) // 8
    cells = cell[ck[:, None, None] % cz, cj[None, :, None] % cy, ci[None, None, :] % cx]
    # zeta_b = 0.9, not 1: with the literal dt (R9) and m_min damping (R10), zeta_b = 1 is
    # marginally unstable for this recipe -- a mode around voxel (67, 209, 160) grows ~5 % per
    # step and the run diverges near step 740 (GPU fp32), 840 (GPU fp64) and 914 (the fp64
    # oracle, independent code); zeta_b <= 0.95 runs 5000 steps flat (R20,
    # tools/stab_sub.py).  BASELINE.json gives C5 no damping value.
    env = _env(gravity=9.81, floor_on=1, zeta_bond=0.9)
    name = "C5-block" if (nx, ny, nz) == (512, 256, 256) else f"C5-block-{nx}x{ny}x{nz}"
    return Scene(name, np.ascontiguousarray(cells), L, mats, env, steps=1000,
                 precision=precision, notes="resting on the floor")


def two_bodies(n=3, gap=2, v=2.0, E=1e6):
    """Two n^3 cubes, `gap` empty planes apart along x, approaching at +-v:
    surface-voxel self collision between separate bodies."""
    nx = 2 * n + gap
    cells = np.zeros((n, n, nx), np.uint8)
    cells[:, :, :n] = 1
    cells[:, :, n + gap:] = 1
    s = Scene("two-bodies", cells, L, [_mat(E, 1000.0)],
              _env(zeta_bond=1.0, zeta_col=0.2, self_collision=1, horizon_voxels=2.0),
              steps=300)
    i = s.voxel_coords()[:, 0]
    s.v0 = np.zeros((len(i), 3))
    s.v0[i < n, 0] = v
    s.v0[i >= n, 0] = -v
    return s


def clapper(n=13, gap=3, cte=0.002, dT=10.0):
    """A clapper-like +-CTE scene: two bimorph strips of
    n x 2 x 2 voxels, `gap` voxels apart in z, held by a fixed base column at
    x = 0.  Strip A (bottom) is +CTE under -CTE and curls up, strip B (top)
    the mirror image; a constant temperature rise dT (T = T_amp sin(pi/2))
    closes them onto each other: surface self contact between the two arms."""
    nz = 4 + gap
    cells = np.zeros((nz, 2, n + 1), np.uint8)
    cells[:, :, 0] = 1                                # base column (passive, fixed)
    cells[0, :, 1:] = 2                               # strip A: +CTE below ...
    cells[1, :, 1:] = 3                               # ... -CTE above -> curls toward B
    cells[nz - 2, :, 1:] = 3                          # strip B: -CTE below ...
    cells[nz - 1, :, 1:] = 2                          # ... +CTE above -> curls toward A
    mats = [_mat(1e6, 1000.0), _mat(1e6, 1000.0, cte=cte), _mat(1e6, 1000.0, cte=-cte)]
    env = _env(zeta_bond=1.0, zeta_col=0.5, self_collision=1, horizon_voxels=2.0,
               T_amp=dT, T_freq=0.0, T_phase=float(np.pi / 2))
    s = Scene("clapper", cells, L, mats, env, steps=3000,
              notes="constant dT via T_phase = pi/2; base column fixed")
    s.fixed = (s.voxel_coords()[:, 0] == 0).astype(np.uint8)
    return s


def app_a_beam():
    """E9: App. A listing: 5x10x5 of 10 MPa, nu 0.3, -Y plane fixed,
    1 kN spread over the +Y plane, SetSlowDampZ(0.013), 400 steps.  Regions
    are given as App. B workspace fractions."""
    cells = np.ones((5, 10, 5), np.uint8)
    env = _env(zeta_bond=1.0, zeta_ground=0.013)
    s = Scene("E9-appA", cells, L, [dict(E=1e7, nu=0.3, rho=1000.0, cte=0.0, mu_s=0.0,
                                         mu_d=0.0)], env, steps=400)
    s.extra["regions"] = [("fixed", (0, 0, 0), (1.0, 0.01, 1.0), (0, 0, 0)),
                          ("forced", (0, 0.99, 0), (1.0, 0.01, 1.0), (0, 0, -1000.0))]
    return s


def strained(scene, seed=1, u=1e-2, rot=1e-2, v=0.05, w=50.0, lift=True):
    """A seeded, strained initial state for ``scene`` (parity cases that load
    every term of Eq. 13-24 and 33-35 from the first step): rest sites plus
    displacements ~ N(0, (u l)^2) per component, orientations near identity
    (unit quaternion (1, r) / |(1, r)|, r ~ N(0, (rot/2)^2)), velocities ~
    N(0, v^2) m/s and angular velocities ~ N(0, w^2) rad/s turned into momenta
    with each voxel's m = rho l^3 and I = m l^2 / 6.  Voxels in the
    bottom layer are lifted by |u_z| (``lift``) so none starts inside the floor;
    with ``lift=False`` about half of them start penetrating it.
    Input generation only: no step of the method is evaluated here."""
    rng = np.random.Generator(np.random.PCG64([SEED, seed]))
    pos, quat, P, phi, latch = scene.initial_state()
    n = len(pos)
    l = scene.lattice_dim
    du = rng.normal(size=(n, 3)) * u * l
    k = scene.voxel_coords()[:, 2]
    if lift:
        du[k == 0, 2] = np.abs(du[k == 0, 2])
    pos = pos + du
    r = rng.normal(size=(n, 3)) * rot / 2
    q = np.concatenate([np.ones((n, 1)), r], 1)
    quat = q / np.linalg.norm(q, axis=1, keepdims=True)
    mats = scene.cells.ravel()[np.flatnonzero(scene.cells.ravel())]
    m = np.array([mm["rho"] for mm in scene.materials])[mats - 1] * l ** 3
    P = P + m[:, None] * rng.normal(size=(n, 3)) * v
    phi = (m * l * l / 6)[:, None] * rng.normal(size=(n, 3)) * w
    return pos, quat, P, phi, latch


CONFIGS = {
    "C1": cantilever,
    "C2": cube,
    "C2c": lambda: cube(contact_variant=True),
    "C3": hollow_sphere,
    "C4": walker,
    "C5": block,
}


def get(name, **kw):
    return CONFIGS[name](**kw)
