"""TEST INFRASTRUCTURE ONLY -- the fp64 CPU oracle for arXiv:1212.2845.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA product path (``paper_1212_2845_b200``); the two meet only through the
seeded input generators in ``workloads/``.

Python side of the oracle: a ctypes wrapper around ``oracle.cpp`` (the stepper,
written from the paper step by step) plus the plain-numpy direct stiffness
method (``oracle.dsm``) and the cantilever elastica (``oracle.elastica``).

Pins (tests/test_oracle_pins.py; DESIGN.md §6 lists them per function): every
oracle function is checked against something other than itself -- the paper's
worked examples and tables (tests/golden/), closed forms, invariants, brute
force.  The floor penalty constants (R14), the friction law's constants (R15)
and the self-collision penalty law (the paper leaves
them open) are readings: they are pinned to the closed forms of the reading
(resting penetration m g / k_f, the Eq. 38 halting threshold, breakaway at
mu_s F_n and deceleration mu_d g, one pair's penalty force and momentum
balance, the brute-force pair definition), not to a number the paper prints.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
# tools/oracle_mutants.py points this at a deliberately broken build of
# oracle.cpp to check that the pins fail (a mutation test of the pins)
_LIB_OVERRIDE = os.environ.get("VX_ORACLE_LIB")


def build(force: bool = False) -> str:
    """Compile oracle.cpp with -O2 -ffp-contract=off (no fast-math), OpenMP."""
    src = os.path.join(_HERE, "oracle.cpp")
    hdr = os.path.join(_HERE, "oracle.h")
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
           "-shared", "-fPIC", "-o", tmp, src]
    subprocess.run(cmd, check=True)
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class OrcMaterial(ctypes.Structure):
    _fields_ = [("E", ctypes.c_double), ("nu", ctypes.c_double), ("rho", ctypes.c_double),
                ("cte", ctypes.c_double), ("mu_s", ctypes.c_double), ("mu_d", ctypes.c_double)]


class OrcEnv(ctypes.Structure):
    _fields_ = [("gravity", ctypes.c_double), ("floor_on", ctypes.c_int32),
                ("floor_z", ctypes.c_double), ("T_ref", ctypes.c_double),
                ("T_amp", ctypes.c_double), ("T_freq", ctypes.c_double),
                ("T_phase", ctypes.c_double), ("zeta_bond", ctypes.c_double),
                ("zeta_ground", ctypes.c_double), ("zeta_col", ctypes.c_double),
                ("horizon_voxels", ctypes.c_double), ("dt_safety", ctypes.c_double),
                ("self_collision", ctypes.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if _LIB_OVERRIDE:
            L = ctypes.CDLL(_LIB_OVERRIDE)
        else:
            build()
            L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        dp = ctypes.POINTER(ctypes.c_double)
        L.orc_create.restype = P
        L.orc_create.argtypes = [ctypes.c_int32] * 3 + [ctypes.c_double, dp, P,
                                                         ctypes.POINTER(OrcMaterial),
                                                         ctypes.c_int32, ctypes.POINTER(OrcEnv)]
        L.orc_destroy.argtypes = [P]
        L.orc_last_error.restype = ctypes.c_char_p
        for f in ("orc_num_voxels", "orc_num_bonds", "orc_num_surface", "orc_get_step"):
            getattr(L, f).restype = ctypes.c_int64
            getattr(L, f).argtypes = [P]
        L.orc_dt.restype = ctypes.c_double
        L.orc_dt.argtypes = [P]
        L.orc_set_boundary.argtypes = [P, P, P]
        L.orc_add_region.argtypes = [P, ctypes.c_int32, dp, dp, dp]
        L.orc_set_state.argtypes = [P, P, P, P, P, P]
        L.orc_read_state.argtypes = [P, P, P, P, P, P]
        L.orc_set_step.argtypes = [P, ctypes.c_int64]
        L.orc_set_threads.argtypes = [P, ctypes.c_int32]
        L.orc_set_dt.argtypes = [P, ctypes.c_double]
        L.orc_step.argtypes = [P, ctypes.c_int64]
        L.orc_composite.argtypes = [ctypes.c_double] * 4 + [dp]
        L.orc_beam_constants.argtypes = [ctypes.c_double] * 3 + [dp]
        L.orc_bond_loads.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, dp, dp,
                                     ctypes.c_double, dp]
        L.orc_contact_pairs.restype = ctypes.c_int64
        L.orc_contact_pairs.argtypes = [P, P, ctypes.c_int64]
        _lib = L
    return _lib


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def composite(E1, nu1, E2, nu2):
    """Eq. 1-3 -> (E_c, G_c, mu_c)."""
    out = np.zeros(3)
    lib().orc_composite(E1, nu1, E2, nu2, _dptr(out))
    return tuple(out)


def beam_constants(Ec, Gc, l):
    """Eq. 4-12 -> (a1, a2, b1, b2, b3)."""
    out = np.zeros(5)
    lib().orc_beam_constants(Ec, Gc, l, _dptr(out))
    return tuple(out)


@dataclass
class State:
    pos: np.ndarray      # (N,3) absolute positions D
    quat: np.ndarray     # (N,4) w,x,y,z
    linmom: np.ndarray   # (N,3) P
    angmom: np.ndarray   # (N,3) phi
    latch: np.ndarray    # (N,) uint8


class OracleSim:
    """fp64 oracle simulation of one lattice (ids = filled cells, x-fastest)."""

    def __init__(self, cells, lattice_dim, materials, env, origin=(0.0, 0.0, 0.0)):
        cells = np.ascontiguousarray(cells, dtype=np.uint8)   # shape (nz, ny, nx)
        nz, ny, nx = cells.shape
        mats = (OrcMaterial * len(materials))()
        for i, m in enumerate(materials):
            mats[i] = OrcMaterial(m["E"], m["nu"], m["rho"], m.get("cte", 0.0),
                                  m.get("mu_s", 0.0), m.get("mu_d", 0.0))
        e = OrcEnv(env.get("gravity", 0.0), int(env.get("floor_on", 0)), env.get("floor_z", 0.0),
                   env.get("T_ref", 0.0), env.get("T_amp", 0.0), env.get("T_freq", 0.0),
                   env.get("T_phase", 0.0), env.get("zeta_bond", 0.0),
                   env.get("zeta_ground", 0.0), env.get("zeta_col", 0.0),
                   env.get("horizon_voxels", 2.0), env.get("dt_safety", 1.0),
                   int(env.get("self_collision", 0)))
        org = np.asarray(origin, dtype=np.float64)
        self._cells = cells
        h = lib().orc_create(nx, ny, nz, float(lattice_dim), _dptr(org),
                             cells.ctypes.data_as(ctypes.c_void_p), mats, len(materials),
                             ctypes.byref(e))
        if not h:
            raise ValueError(lib().orc_last_error().decode())
        self._h = h
        self.n = int(lib().orc_num_voxels(h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.orc_destroy(h)
            self._h = None

    # --- queries ---
    @property
    def dt(self):
        return lib().orc_dt(self._h)

    @property
    def num_bonds(self):
        return int(lib().orc_num_bonds(self._h))

    @property
    def num_surface(self):
        return int(lib().orc_num_surface(self._h))

    @property
    def step_count(self):
        return int(lib().orc_get_step(self._h))

    # --- setup ---
    def set_threads(self, n):
        lib().orc_set_threads(self._h, int(n))

    def set_dt(self, dt):
        lib().orc_set_dt(self._h, float(dt))

    def set_boundary(self, fixed=None, fext=None):
        f = None if fixed is None else np.ascontiguousarray(fixed, dtype=np.uint8)
        x = None if fext is None else np.ascontiguousarray(fext, dtype=np.float64)
        lib().orc_set_boundary(self._h, None if f is None else f.ctypes.data,
                               None if x is None else x.ctypes.data)

    def add_region(self, kind, origin, size, force=(0.0, 0.0, 0.0)):
        o = np.asarray(origin, np.float64)
        s = np.asarray(size, np.float64)
        f = np.asarray(force, np.float64)
        k = {"fixed": 0, "forced": 1}.get(kind, kind)
        if lib().orc_add_region(self._h, int(k), _dptr(o), _dptr(s), _dptr(f)):
            raise ValueError(lib().orc_last_error().decode())

    def set_state(self, pos=None, quat=None, linmom=None, angmom=None, latch=None):
        arrs = []
        for a, dt_ in ((pos, np.float64), (quat, np.float64), (linmom, np.float64),
                       (angmom, np.float64), (latch, np.uint8)):
            arrs.append(None if a is None else np.ascontiguousarray(a, dtype=dt_))
        lib().orc_set_state(self._h, *[None if a is None else a.ctypes.data for a in arrs])

    def set_step(self, n):
        lib().orc_set_step(self._h, int(n))

    def read_state(self) -> State:
        n = self.n
        s = State(np.zeros((n, 3)), np.zeros((n, 4)), np.zeros((n, 3)), np.zeros((n, 3)),
                  np.zeros(n, np.uint8))
        lib().orc_read_state(self._h, s.pos.ctypes.data, s.quat.ctypes.data,
                             s.linmom.ctypes.data, s.angmom.ctypes.data, s.latch.ctypes.data)
        return s

    def step(self, n=1):
        r = lib().orc_step(self._h, int(n))
        if r:
            raise FloatingPointError(lib().orc_last_error().decode())

    def bond_loads(self, a_mat, b_mat, axis, state_a, state_b, dT=0.0):
        sa = np.ascontiguousarray(state_a, np.float64)
        sb = np.ascontiguousarray(state_b, np.float64)
        out = np.zeros(12)
        lib().orc_bond_loads(self._h, a_mat, b_mat, axis, _dptr(sa), _dptr(sb), float(dT),
                             _dptr(out))
        return out[0:3], out[3:6], out[6:9], out[9:12]

    def contact_pairs(self, cap=1 << 20):
        buf = np.zeros(2 * cap, np.int32)
        n = int(lib().orc_contact_pairs(self._h, buf.ctypes.data, cap))
        return buf[:2 * min(n, cap)].reshape(-1, 2)
