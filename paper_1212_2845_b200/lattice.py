"""Thin Python binding of the C ABI (include/voxsim.h): same names, argument
marshalling only -- every step of the path runs in libvoxsim.so's kernels."""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N


class VoxError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[{status}] {msg}")
        self.status = status


class DivergedError(VoxError):
    pass


class NoDeviceError(VoxError):
    pass


def _check(status):
    if status != N.VX_OK:
        msg = N.load().vx_last_error().decode()
        cls = {N.VX_ERR_DIVERGED: DivergedError, N.VX_ERR_NO_DEVICE: NoDeviceError}.get(status, VoxError)
        raise cls(status, msg)


def _ptr(a):
    return None if a is None else a.ctypes.data


def _arr(a, n, cols, dtype, name, out=False):
    """A C-contiguous array of shape (n, cols) (cols 0: (n,)) and the dtype the
    C ABI reads or writes; the library copies n * cols elements, so a short or
    mistyped buffer is refused here rather than overrun there."""
    if a is None:
        return None
    shape = (n,) if cols == 0 else (n, cols)
    if out:
        if not (isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous
                and a.shape == shape):
            raise ValueError(f"{name}: need a C-contiguous {np.dtype(dtype).name} array of shape "
                             f"{shape}, got {getattr(a, 'dtype', type(a))} {getattr(a, 'shape', '')}")
        return a
    a = np.ascontiguousarray(a, dtype=dtype)
    if a.shape != shape and not (cols and a.shape == (n * cols,)):
        raise ValueError(f"{name}: need shape {shape}, got {a.shape}")
    return a


@dataclass
class State:
    pos: np.ndarray      # (n,3) absolute positions D, m
    quat: np.ndarray     # (n,4) w,x,y,z
    linmom: np.ndarray   # (n,3) P
    angmom: np.ndarray   # (n,3) phi
    latch: np.ndarray    # (n,) uint8


def slab_planes(nx, nranks, rank):
    """(x_begin, x_end) of rank's x-slab (vx_slab_planes; host-only)."""
    a, b = ctypes.c_int32(), ctypes.c_int32()
    _check(N.load().vx_slab_planes(int(nx), int(nranks), int(rank), ctypes.byref(a),
                                   ctypes.byref(b)))
    return a.value, b.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(N.load().vx_nccl_unique_id(buf))
    return buf.raw


class Lattice:
    """One voxel lattice on one GPU (one x-slab of it when nranks > 1)."""

    def __init__(self, handle, n):
        self._h = handle
        self.n = n

    # ------------------------------------------------------------ vx_create_lattice
    @classmethod
    def create_lattice(cls, cells, lattice_dim, origin=(0.0, 0.0, 0.0), precision=32, device=0,
                       rank=0, nranks=1, nccl_id=None):
        """cells: uint8 array of shape (nz, ny, nx) (flat order x-fastest)."""
        L = N.load()
        cells = np.ascontiguousarray(cells, dtype=np.uint8)
        nz, ny, nx = cells.shape
        d = N.vx_lattice_desc()
        d.nx, d.ny, d.nz = nx, ny, nz
        d.lattice_dim = float(lattice_dim)
        d.origin = (ctypes.c_double * 3)(*[float(x) for x in origin])
        d.cells = cells.ctypes.data
        d.precision = int(precision)
        d.device, d.rank, d.nranks = int(device), int(rank), int(nranks)
        idbuf = None
        if nccl_id is not None:
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            d.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
        h = ctypes.c_void_p()
        _check(L.vx_create_lattice(ctypes.byref(d), ctypes.byref(h)))
        return cls(h, int(L.vx_num_voxels(h)))

    def destroy(self):
        if getattr(self, "_h", None):
            N.load().vx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    # ------------------------------------------------------------ setup
    def set_materials(self, materials):
        arr = (N.vx_material * len(materials))()
        for i, m in enumerate(materials):
            arr[i] = N.vx_material(m["E"], m["nu"], m["rho"], m.get("cte", 0.0),
                                   m.get("mu_s", 0.0), m.get("mu_d", 0.0))
        _check(N.load().vx_set_materials(self._h, arr, len(materials)))

    def set_environment(self, env):
        e = N.vx_env(env.get("gravity", 0.0), int(env.get("floor_on", 0)),
                     env.get("floor_z", 0.0), env.get("T_ref", 0.0), env.get("T_amp", 0.0),
                     env.get("T_freq", 0.0), env.get("T_phase", 0.0),
                     env.get("zeta_bond", 0.0), env.get("zeta_ground", 0.0),
                     env.get("zeta_col", 0.0), env.get("horizon_voxels", 2.0),
                     env.get("dt_safety", 1.0), int(env.get("self_collision", 0)))
        _check(N.load().vx_set_environment(self._h, ctypes.byref(e)))

    def set_boundary(self, fixed=None, f_ext=None):
        f = _arr(fixed, self.n, 0, np.uint8, "fixed")
        x = _arr(f_ext, self.n, 3, np.float64, "f_ext")
        _check(N.load().vx_set_boundary(self._h, _ptr(f), _ptr(x)))

    def add_region(self, kind, origin, size, force=(0.0, 0.0, 0.0)):
        k = {"fixed": 0, "forced": 1}.get(kind, kind)
        o = (ctypes.c_double * 3)(*map(float, origin))
        s = (ctypes.c_double * 3)(*map(float, size))
        f = (ctypes.c_double * 3)(*map(float, force))
        _check(N.load().vx_add_region(self._h, int(k), o, s, f))

    def set_state(self, pos=None, quat=None, linmom=None, angmom=None, latch=None):
        arrs = [_arr(a, self.n, c, t, nm)
                for a, c, t, nm in ((pos, 3, np.float64, "pos"), (quat, 4, np.float64, "quat"),
                                    (linmom, 3, np.float64, "linmom"),
                                    (angmom, 3, np.float64, "angmom"), (latch, 0, np.uint8, "latch"))]
        _check(N.load().vx_set_state(self._h, *[_ptr(a) for a in arrs]))

    def save_checkpoint(self) -> bytes:
        """Exact device-state snapshot (bitwise resume)."""
        n = int(N.load().vx_checkpoint_bytes(self._h))
        buf = ctypes.create_string_buffer(n)
        _check(N.load().vx_save_checkpoint(self._h, buf, n))
        return buf.raw

    def load_checkpoint(self, blob: bytes):
        buf = ctypes.create_string_buffer(bytes(blob), len(blob))
        _check(N.load().vx_load_checkpoint(self._h, buf, len(blob)))

    def set_step(self, n):
        _check(N.load().vx_set_step(self._h, int(n)))

    # ------------------------------------------------------------ stepping
    def prepare_steps(self, n):
        """Build the CUDA graphs step(n) will replay, without advancing the state."""
        _check(N.load().vx_prepare_steps(self._h, int(n)))

    def step(self, n=1):
        _check(N.load().vx_step(self._h, int(n)))

    def read_state(self, out: State | None = None) -> State:
        n = self.n
        if out is None:
            out = State(np.empty((n, 3)), np.empty((n, 4)), np.empty((n, 3)), np.empty((n, 3)),
                        np.empty(n, np.uint8))
        else:
            for a, c, t, nm in ((out.pos, 3, np.float64, "pos"), (out.quat, 4, np.float64, "quat"),
                                (out.linmom, 3, np.float64, "linmom"),
                                (out.angmom, 3, np.float64, "angmom"),
                                (out.latch, 0, np.uint8, "latch")):
                _arr(a, n, c, t, nm, out=True)
        _check(N.load().vx_read_state(self._h, _ptr(out.pos), _ptr(out.quat), _ptr(out.linmom),
                                      _ptr(out.angmom), _ptr(out.latch)))
        return out

    # ------------------------------------------------------------ owned-voxel I/O
    def owned_ids(self):
        """External ids of the voxels in this rank's slab, ascending (vx_owned_ids)."""
        m = int(N.load().vx_num_owned(self._h))
        if m < 0:
            raise VoxError(m, "vx_num_owned failed")
        ids = np.empty(m, np.int64)
        if m:
            _check(N.load().vx_owned_ids(self._h, ids.ctypes.data))
        return ids

    def set_state_owned(self, pos=None, quat=None, linmom=None, angmom=None, latch=None):
        """State of this rank's voxels only, in owned_ids() order (vx_set_state_owned)."""
        m = int(N.load().vx_num_owned(self._h))
        arrs = [_arr(a, m, c, t, nm)
                for a, c, t, nm in ((pos, 3, np.float64, "pos"), (quat, 4, np.float64, "quat"),
                                    (linmom, 3, np.float64, "linmom"),
                                    (angmom, 3, np.float64, "angmom"), (latch, 0, np.uint8, "latch"))]
        _check(N.load().vx_set_state_owned(self._h, *[_ptr(a) for a in arrs]))

    def read_state_owned(self, out: State | None = None) -> State:
        """State of this rank's voxels, in owned_ids() order (vx_read_state_owned)."""
        m = int(N.load().vx_num_owned(self._h))
        if out is None:
            out = State(np.empty((m, 3)), np.empty((m, 4)), np.empty((m, 3)), np.empty((m, 3)),
                        np.empty(m, np.uint8))
        else:
            for a, c, t, nm in ((out.pos, 3, np.float64, "pos"), (out.quat, 4, np.float64, "quat"),
                                (out.linmom, 3, np.float64, "linmom"),
                                (out.angmom, 3, np.float64, "angmom"),
                                (out.latch, 0, np.uint8, "latch")):
                _arr(a, m, c, t, nm, out=True)
        _check(N.load().vx_read_state_owned(self._h, _ptr(out.pos), _ptr(out.quat), _ptr(out.linmom),
                                            _ptr(out.angmom), _ptr(out.latch)))
        return out

    def read_voxels(self, ids) -> State:
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        n = len(ids)
        out = State(np.empty((n, 3)), np.empty((n, 4)), np.empty((n, 3)), np.empty((n, 3)),
                    np.empty(n, np.uint8))
        _check(N.load().vx_read_voxels(self._h, _ptr(ids), n, _ptr(out.pos), _ptr(out.quat),
                                       _ptr(out.linmom), _ptr(out.angmom), _ptr(out.latch)))
        return out

    # ------------------------------------------------------------ queries
    @property
    def dt(self):
        return N.load().vx_dt(self._h)

    @property
    def num_voxels(self):
        return int(N.load().vx_num_voxels(self._h))

    @property
    def num_bonds(self):
        return int(N.load().vx_num_bonds(self._h))

    @property
    def num_surface(self):
        return int(N.load().vx_num_surface(self._h))

    @property
    def steps_done(self):
        return int(N.load().vx_steps_done(self._h))

    @property
    def num_contact_pairs(self):
        return int(N.load().vx_num_contact_pairs(self._h))

    @property
    def num_rebuilds(self):
        return int(N.load().vx_num_rebuilds(self._h))

    def contact_pairs(self, cap=1 << 22):
        """Current collision shortlist as (n,2) external ids, a < b."""
        buf = np.zeros(2 * cap, np.int64)
        n = int(N.load().vx_contact_pairs(self._h, buf.ctypes.data, cap))
        if n < 0:
            raise VoxError(n, "vx_contact_pairs failed")
        return buf[:2 * min(n, cap)].reshape(-1, 2)

    def owned_planes(self):
        a, b = ctypes.c_int32(), ctypes.c_int32()
        N.load().vx_owned_planes(self._h, ctypes.byref(a), ctypes.byref(b))
        return a.value, b.value

    @property
    def stream(self) -> int:
        """cudaStream_t of the library (wrap with torch.cuda.ExternalStream)."""
        return int(N.load().vx_stream(self._h) or 0)

    def set_instrumentation(self, on=True, stride=1):
        """Per-launch CUDA-event timing inside the step graphs, on every
        `stride`-th step (vx_set_instrumentation)."""
        _check(N.load().vx_set_instrumentation(self._h, int(stride) if on else 0))

    def kernel_times(self):
        ms = (ctypes.c_double * 4)()
        cnt = (ctypes.c_int64 * 4)()
        _check(N.load().vx_kernel_times(self._h, ms, cnt))
        names = ("bonds", "integrate", "other", "all")
        return {k: (ms[i], cnt[i]) for i, k in enumerate(names)}

    def set_batch(self, stride):
        """Declare K scenes packed along x, `stride` planes each (incl. separator)."""
        _check(N.load().vx_set_batch(self._h, int(stride)))

    def set_batch_y(self, stride):
        """Declare scenes stacked along y as well, `stride` rows each (incl. separator)."""
        _check(N.load().vx_set_batch_y(self._h, int(stride)))

    def set_batch_z(self, stride):
        """Declare scenes stacked along z as well, `stride` layers each (incl. separator)."""
        _check(N.load().vx_set_batch_z(self._h, int(stride)))

    @property
    def num_scenes(self):
        return int(N.load().vx_num_scenes(self._h))

    ENGINES = {"two_pass": 0, "fused": 1, "auto": 2}

    def set_engine(self, engine):
        """'two_pass' (K3 + K4), 'fused' (one kernel per step) or 'auto' (the
        default: the faster one for this lattice, chosen at the first step)."""
        _check(N.load().vx_set_engine(self._h, self.ENGINES.get(engine, engine)))

    @property
    def engine(self):
        e = int(N.load().vx_get_engine(self._h))
        return {v: k for k, v in self.ENGINES.items()}.get(e, e)

    @property
    def launches_per_step(self):
        return int(N.load().vx_launches_per_step(self._h))


def create_lattice(*a, **kw) -> Lattice:
    return Lattice.create_lattice(*a, **kw)


def from_scene(scene, precision=None, device=0, rank=0, nranks=1, nccl_id=None,
               init_state=True, engine=None) -> Lattice:
    """Convenience: a Lattice set up from a workloads.Scene (no arithmetic).
    ``init_state=False`` keeps the library's initial state (at rest on the
    lattice sites), which equals the scene's when it has no v0."""
    lat = Lattice.create_lattice(scene.cells, scene.lattice_dim, scene.origin,
                                 precision or scene.precision, device, rank, nranks, nccl_id)
    lat.set_materials(scene.materials)
    lat.set_environment(scene.env)
    if engine is not None:
        lat.set_engine(engine)
    if scene.fixed is not None or scene.fext is not None:
        lat.set_boundary(scene.fixed, scene.fext)
    for kind, org, size, force in scene.extra.get("regions", []):
        lat.add_region(kind, org, size, force)
    if init_state:
        lat.set_state(*scene.initial_state())
    return lat
