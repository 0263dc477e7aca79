"""ctypes declarations of include/voxsim.h (argument marshalling only).

Loading fails loudly when libvoxsim.so is missing: there is no CPU fallback.
Build it with ``python -m paper_1212_2845_b200.build`` or
``__graft_entry__.build()``.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# VX_LIB=checked loads the checked build (device bounds checks and shared-memory
# race tags; paper_1212_2845_b200/build.py) -- for test runs, never the product path
LIB_PATH = os.path.join(HERE, {"checked": "libvoxsim_checked.so",
                               "oldparity": "libvoxsim_oldparity.so"}.get(os.environ.get("VX_LIB", ""),
                                                                       "libvoxsim.so"))

# status codes (vx_status)
VX_OK = 0
VX_ERR_INVALID_ARG = -1
VX_ERR_OUT_OF_RANGE = -2
VX_ERR_CUDA = -3
VX_ERR_NCCL = -4
VX_ERR_OOM = -5
VX_ERR_DIVERGED = -6
VX_ERR_STATE = -7
VX_ERR_NO_DEVICE = -8


class vx_lattice_desc(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("lattice_dim", ctypes.c_double), ("origin", ctypes.c_double * 3),
                ("cells", ctypes.c_void_p), ("precision", ctypes.c_int32),
                ("device", ctypes.c_int32), ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("nccl_id", ctypes.c_void_p)]


class vx_material(ctypes.Structure):
    _fields_ = [("E", ctypes.c_double), ("nu", ctypes.c_double), ("rho", ctypes.c_double),
                ("cte", ctypes.c_double), ("mu_s", ctypes.c_double), ("mu_d", ctypes.c_double)]


class vx_env(ctypes.Structure):
    _fields_ = [("gravity", ctypes.c_double), ("floor_on", ctypes.c_int32),
                ("floor_z", ctypes.c_double), ("T_ref", ctypes.c_double),
                ("T_amp", ctypes.c_double), ("T_freq", ctypes.c_double),
                ("T_phase", ctypes.c_double), ("zeta_bond", ctypes.c_double),
                ("zeta_ground", ctypes.c_double), ("zeta_col", ctypes.c_double),
                ("horizon_voxels", ctypes.c_double), ("dt_safety", ctypes.c_double),
                ("self_collision", ctypes.c_int32)]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double
_DP = ctypes.POINTER(ctypes.c_double)

# name -> (restype, argtypes); every symbol declared in include/voxsim.h
SIGNATURES = {
    "vx_create_lattice": (_I32, [ctypes.POINTER(vx_lattice_desc), ctypes.POINTER(_P)]),
    "vx_set_materials": (_I32, [_P, ctypes.POINTER(vx_material), _I32]),
    "vx_set_environment": (_I32, [_P, ctypes.POINTER(vx_env)]),
    "vx_set_boundary": (_I32, [_P, _P, _P]),
    "vx_add_region": (_I32, [_P, _I32, _DP, _DP, _DP]),
    "vx_set_state": (_I32, [_P, _P, _P, _P, _P, _P]),
    "vx_set_step": (_I32, [_P, _I64]),
    "vx_checkpoint_bytes": (_I64, [_P]),
    "vx_save_checkpoint": (_I32, [_P, _P, _I64]),
    "vx_load_checkpoint": (_I32, [_P, _P, _I64]),
    "vx_step": (_I32, [_P, _I64]),
    "vx_prepare_steps": (_I32, [_P, _I64]),
    "vx_read_state": (_I32, [_P, _P, _P, _P, _P, _P]),
    "vx_read_voxels": (_I32, [_P, _P, _I64, _P, _P, _P, _P, _P]),
    "vx_dt": (_D, [_P]),
    "vx_num_voxels": (_I64, [_P]),
    "vx_num_bonds": (_I64, [_P]),
    "vx_num_surface": (_I64, [_P]),
    "vx_steps_done": (_I64, [_P]),
    "vx_num_contact_pairs": (_I64, [_P]),
    "vx_num_rebuilds": (_I64, [_P]),
    "vx_owned_planes": (_I32, [_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "vx_stream": (_P, [_P]),
    "vx_contact_pairs": (_I64, [_P, _P, _I64]),
    "vx_set_instrumentation": (_I32, [_P, _I32]),
    "vx_kernel_times": (_I32, [_P, _DP, ctypes.POINTER(_I64)]),
    "vx_launches_per_step": (_I32, [_P]),
    "vx_set_engine": (_I32, [_P, _I32]),
    "vx_set_batch": (_I32, [_P, _I32]),
    "vx_set_batch_z": (_I32, [_P, _I32]),
    "vx_set_batch_y": (_I32, [_P, _I32]),
    "vx_num_scenes": (_I32, [_P]),
    "vx_get_engine": (_I32, [_P]),
    "vx_destroy": (None, [_P]),
    "vx_last_error": (ctypes.c_char_p, []),
    "vx_nccl_unique_id": (_I32, [_P]),
    "vx_slab_planes": (_I32, [_I32, _I32, _I32, ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "vx_abi_version": (_I32, []),
    "vx_num_owned": (_I64, [_P]),
    "vx_owned_ids": (_I32, [_P, _P]),
    "vx_set_state_owned": (_I32, [_P, _P, _P, _P, _P, _P]),
    "vx_read_state_owned": (_I32, [_P, _P, _P, _P, _P, _P]),
}

_lib = None


ABI_VERSION = 3   # include/voxsim.h VOXSIM_ABI_VERSION


def load():
    """Load libvoxsim.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build the CUDA extension with "
                              "`python -m paper_1212_2845_b200.build` (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        # the ABI version first: a stale library may lack later symbols
        ver = getattr(L, "vx_abi_version", None)
        if ver is not None:
            ver.restype, ver.argtypes = _I32, []
        have = ver() if ver is not None else None
        if have != ABI_VERSION:
            raise ImportError(f"{LIB_PATH} has ABI {have}, this binding needs "
                              f"{ABI_VERSION}: rebuild with `python -m paper_1212_2845_b200.build`")
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
