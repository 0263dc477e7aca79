"""B200-native voxel soft-body stepper (Hiller & Lipson, arXiv:1212.2845).

The product path is libvoxsim.so (hand-written CUDA for sm_100a behind the C
ABI of include/voxsim.h); this package is its thin ctypes binding.
"""
from .lattice import (DivergedError, Lattice, NoDeviceError, State, VoxError, create_lattice, slab_planes,
                      from_scene, nccl_unique_id)

__all__ = ["Lattice", "State", "VoxError", "DivergedError", "NoDeviceError", "create_lattice",
           "from_scene", "nccl_unique_id", "slab_planes"]
