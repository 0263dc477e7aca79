"""Build libvoxsim.so (sm_100a) in-tree with nvcc.

    python -m paper_1212_2845_b200.build

Links torch's bundled NCCL (nvidia/nccl, 2.28.x) -- never the system copy --
so the library and torch.distributed share one NCCL in a process.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libvoxsim.so")
# build variants: the product library, the checked one (device bounds checks and
# shared-memory race tags, vx_common.cuh; `VX_LIB=checked` selects it) and the
# checked one with round 1's zrec parity restored (the race probe's positive control)
VARIANTS = {None: ("libvoxsim.so", []),
            "checked": ("libvoxsim_checked.so", ["-DVX_CHECKED"]),
            "oldparity": ("libvoxsim_oldparity.so", ["-DVX_CHECKED", "-DVX_RACE_OLDPARITY"])}


def lib_path(variant=None) -> str:
    return os.path.join(HERE, VARIANTS[variant][0])
SOURCES = [os.path.join(HERE, "csrc", "voxsim.cu")]
DEPS = SOURCES + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [
    os.path.join(ROOT, "include", "voxsim.h")]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import nvidia  # the torch wheel's CUDA components
    for p in nvidia.__path__:
        d = os.path.join(p, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("torch-bundled NCCL (nvidia/nccl) not found")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def needs_build(variant=None) -> bool:
    lib = lib_path(variant)
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, variant=None) -> str:
    lib = lib_path(variant)
    if not force and not needs_build(variant):
        return lib
    nd = nccl_dir()
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"),
           "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
           "-Xlinker", "-rpath," + os.path.join(nd, "lib"), *VARIANTS[variant][1], "-o", tmp, *SOURCES,
           *os.environ.get("VX_NVCC_EXTRA", "").split()]   # experiments only
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), None)
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, variant=var))
