"""C ABI: the library loads and exports every symbol include/voxsim.h declares;
without a GPU it refuses to run (no CPU fallback).  CPU only."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "voxsim.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vx_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("vx_create_lattice", "vx_set_materials", "vx_set_environment", "vx_step",
              "vx_read_state", "vx_destroy", "vx_last_error"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_1212_2845_b200 import _native
    lib = _native.load()
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_declared()) == set(_native.SIGNATURES)
    assert lib.vx_abi_version() == 3


def test_no_cpu_fallback_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1212_2845_b200 import Lattice, NoDeviceError
    with pytest.raises(NoDeviceError):
        Lattice.create_lattice(np.ones((1, 1, 2), np.uint8), 1e-3)


def test_invalid_arguments_rejected_before_device():
    from paper_1212_2845_b200 import Lattice, VoxError
    with pytest.raises(VoxError) as e:
        Lattice.create_lattice(np.ones((1, 1, 2), np.uint8), -1.0)
    assert e.value.status == -1
    with pytest.raises(VoxError):
        Lattice.create_lattice(np.ones((1, 1, 2), np.uint8), 1e-3, precision=16)


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1212_2845_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt
                assert "oracle.h" not in txt
