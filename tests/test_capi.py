"""The C-ABI library loads and exports every symbol include/fdmgpu.h declares
(no compute calls without a GPU); without a device the ABI fails loudly."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header, prefix="fdmgpu"):
    text = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"\b(" + prefix + r"_[a-z_]+)\s*\(", text)))


def test_header_symbols_exported(pkg):
    lib = ctypes.CDLL(pkg.LIB_PATH)
    names = declared("fdmgpu.h")
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_host_setup_symbols(pkg):
    lib = ctypes.CDLL(pkg.LIB_PATH)
    names = declared("fdmhost.h", "fdmhost")
    assert len(names) >= 15 and "fdmhost_attach" in names
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a(pkg):
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pkg.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_device_fails_loudly(pkg):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    h = ctypes.c_void_p()
    lib = pkg.lib()
    rc = lib.fdmgpu_create(ctypes.byref(h), 3, 3, 8, 100, 0)
    assert rc == 5 and not h.value  # FDMGPU_CUDA_ERROR, no CPU fallback
    with pytest.raises(pkg.FdmGpuError):
        pkg.Solver(pkg.Problem(2, 2, 2))


def test_status_strings(pkg):
    lib = pkg.lib()
    lib.fdmgpu_status_string.restype = ctypes.c_char_p
    assert lib.fdmgpu_status_string(2) == b"matrix not SPD"
