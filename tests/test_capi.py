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


def test_python_structs_match_the_header(pkg, tmp_path):
    """The ctypes mirrors of fdmgpu_layout / fdmgpu_krylov_report have the C
    layout of include/fdmgpu.h (size and every field offset, compiled here)."""
    import subprocess

    checks = []
    for cname, py in (("fdmgpu_layout", pkg.Layout), ("fdmgpu_krylov_report", pkg.KrylovReport)):
        checks.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            checks.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    src = tmp_path / "layout.c"
    src.write_text('#include <stddef.h>\n#include <stdio.h>\n#include "fdmgpu.h"\nint main(void) {\n' +
                   "\n".join(checks) + "\nreturn 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                       check=True).stdout.splitlines())
    for cname, py in (("fdmgpu_layout", pkg.Layout), ("fdmgpu_krylov_report", pkg.KrylovReport)):
        assert int(got[cname]) == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert int(got[f"{cname}.{f}"]) == getattr(py, f).offset, (cname, f)
