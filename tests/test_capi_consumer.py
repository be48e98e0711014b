"""The drop-in boundary from C++: tests/integration/capi_consumer.cpp (a caller
compiled against include/fdmgpu.h + fdmhost.h only, linked against
lib/libfdmgpu.so) and the INTEGRATION.md adapter gpu_twolevel.hpp (compiled
against declaration stubs of the reference headers), both built by
csrc/Makefile in build()."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_2107_14758_b200", "build")
CONSUMER = os.path.join(BUILD, "capi_consumer")


def test_consumer_and_adapter_built(pkg):
    assert os.path.exists(os.path.join(BUILD, "gpu_twolevel_adapter.o"))
    assert os.access(CONSUMER, os.X_OK)
    # links against the in-tree library and starts (usage, no device needed)
    res = subprocess.run([CONSUMER], capture_output=True, text=True, timeout=60)
    assert res.returncode == 2 and "usage" in res.stderr
    ldd = subprocess.run(["ldd", CONSUMER], capture_output=True, text=True, timeout=60).stdout
    assert "libfdmgpu.so" in ldd and "not found" not in ldd


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [(2, 0, 0), (1, 0, 0), (4, 3, 5)])
def test_cpp_consumer_matches_python_path(pkg, cfg):
    import torch

    res = subprocess.run([CONSUMER, *map(str, cfg)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr
    out = json.loads(res.stdout.strip().splitlines()[-1])
    prob = pkg.Problem(*cfg)
    sol = pkg.Solver(prob)
    sol.factor()
    w = sol.calibrate_damping()
    _, rep = sol.pcg(torch.from_numpy(prob.rhs()).cuda(), rtol=1e-8, maxit=200)
    assert out["ndof"] == prob.ndof and out["npatch"] == prob.npatches
    assert abs(out["omega"] - w["omega"]) <= 1e-10 * w["omega"]
    assert out["converged"] == 1 and out["iterations"] == rep["iterations"]
    assert abs(out["kappa"] - rep["kappa"]) <= 1e-8 * rep["kappa"]
    vn = np.linalg.norm(sol.vcycle(prob.rhs(), omega=out["omega"]))
    assert abs(out["vcycle_norm"] - vn) <= 1e-11 * vn
    assert out["not_spd_status"] == 2 and out["not_spd_message"].startswith("cholesky: matrix not SPD at pivot 0")
