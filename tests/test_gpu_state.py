"""GPU tests of handle state across setter calls (include/fdmgpu.h documents
re-calling the setters on a live handle): the captured PCG graph and the
split-tail solve lists must follow the state they were built for."""
import os

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as T

    assert T.cuda.is_available(), "GPU tests need a CUDA device"
    return T


def test_pcg_graph_follows_new_coefficients(pkg, torch):
    """pcg -> set_cell_coeffs(2 mu) -> factor -> pcg with the same preconditioner
    and omega replays a re-captured graph: same answer as a fresh handle
    (precond 1, the smoother alone: the coarse inverse is not rescaled)."""
    prob = pkg.Problem(2, 3, 5)
    b = torch.from_numpy(prob.rhs()).cuda()
    mu2 = 2.0 * prob.geometry()["mu"]
    sol = pkg.Solver(prob)
    sol.factor()
    sol.calibrate_damping()
    w = sol.omega
    x1, rep1 = sol.pcg(b, precond=1)
    sol.set_cell_coeffs(mu2)
    sol.factor()
    sol.omega = w
    x2, rep2 = sol.pcg(b, precond=1)
    fresh = pkg.Solver(prob)
    fresh.set_cell_coeffs(mu2)
    fresh.factor()
    fresh.omega = w
    x3, rep3 = fresh.pcg(b, precond=1)
    assert rep2["iterations"] == rep3["iterations"]
    assert torch.equal(x2, x3)
    # A and the relaxation's inverse both scale (by 2 and 1/2): same
    # iterations, half the solution
    assert rep2["iterations"] == rep1["iterations"]
    assert rel(x2.cpu().numpy(), 0.5 * x1.cpu().numpy()) <= 1e-7


@pytest.mark.parametrize("cfg", [(4, 3, 15), (3, 0, 0)])
def test_set_patches_again_rebuilds_split_solve(pkg, oracle, torch, cfg):
    """set_patches re-called with the other separator order (a different tile
    pattern) on a handle whose split-tail cluster solve already ran: the
    relaxation matches the oracle before and after, and a pcg captured in
    between is re-captured."""
    prob = pkg.Problem(*cfg)
    ref = oracle.Problem(*cfg, build_global=False, threads=os.cpu_count())
    ref.factor()
    rt = ref.apply_St(prob.rhs())
    z_ref = ref.patch_apply(rt)
    sol = pkg.Solver(prob)
    sol.factor()
    L0 = sol.layout()
    assert rel(sol.patch_apply(rt), z_ref) <= 1e-11
    sol.calibrate_damping()
    b = torch.from_numpy(prob.rhs()).cuda()
    _, rep0 = sol.pcg(b)
    for order in ("reference", "plane"):
        sol.set_patches(separator_order=order)
        sol.factor()
        L1 = sol.layout()
        assert L1["separator_order"] == (1 if order == "reference" else 0)
        assert rel(sol.patch_apply(rt), z_ref) <= 1e-11
        _, rep = sol.pcg(b)
        assert rep["converged"] and rep["iterations"] == rep0["iterations"]
    assert L1["nnz_L"] == L0["nnz_L"]


def test_apply_async_after_sync_use(pkg, torch):
    """apply_async set-up happens once and survives repeated use."""
    prob = pkg.Problem(2, 3, 5)
    sol = pkg.Solver(prob)
    sol.factor()
    x = torch.from_numpy(prob.rhs()).pin_memory().numpy()
    y = torch.empty(prob.ndof, dtype=torch.float64).pin_memory().numpy()
    for _ in range(3):
        sol.apply_async(pkg.OP_SMOOTH, x, y)
        sol.synchronize()
        assert np.array_equal(y, sol.smooth(prob.rhs()))
