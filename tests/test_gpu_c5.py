"""GPU parity at p = 31 (config C5) against the CPU oracle.

C5 is the largest configuration (8^3 perturbed hexes, Q31, 343 patches of
226,981 DOFs).  The oracle cannot factor all of it (~160 GB
of reference-layout factors, 143 s per patch), so parity is established on

* the one-patch C5 mesh (2^3 cells, p = 31, the centre vertex perturbed): the
  whole relaxation path -- patch solve, smooth, V-cycle, damping, PCG count --
  against the oracle at the north-star tolerances (one oracle factorisation of
  8.66e10 multiply-adds, src/cholesky.cpp:9-87);
* sampled patches of the full C5 problem: CholFactor::solve of patch j
  (src/cholesky.cpp:89-110) through fdmgpu_patch_solve_one against the oracle's
  factor of the same patch, factored on the fly.

Tolerances as tests/test_gpu_parity.py: patch solve / relaxation / V-cycle
rel-l2 <= 1e-11, S / S^T / A <= 1e-12, identical PCG counts, omega <= 1e-10.
"""
import os

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu
TOL_RELAX = 1e-11
TOL_TRANSFORM = 1e-12


@pytest.fixture(scope="module")
def torch():
    import torch as T

    assert T.cuda.is_available(), "GPU tests need a CUDA device"
    return T


@pytest.fixture(scope="module")
def one_patch(pkg, oracle, torch):
    cfg = (5, 2, 31)
    prob = pkg.Problem(*cfg)
    sol = pkg.Solver(prob)
    sol.factor()
    ref = oracle.Problem(*cfg, build_global=True, threads=os.cpu_count())
    ref.factor()  # one p = 31 patch: 8.66e10 multiply-adds on one core
    return prob, sol, ref


def test_p31_relaxation_matches_oracle(one_patch):
    prob, sol, ref = one_patch
    assert prob.npatches == 1 and prob.p == 31
    r = prob.rhs()
    rt = ref.apply_St(r)
    assert rel(sol.apply_St(r), rt) <= TOL_TRANSFORM
    assert rel(sol.apply_A(r), ref.apply_A(r)) <= TOL_TRANSFORM
    # PatchSolver::apply (src/schwarz.cpp:41-54) and TwoLevel::smooth (:121-123)
    assert rel(sol.patch_apply(rt), ref.patch_apply(rt)) <= TOL_RELAX
    assert rel(sol.smooth(r), ref.smooth(r)) <= TOL_RELAX
    # the lone patch's CholFactor::solve
    n = int(ref.patches_n(0))
    rj = np.random.default_rng(31).uniform(-1, 1, n)
    assert rel(sol.patch_solve_one(0, rj), ref.patch_solve_one(0, rj)) <= TOL_RELAX


def test_p31_smooth_keeps_interior_rhs_cell_local(one_patch):
    """The slab path sums only the cell-boundary entries of S^T r over the cells and rebuilds the
    cell interiors from the E-vector of the S^T pass (single-owner entries: the same values the
    full gather would copy).  FDMGPU_SMOOTH_LOCAL=0 is the full gather: identical bits, also on a
    second right-hand side (nothing stale is read)."""
    prob, sol, ref = one_patch
    rng = np.random.default_rng(5)
    for r in (prob.rhs(), rng.uniform(-1, 1, prob.ndof)):
        z_local = np.array(sol.smooth(r), copy=True)
        os.environ["FDMGPU_SMOOTH_LOCAL"] = "0"
        try:
            z_full = np.array(sol.smooth(r), copy=True)
        finally:
            del os.environ["FDMGPU_SMOOTH_LOCAL"]
        assert np.array_equal(z_local, z_full)
        assert rel(z_local, ref.smooth(r)) <= TOL_RELAX


def test_p31_two_level_and_pcg_match_oracle(one_patch, torch):
    prob, sol, ref = one_patch
    w = sol.calibrate_damping()
    ref.build_twolevel()
    tl = ref.twolevel_info()
    assert abs(w["omega"] - tl["omega"]) <= 1e-10 * tl["omega"]
    assert abs(w["lambda_max"] - tl["lambda_max"]) <= 1e-10 * tl["lambda_max"]
    r = prob.rhs()
    assert rel(sol.vcycle(r), ref.vcycle(r)) <= TOL_RELAX
    x, rep = sol.pcg(torch.from_numpy(r).cuda(), rtol=1e-8, maxit=200)
    xr, rr = ref.pcg(r, rtol=1e-8, maxit=200)
    assert rep["converged"] and rep["iterations"] == rr["iterations"]
    assert abs(rep["kappa"] - rr["kappa"]) <= 1e-8 * rr["kappa"]
    assert rel(x.cpu().numpy(), xr) <= 1e-9


def test_c5_sampled_patch_solves_match_oracle(pkg, oracle, torch):
    """Full C5: 2-3 patches (corner, centre, last) solved on the device against the
    oracle's factors of the same patches, factored on the fly in parallel."""
    prob = pkg.Problem(5)
    sol = pkg.Solver(prob)
    sol.factor()
    ref = oracle.Problem(5, build_global=False, threads=os.cpu_count())
    sample = [0, 171, 342]
    ref.factor(sample, threads=len(sample))
    pt = ref.patches()
    gp = prob.patches()
    rng = np.random.default_rng(5)
    for j in sample:
        assert np.array_equal(pt["dofs"][pt["ptr"][j]:pt["ptr"][j + 1]], gp["dofs"][gp["ptr"][j]:gp["ptr"][j + 1]])
        n = int(ref.patches_n(j))
        rj = rng.uniform(-1, 1, n)
        x_ref = ref.patch_solve_one(j, rj)
        x_gpu = sol.patch_solve_one(j, rj)
        assert rel(x_gpu, x_ref) <= TOL_RELAX, (j, rel(x_gpu, x_ref))
    # the batched relaxation at full size: symmetric, linear, deterministic
    con = prob.maps()["constrained"].astype(bool)
    x, y = rng.standard_normal(prob.ndof), rng.standard_normal(prob.ndof)
    x[con] = y[con] = 0
    Px, Py = sol.smooth(x), sol.smooth(y)
    assert abs(x @ Py - y @ Px) <= 1e-12 * abs(x @ Py)
    assert np.array_equal(sol.smooth(x), Px)
