"""GPU parity of the SIPG-DG device path (second half)
against the oracle's restatement of src/sipg.cpp (oracle/sipg.cpp).

The two-level DG solver of tests/test_sipg.cpp:184-197 on the device:
dg_poisson_operator (src/sipg.cpp:176-250) as A, the vertex-star patches of
transformed_dg_poisson (src/sipg.cpp:252-364, (2p+2)^d DOFs each) as the
relaxation, the continuous Q1 coarse level with build_prolongation from the DG
space.  Tolerances as tests/test_gpu_parity.py: S, S^T, A rel-l2 <= 1e-12;
patch solve, relaxation, V-cycle <= 1e-11; omega <= 1e-10; identical PCG
counts; patch lists bit-exact."""
import json
import os

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu
CASES = [(2, 4, 4, False), (2, 3, 3, True), (2, 4, 7, False), (3, 3, 3, False), (3, 2, 5, False)]


@pytest.fixture(scope="module")
def torch():
    import torch as T

    assert T.cuda.is_available(), "GPU tests need a CUDA device"
    return T


@pytest.fixture(scope="module", params=CASES, ids=lambda c: "d%d_n%d_p%d%s" % (c[0], c[1], c[2], "_skip" if c[3] else ""))
def dg_pair(request, pkg, oracle, torch):
    dim, n, p, skip = request.param
    prob = pkg.Problem.sipg(dim, n, p, skip_boundary_patches=skip)
    sol = pkg.Solver(prob)
    sol.factor()
    ref = oracle.DGProblem(dim, n, p, skip_boundary_patches=skip, threads=os.cpu_count())
    ref.build(calibrate=True)
    return prob, sol, ref


def test_dg_setup_matches_oracle(dg_pair):
    prob, sol, ref = dg_pair
    assert prob.ndof == ref.ndof
    assert rel(prob.rhs(), ref.rhs()) <= 1e-14  # load_vector(f = 1)
    pt, gp = ref.patches(), prob.patches()
    assert np.array_equal(pt["vertex"], gp["vertex"]) and np.array_equal(pt["ptr"], gp["ptr"])
    assert np.array_equal(pt["dofs"], gp["dofs"])
    L = sol.layout()
    full = (2 * prob.p + 2) ** prob.dim
    assert L["n"] == full and L["n_interior"] == 0 and L["n_interface"] == full
    # the shared symbolic factor (the first full star's patch_ordering, by position)
    # equals the reference cholesky's factor of that star
    sizes = np.diff(pt["ptr"])
    first_full = int(np.flatnonzero(sizes == full)[0])
    assert L["nnz_L"] == pt["nnz"][first_full]


def test_dg_rejects_cg_only_entries(pkg, dg_pair):
    prob, sol, ref = dg_pair
    with pytest.raises(pkg.FdmGpuError, match="scalar CG handles only"):
        sol.patch_schur(0)
    with pytest.raises(pkg.FdmGpuError, match="scalar CG handles only"):
        sol.patch_solve_one(0, np.zeros(10))


def test_dg_operators_match_oracle(dg_pair):
    prob, sol, ref = dg_pair
    rng = np.random.default_rng(prob.p)
    x = rng.uniform(-1, 1, prob.ndof)
    assert rel(sol.apply_A(x), ref.apply("A", x)) <= 1e-12
    assert rel(sol.apply_St(x), ref.apply("St", x)) <= 1e-12
    assert rel(sol.apply_S(x), ref.apply("S", x)) <= 1e-12
    xt = ref.apply("St", x)
    assert rel(sol.patch_apply(xt), ref.op("patch", xt)) <= 1e-11
    assert rel(sol.smooth(x), ref.op("smooth", x)) <= 1e-11


def test_dg_two_level_matches_oracle(dg_pair, torch):
    prob, sol, ref = dg_pair
    w = sol.calibrate_damping()
    b = prob.rhs()
    xr, rr = ref.pcg(b, 1e-8, 200)
    assert abs(w["omega"] - rr["omega"]) <= 1e-10 * rr["omega"]
    sol.omega = rr["omega"]
    assert rel(sol.vcycle(b), ref.op("vcycle", b)) <= 1e-11
    x, rep = sol.pcg(torch.from_numpy(b).cuda(), rtol=1e-8, maxit=200)
    assert rep["converged"] and rep["iterations"] == rr["iterations"]
    assert abs(rep["kappa"] - rr["kappa"]) <= 1e-8 * rr["kappa"]
    assert rel(x.cpu().numpy(), xr) <= 1e-9
    if (prob.dim, prob.n, prob.p) == (2, 4, 4) and not prob.skip_boundary_patches:
        g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "variants", "dg_two_level.json")))
        assert rep["iterations"] == g["iterations"] == 8 and prob.npatches == g["npatches"]
        assert abs(np.linalg.norm(x.cpu().numpy()) - g["x_norm"]) <= 1e-9 * g["x_norm"]
